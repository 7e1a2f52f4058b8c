"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2209_13168_b200.events import EventBatch, SensorGeometry  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libevd.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def f64(hexbits: str) -> float:
    return float(np.frombuffer(bytes.fromhex(hexbits), dtype=np.float64)[0])


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


@pytest.fixture(scope="session")
def seg_golden():
    return dict(np.load(os.path.join(GOLDEN, "segments.npz")))


@pytest.fixture(scope="session")
def img_golden():
    with open(os.path.join(GOLDEN, "images.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, "images.npz")))
    cases = []
    for m in meta:
        name = m["name"]
        batch = EventBatch(arrays[f"{name}/x"], arrays[f"{name}/y"], arrays[f"{name}/t"],
                           f64(m["tau"]), SensorGeometry(m["width"], m["height"]))
        cases.append((m, batch, {k.split("/", 1)[1]: v for k, v in arrays.items()
                                 if k.startswith(name + "/")}))
    return cases


@pytest.fixture(scope="session")
def bnb_golden():
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        meta = json.load(fh)
    arrays = dict(np.load(os.path.join(GOLDEN, "bnb_windows.npz")))
    windows = []
    for j, w in enumerate(meta["small"]):
        windows.append((w, EventBatch(arrays[f"w{j}/x"], arrays[f"w{j}/y"], arrays[f"w{j}/t"],
                                      f64(w["tau"]), SensorGeometry(w["width"], w["height"]),
                                      t_start=f64(w["t_start"]))))
    return meta, windows


def golden_segment_sets(g):
    """[(segment, (w, h), set of pixels)] from segments.npz."""
    out = []
    offs, pix = g["offsets"], g["pixels"]
    for j, s in enumerate(g["segs"]):
        cells = {(int(a), int(b)) for a, b in pix[offs[j]:offs[j + 1]]}
        out.append((s, tuple(int(v) for v in g["dims"][j]), cells))
    return out


def random_batch(rng, width=64, height=64, n=500, tau=0.5):
    """Uniform events, no scene structure (reference tests/conftest.py:21-26)."""
    x = rng.uniform(0, width, n)
    y = rng.uniform(0, height, n)
    t = np.sort(rng.uniform(0, tau, n))
    return EventBatch(x, y, t, tau, SensorGeometry(width, height))
