"""Windows with NaN, infinite or huge coordinates and NaN timestamps (the
reference's EventBatch checks only the t range, so they reach the path): the
CUDA path gives the reference's images, bit patterns and BnB result
(tests/golden/nonfinite.*, made by the reference itself)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, f64
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200.events import EventBatch, SensorGeometry
from paper_2209_13168_b200.geometry import VelocityInterval

pytestmark = pytest.mark.gpu


def _cases():
    with open(os.path.join(GOLDEN, "nonfinite.json")) as fh:
        meta = json.load(fh)
    arr = np.load(os.path.join(GOLDEN, "nonfinite.npz"))
    for m in meta:
        n = m["name"]
        b = EventBatch(arr[f"{n}/x"], arr[f"{n}/y"], arr[f"{n}/t"], 0.5,
                       SensorGeometry(m["width"], m["height"]))
        yield m, b, arr


def _same_bits(a, b):
    return np.float64(a).tobytes() == np.float64(b).tobytes()


def test_nonfinite_images_and_bounds():
    for m, b, arr in _cases():
        n = m["name"]
        for j, p in enumerate(m["points"]):
            img = evd.accumulate_image(b, f64(p["nu"]))
            assert np.array_equal(img.counts, arr[f"{n}/point{j}"].astype(np.float64)), (n, j)
            assert img.in_image_events == p["in_image"]
            assert _same_bits(evd.image_contrast(img), f64(p["contrast"])), (n, j)
        for j, q in enumerate(m["bounds"]):
            iv = VelocityInterval(f64(q["lo"]), f64(q["hi"]))
            ub = evd.upper_bound_image(b, iv)
            assert np.array_equal(ub.counts, arr[f"{n}/bound{j}"].astype(np.float64)), (n, j)
            assert ub.in_image_events == q["marks"]
            assert _same_bits(evd.bound_terms(b, iv).c_bar, f64(q["c_bar"])), (n, j)


def test_nonfinite_bnb():
    for m, b, _ in _cases():
        r = evd.maximise_contrast_bnb(b, evd.SolverParams())
        ref = m["result"]
        assert (_same_bits(r.nu, f64(ref["nu"])), _same_bits(r.contrast, f64(ref["contrast"])),
                r.iterations) == (True, True, ref["iterations"]), m["name"]
