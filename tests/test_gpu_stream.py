"""Whole-stream pipeline on the device (evd_solve_stream)
against the host pipeline estimate_stream_divergence(batch_stream(...)), which
the window tests pin to the reference, and against the CPU oracle."""

import numpy as np
import pytest

from oracle import oracle as orc
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import synth
from paper_2209_13168_b200.events import EventStream
from paper_2209_13168_b200.geometry import divergence_from_velocity

pytestmark = pytest.mark.gpu


def _key(samples):
    return [(s.t, s.divergence, s.contrast, s.bound_gap, s.iterations) for s in samples]


def _stream(n_desc=3, w=96, h=72, pts=300, seed=5):
    parts = [synth.landing_stream(synth.Descent(w, h, pts, nu=-0.1 - 0.15 * i, duration=2.0,
                                                seed=seed + i)) for i in range(n_desc)]
    return synth.concat_streams(parts, 2.0)


@pytest.mark.parametrize("tau", [0.5, 0.3, 0.7])
def test_stream_matches_host_pipeline(tau):
    s = _stream()
    params = evd.SolverParams(tau=tau)
    host = evd.estimate_stream_divergence(evd.batch_stream(s, tau), params)
    dev = evd.stream_divergence(s, params)
    assert len(dev) > 4
    assert _key(dev) == _key(host)


def test_stream_matches_oracle():
    s = _stream(n_desc=2, w=64, h=48, pts=150)
    params = evd.SolverParams()
    dev = evd.stream_divergence(s, params)
    ref = []
    for b in evd.batch_stream(s, 0.5):
        if b.n == 0:
            continue
        r = orc.maximise_contrast_bnb(b)
        ref.append((b.t_end, divergence_from_velocity(r.nu, b.tau), r.contrast, r.bound_gap,
                    r.iterations))
    assert _key(dev) == ref


def test_stream_gaps_offset_start_and_iteration_limit():
    s = _stream()
    keep = (s.t < 1.2) | (s.t >= 2.9)  # windows [1.5, 2.0), [2.0, 2.5) become empty
    keep &= s.t >= 0.6                 # stream starts in window k0 = 1
    g = EventStream(s.x[keep], s.y[keep], s.t[keep], s.polarity[keep], s.geometry)
    for params in (evd.SolverParams(), evd.SolverParams(max_iterations=3)):
        host = evd.estimate_stream_divergence(evd.batch_stream(g, 0.5), params)
        dev = evd.stream_divergence(g, params)
        assert _key(dev) == _key(host)
    assert evd.stream_divergence(EventStream(np.empty(0), np.empty(0), np.empty(0),
                                             np.empty(0), s.geometry), evd.SolverParams()) == []


# ------------------------------------------------------------------ EVD1 files
def _evd1():
    import json
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "evd1.npz"))
    return z, json.loads(bytes(z["meta"]).decode())


def _resident_bound(ctx, lo=-1.2, hi=-0.4):
    """bound_terms of one interval over the context's resident window set."""
    import ctypes
    from paper_2209_13168_b200 import _lib
    out = [np.zeros(1, dtype=np.uint64), np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.uint64)]
    lo_a, hi_a = np.array([lo]), np.array([hi])
    rc = ctx.lib.evd_bound_images(ctx.h, _lib.ptr(lo_a), _lib.ptr(hi_a), 1,
                                  _lib.ptr(out[0], _lib._u64p), _lib.ptr(out[1], _lib._i64p),
                                  _lib.ptr(out[2], _lib._u64p), ctypes.POINTER(ctypes.c_uint32)())
    assert rc == 0
    return [int(a[0]) for a in out]


@pytest.mark.parametrize("chunk", [1024, 5000, 1 << 16])
def test_stream_overlapped_upload(chunk):
    """Host arrays: the raw stream is uploaded in chunks while the solve runs
    (each window's group waits for its events); samples and the resident
    window set equal the upload-then-solve path's, for pageable and pinned
    inputs, with gaps and an offset start."""
    import torch
    from paper_2209_13168_b200 import _lib
    s = _stream(n_desc=4)
    keep = ((s.t < 1.2) | (s.t >= 2.9)) & (s.t >= 0.6)
    g = EventStream(s.x[keep], s.y[keep], s.t[keep], s.polarity[keep], s.geometry)
    params = evd.SolverParams()
    ctx = _lib.Context(0)
    ctx.set_option("stream_overlap", 0)
    want = _key(evd.stream_divergence(g, params, ctx=ctx))
    want_res = _resident_bound(ctx)
    ctx.set_option("stream_overlap", 1)
    ctx.set_option("stream_chunk", chunk)
    got = evd.stream_divergence(g, params, ctx=ctx)
    assert _key(got) == want
    assert _resident_bound(ctx) == want_res
    pinned = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (g.x, g.y, g.t)]
    gp = EventStream(*(p.numpy() for p in pinned), g.polarity, g.geometry)
    assert _key(evd.stream_divergence(gp, params, ctx=ctx)) == want
    assert _resident_bound(ctx) == want_res
    with pytest.raises(_lib.EvdError):
        ctx.set_option("stream_chunk", 10)


def test_parse_event_bin_matches_reference():
    z, meta = _evd1()
    for name in meta["valid"]:
        s = evd.parse_event_bin(z[f"{name}_data"].tobytes())
        for k, attr in (("x", "x"), ("y", "y"), ("t", "t"), ("p", "polarity")):
            assert np.array_equal(getattr(s, attr), z[f"{name}_{k}"]), (name, k)
        assert [s.geometry.width, s.geometry.height] == z[f"{name}_geom"].tolist()
    cls = {"EventFormatError": evd.EventFormatError,
           "EventValidationError": evd.EventValidationError}
    for name, (kind, msg) in meta["invalid"].items():
        with pytest.raises(cls[kind]) as ei:
            evd.parse_event_bin(z[f"bad_{name}_data"].tobytes())
        assert str(ei.value) == msg, name


def test_bin_unsorted_large_matches_oracle(rng):
    """A shuffled 200k-record file: device radix sort == numpy stable argsort."""
    import struct
    n = 200_000
    rec = np.dtype([("t_us", "<u8"), ("x", "<f4"), ("y", "<f4"), ("p", "i1")])
    r = np.empty(n, dtype=rec)
    r["t_us"] = rng.integers(0, 50_000, n)  # many ties
    r["x"], r["y"] = rng.uniform(0, 240, n), rng.uniform(0, 180, n)
    r["p"] = rng.choice([-1, 1], n)
    data = struct.pack("<4sIIQ", b"EVD1", 240, 180, n) + r.tobytes()
    x, y, t, p, _ = orc.parse_bin(data)
    s = evd.parse_event_bin(data)
    assert np.array_equal(s.x, x) and np.array_equal(s.y, y)
    assert np.array_equal(s.t, t) and np.array_equal(s.polarity, p)


def test_bin_to_samples_equals_host_pipeline(tmp_path):
    s = _stream()
    path = tmp_path / "s.bin"
    evd.write_event_bin(s, path)
    data = path.read_bytes()
    params = evd.SolverParams()
    host = evd.estimate_stream_divergence(evd.batch_stream(evd.parse_event_bin(data), 0.5),
                                          params)
    dev = evd.stream_divergence_bin(data, params)
    assert len(dev) > 4 and _key(dev) == _key(host)


# ------------------------------------------------------------------ preprocessing
def _preproc():
    import json
    import os
    from conftest import GOLDEN
    z = np.load(os.path.join(GOLDEN, "preproc.npz"))
    return z, json.loads(bytes(z["meta"]).decode())


def _as_stream(z, n, w, h):
    from paper_2209_13168_b200.events import SensorGeometry
    return EventStream(z[f"{n}_x"], z[f"{n}_y"], z[f"{n}_t"], z[f"{n}_p"], SensorGeometry(w, h))


def test_preprocessing_matches_reference():
    from paper_2209_13168_b200.events import SensorGeometry
    z, meta = _preproc()
    for c in meta["hot"]:
        n = c["name"]
        s = _as_stream(z, n, c["w"], c["h"])
        assert np.array_equal(evd.pixel_counts(s), z[f"{n}_counts"]), n
        kept = evd.remove_hot_pixels(s, k=c["k"])
        for attr, key in (("x", "kx"), ("y", "ky"), ("t", "kt"), ("polarity", "kp")):
            assert np.array_equal(getattr(kept, attr), z[f"{n}_{key}"]), (n, key)
    for c in meta["rescale"]:
        n = c["name"]
        r = evd.rescale_events(_as_stream(z, n, c["w"], c["h"]), SensorGeometry(c["w2"], c["h2"]))
        assert np.array_equal(r.x, z[f"{n}_rx"]) and np.array_equal(r.y, z[f"{n}_ry"]), n
        assert (r.geometry.width, r.geometry.height) == (c["w2"], c["h2"])
    with pytest.raises(ValueError):
        evd.remove_hot_pixels(_as_stream(z, "hot", 8, 8), k=0)


def test_bin_preprocessed_pipeline_equals_host(tmp_path):
    """EVD1 bytes -> hot-pixel removal -> rescale -> windows -> solves, all on the
    device, equals the host composition of the same steps."""
    from paper_2209_13168_b200.events import SensorGeometry
    s = _stream()
    hot = (np.abs(s.x - 10.5) < 0.5) & (np.abs(s.y - 8.5) < 0.5)
    keep = ~hot | (np.arange(s.n) % 2 == 0)
    s = EventStream(s.x[keep], s.y[keep], s.t[keep], s.polarity[keep], s.geometry)
    path = tmp_path / "s.bin"
    evd.write_event_bin(s, path)
    data = path.read_bytes()
    params = evd.SolverParams()
    target = SensorGeometry(80, 60)
    host_stream = evd.rescale_events(evd.remove_hot_pixels(evd.parse_event_bin(data), k=8.0), target)
    host = evd.estimate_stream_divergence(evd.batch_stream(host_stream, 0.5), params)
    dev = evd.stream_divergence_bin(data, params, hot_pixel_k=8.0, rescale_to=target)
    assert _key(dev) == _key(host)
