"""Pin the CPU oracle to fixtures produced by the reference itself (CPU only).

The oracle (oracle/) is the checker of the CUDA path; before trusting it, it
must reproduce every golden vector the reference generated
(tests/golden/make_golden.py) bit for bit.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, f64, golden_segment_sets
from oracle import oracle as orc


def test_segments_match_reference(seg_golden):
    bad = 0
    for seg, (w, h), cells in golden_segment_sets(seg_golden):
        if orc.rasterize_segment(seg[:2], seg[2:], w, h) != cells:
            bad += 1
    assert bad == 0


def test_point_images_and_contrast(img_golden):
    for meta, batch, arr in img_golden:
        for j, p in enumerate(meta["points"]):
            counts, inside = orc.point_image(batch, f64(p["nu"]))
            assert np.array_equal(counts, arr[f"point{j}"]), (meta["name"], j)
            assert inside == p["in_image"]
            assert orc.image_contrast(counts, inside) == f64(p["contrast"])


def test_bound_images_and_terms(img_golden):
    for meta, batch, arr in img_golden:
        m = meta["width"] * meta["height"]
        for j, b in enumerate(meta["bounds"]):
            s_bar, mu_lower, c_bar, fi, counts = orc.bound_terms(batch, f64(b["lo"]), f64(b["hi"]))
            assert np.array_equal(counts, arr[f"bound{j}"]), (meta["name"], j)
            assert fi == b["fully_inside"]
            assert int(counts.sum()) == b["marks"]
            assert s_bar == f64(b["s_bar"]) and mu_lower == f64(b["mu_lower"])
            assert c_bar == f64(b["c_bar"])
            assert fi / m == f64(b["mu_lower"])


def test_bnb_small_windows(bnb_golden):
    meta, windows = bnb_golden
    for w, batch in windows:
        r = orc.maximise_contrast_bnb(batch)
        ref = w["result"]
        assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (
            f64(ref["nu"]), f64(ref["contrast"]), f64(ref["bound_gap"]), ref["iterations"])


def test_bnb_config1():
    from paper_2209_13168_b200 import synth
    import json, os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        ref = json.load(fh)["configs"]["1"]["result"]
    orc.THREADS = 4
    try:
        r = orc.maximise_contrast_bnb(synth.config_window(1))
    finally:
        orc.THREADS = 1
    assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (
        f64(ref["nu"]), f64(ref["contrast"]), f64(ref["bound_gap"]), ref["iterations"])


def test_grid_search(bnb_golden):
    meta, windows = bnb_golden
    for g in meta["grid"]:
        nu, c = orc.grid_search(windows[g["window"]][1], g["n_points"])
        assert (nu, c) == (f64(g["nu"]), f64(g["c"]))


@pytest.mark.parametrize("m", list(range(1, 140)) + [255, 256, 257, 1000, 43200, 89960])
def test_pairwise_restatement_matches_numpy(m):
    r = np.random.default_rng(m)
    a = (r.integers(0, 9, m).astype(np.float64) - r.random()) ** 2
    assert orc.pairwise_sum(a) == np.sum(a)


def test_multithreaded_oracle_is_deterministic(img_golden):
    meta, batch, arr = img_golden[3]
    b = meta["bounds"][0]
    c1, f1 = orc.bound_image(batch, f64(b["lo"]), f64(b["hi"]))
    orc.THREADS = 5
    try:
        c5, f5 = orc.bound_image(batch, f64(b["lo"]), f64(b["hi"]))
    finally:
        orc.THREADS = 1
    assert np.array_equal(c1, c5) and f1 == f5


def _evd1_golden():
    z = np.load(os.path.join(GOLDEN, "evd1.npz"))
    return z, json.loads(bytes(z["meta"]).decode())


def test_evd1_oracle_matches_reference_parser():
    z, meta = _evd1_golden()
    for name in meta["valid"]:
        x, y, t, p, geom = orc.parse_bin(z[f"{name}_data"].tobytes())
        for k, v in (("x", x), ("y", y), ("t", t), ("p", p)):
            assert np.array_equal(v, z[f"{name}_{k}"]), (name, k)
            assert v.dtype == z[f"{name}_{k}"].dtype
        assert list(geom) == z[f"{name}_geom"].tolist()
    cls = {"EventFormatError": orc.FormatError, "EventValidationError": orc.ValidationError}
    for name, (kind, msg) in meta["invalid"].items():
        with pytest.raises(cls[kind]) as ei:
            orc.parse_bin(z[f"bad_{name}_data"].tobytes())
        assert str(ei.value) == msg


def _preproc_golden():
    z = np.load(os.path.join(GOLDEN, "preproc.npz"))
    return z, json.loads(bytes(z["meta"]).decode())


def test_preprocessing_oracle_matches_reference():
    z, meta = _preproc_golden()
    for c in meta["hot"]:
        n = c["name"]
        x, y, t, p = (z[f"{n}_{k}"] for k in ("x", "y", "t", "p"))
        assert np.array_equal(orc.pixel_counts(x, y, c["w"], c["h"]), z[f"{n}_counts"])
        kx, ky, kt, kp, thr = orc.remove_hot_pixels(x, y, t, p, c["w"], c["h"], c["k"])
        for got, key in ((kx, "kx"), (ky, "ky"), (kt, "kt"), (kp, "kp")):
            assert np.array_equal(got, z[f"{n}_{key}"]), (n, key)
        assert thr == f64(c["threshold"])
    for c in meta["rescale"]:
        n = c["name"]
        rx, ry = orc.rescale(z[f"{n}_x"], z[f"{n}_y"], c["w"], c["h"], c["w2"], c["h2"])
        assert np.array_equal(rx, z[f"{n}_rx"]) and np.array_equal(ry, z[f"{n}_ry"])


def test_cfg3_frontier_golden_sample():
    """frontier_cfg3.npz holds the reference's own bound of all 4096 depth-12
    leaves of the 999,557-event cfg-3 window (make_golden.py frontier); the
    leaves are the bisection's endpoints, and the oracle agrees on a sample."""
    from paper_2209_13168_b200 import frontier as fr, synth
    from paper_2209_13168_b200.geometry import velocity_domain
    g = np.load(os.path.join(GOLDEN, "frontier_cfg3.npz"))
    lo, hi = fr.uniform_frontier(velocity_domain(0.5), 12)
    assert np.array_equal(lo, g["lo"]) and np.array_equal(hi, g["hi"])
    assert int(g["marks"].sum()) == 1787442891
    b = synth.config_window(3)
    orc.THREADS = os.cpu_count() or 1
    try:
        for j in (0, 700, 1500, 2600, 3300, 4095):
            counts, fi = orc.bound_image(b, lo[j], hi[j])
            c = counts.astype(np.uint64)
            assert fi == int(g["fully_inside"][j]), j
            assert int(c.sum()) == int(g["marks"][j]), j
            assert int((c * c).sum()) == int(g["s_bar"][j]), j
    finally:
        orc.THREADS = 1
