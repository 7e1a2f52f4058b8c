"""Parity of the CUDA path (through the C ABI) with the reference (GPU).

Bar: bit-exact for every integer image, count and bound, and for every
float64 contrast / c_bar bit pattern; BnbResult fields identical (runtime
excepted).  Checked against fixtures made by the reference itself
(tests/golden/) and, on fresh seeded inputs, against the pinned CPU oracle.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, f64, golden_segment_sets, random_batch
from oracle import oracle as orc
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import _lib, contrast as con, solver as sol, synth
from paper_2209_13168_b200.events import EventBatch, SensorGeometry
from paper_2209_13168_b200.geometry import VelocityInterval, velocity_domain

pytestmark = pytest.mark.gpu


def test_native_library_is_loaded():
    ctx = _lib.context()
    assert ctx.sms > 0
    with open("/proc/self/maps") as fh:
        assert _lib.LIB_PATH in fh.read()


# ------------------------------------------------------------------ raster
@pytest.mark.parametrize("chunk", [0, 1, 2, 3, 7])
def test_segments_match_reference(seg_golden, chunk):
    """Every chunk size (seams between lanes) gives the reference's pixel sets."""
    by_dims = {}
    for seg, dims, cells in golden_segment_sets(seg_golden):
        by_dims.setdefault(dims, []).append((seg, cells))
    bad = 0
    for (w, h), items in by_dims.items():
        got = con.rasterize_segments([s for s, _ in items], SensorGeometry(w, h), chunk=chunk)
        bad += sum(g != c for g, (_, c) in zip(got, items))
    assert bad == 0


def test_fresh_adversarial_segments_vs_oracle():
    r = np.random.default_rng(99)
    g = SensorGeometry(32, 24)
    segs = np.concatenate([
        r.uniform(-4, 36, (6000, 4)),
        r.integers(-2, 35, (3000, 4)).astype(float),
        np.round(r.uniform(-2, 34, (2000, 4)) * 2) / 2,
    ])
    got = con.rasterize_segments(segs, g)
    bad = sum(got[j] != orc.rasterize_segment(s[:2], s[2:], 32, 24) for j, s in enumerate(segs))
    assert bad == 0


def test_reference_raster_examples():
    g = SensorGeometry(8, 8)
    assert evd.rasterize_segment((2.5, 2.5), (2.5, 2.5), g) == {(2, 2)}
    assert evd.rasterize_segment((0.5, 0.5), (2.5, 0.5), g) == {(0, 0), (1, 0), (2, 0)}
    assert evd.rasterize_segment((-5.0, -5.0), (-1.0, -2.0), g) == set()
    px = evd.rasterize_segment((3.0, 3.0), (5.0, 5.0), g)
    assert {(3, 3), (4, 4), (3, 4), (4, 3)} <= px


# ------------------------------------------------------------------ images
def test_point_images_and_contrast_bits(img_golden):
    for meta, batch, arr in img_golden:
        for j, p in enumerate(meta["points"]):
            nu = f64(p["nu"])
            img = evd.accumulate_image(batch, nu)
            assert np.array_equal(img.counts, arr[f"point{j}"].astype(np.float64)), (meta["name"], j)
            assert img.in_image_events == p["in_image"]
            assert evd.contrast_at(batch, nu) == f64(p["contrast"])
            assert evd.image_contrast(img) == f64(p["contrast"])
            assert evd.image_contrast_expanded(img) == f64(p["contrast_expanded"])


def test_bound_images_and_terms_bits(img_golden):
    for meta, batch, arr in img_golden:
        for j, b in enumerate(meta["bounds"]):
            iv = VelocityInterval(f64(b["lo"]), f64(b["hi"]))
            ub = evd.upper_bound_image(batch, iv)
            assert np.array_equal(ub.counts, arr[f"bound{j}"].astype(np.float64)), (meta["name"], j)
            assert ub.in_image_events == b["marks"]
            bt = evd.bound_terms(batch, iv)
            assert (bt.s_bar, bt.mu_lower, bt.c_bar) == (
                f64(b["s_bar"]), f64(b["mu_lower"]), f64(b["c_bar"])), (meta["name"], j)


def test_batched_bounds_equal_single_calls(img_golden):
    meta, batch, arr = img_golden[0]
    lo = [f64(b["lo"]) for b in meta["bounds"]]
    hi = [f64(b["hi"]) for b in meta["bounds"]]
    s, fi, marks, counts = con.bound_terms_many(batch, lo, hi, images=True)
    for j, b in enumerate(meta["bounds"]):
        assert np.array_equal(counts[j], arr[f"bound{j}"])
        assert int(fi[j]) == b["fully_inside"] and int(marks[j]) == b["marks"]
        assert float(s[j]) == f64(b["s_bar"])


def test_full_size_bound_images_vs_oracle():
    """Whole (batch, interval) images at config-1 size, incl. the near-singular root."""
    b = synth.config_window(1)
    dom = velocity_domain(b.tau)
    ivs = [(dom.lo, dom.hi), dom.split()[0], (dom.lo, dom.lo + 1e-3), (-0.45, -0.35),
           (-0.40001, -0.39999), (-0.4, -0.4), (-1.5, -1.2)]
    ivs = [(iv.lo, iv.hi) if isinstance(iv, VelocityInterval) else iv for iv in ivs]
    s, fi, marks, counts = con.bound_terms_many(b, [a for a, _ in ivs], [c for _, c in ivs],
                                                images=True)
    orc.THREADS = 8
    try:
        for j, (lo, hi) in enumerate(ivs):
            oc, ofi = orc.bound_image(b, lo, hi)
            assert np.array_equal(counts[j], oc), (lo, hi)
            assert int(fi[j]) == ofi and int(marks[j]) == int(oc.sum())
            assert int(s[j]) == int((oc.astype(np.uint64) ** 2).sum())
    finally:
        orc.THREADS = 1


def test_warp_bits_vs_oracle():
    b = synth.config_window(1)
    for nu in (0.0, -0.4, -1.999998, -1e-300, -0.7):
        x, y = evd.warp_batch(b, nu)
        ox, oy = orc.warp(b.x, b.y, b.t, nu, b.tau, 240, 180)
        assert np.array_equal(x, ox) and np.array_equal(y, oy)
    s = evd.warp_scale(b.t, -0.4, 0.5)
    assert np.array_equal(s, (1.0 + -0.4 * b.t) / (1.0 + -0.4 * 0.5))


# ------------------------------------------------------------------ solver
def _same(r, ref):
    return (r.nu, r.contrast, r.bound_gap, r.iterations) == (
        f64(ref["nu"]), f64(ref["contrast"]), f64(ref["bound_gap"]), ref["iterations"])


def test_bnb_small_windows(bnb_golden):
    meta, windows = bnb_golden
    for w, batch in windows:
        r = evd.maximise_contrast_bnb(batch, evd.SolverParams())
        assert _same(r, w["result"]), w["result"]


@pytest.mark.parametrize("path", ["0", "1"])
def test_bnb_both_event_paths(bnb_golden, monkeypatch, path):
    """The solve kernel's exact-only and filtered (approximate warp, exact
    fallback) event paths, forced on every golden window and config 1/2."""
    monkeypatch.setenv("EVD_SOLVE_FILTER", path)
    meta, windows = bnb_golden
    for w, batch in windows:
        assert _same(evd.maximise_contrast_bnb(batch, evd.SolverParams()), w["result"])
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        cfgs = json.load(fh)["configs"]
    for cfg in ("1", "2"):
        r, st = sol.solve_window(synth.config_window(int(cfg)), evd.SolverParams())
        assert _same(r, cfgs[cfg]["result"])


@pytest.mark.parametrize("k", ["1", "2", "4"])
def test_bnb_speculative_rounds(bnb_golden, monkeypatch, k):
    """Speculative rounds (k_solve_spec, up to k node evaluations per round) and
    the one-node kernel give the reference's results on every golden window,
    configs 1-2 and the grouped window solver."""
    monkeypatch.setenv("EVD_SPEC_K", k)
    meta, windows = bnb_golden
    for w, batch in windows:
        assert _same(evd.maximise_contrast_bnb(batch, evd.SolverParams()), w["result"])
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        gold = json.load(fh)
    for cfg in ("1", "2"):
        r, st = sol.solve_window(synth.config_window(int(cfg)), evd.SolverParams())
        assert _same(r, gold["configs"][cfg]["result"])
    seq = gold["sequence"]
    res, _, _ = sol.solve_windows([synth.sequence_window(s["k"]) for s in seq],
                                  evd.SolverParams(), groups=2)
    for r, s in zip(res, seq):
        assert r.status == 0 and _same(r, s["result"])


@pytest.mark.parametrize("block", ["384", "512", "768"])
@pytest.mark.parametrize("k", ["1", "2"])
def test_bnb_every_block_size(bnb_golden, monkeypatch, block, k):
    """Each CTA size the solve kernels are built at (384 / 512 / 768 threads,
    with and without speculative rounds) gives the reference's results."""
    monkeypatch.setenv("EVD_SOLVE_BLOCK", block)
    monkeypatch.setenv("EVD_SPEC_K", k)
    meta, windows = bnb_golden
    for w, batch in windows:
        assert _same(evd.maximise_contrast_bnb(batch, evd.SolverParams()), w["result"])
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        gold = json.load(fh)
    for cfg in ("1", "2"):
        r, st = sol.solve_window(synth.config_window(int(cfg)), evd.SolverParams())
        assert _same(r, gold["configs"][cfg]["result"])


def test_bnb_trace_nodes(bnb_golden):
    """Every node the reference evaluated: centre contrast and both child c_bar bits."""
    meta, windows = bnb_golden
    for w, batch in windows[:4]:
        m = batch.geometry.n_pixels
        nodes = [n for n in w["trace"] if n["kind"] == "node"]
        if not nodes:
            continue
        los = [f64(n["lo"]) for n in nodes]
        his = [f64(n["hi"]) for n in nodes]
        cs = [0.5 * (a + b) for a, b in zip(los, his)]
        _, contrast, _ = con.point_terms(batch, cs)
        s, fi, _, _ = con.bound_terms_many(batch, los + cs, cs + his)
        k = len(nodes)
        for j, n in enumerate(nodes):
            assert contrast[j] == f64(n["c_center"])
            for side, idx in ((0, j), (1, k + j)):
                cb = con.assemble_bound(int(s[idx]), int(fi[idx]), m)
                assert cb.c_bar == f64(n["children"][side]["c_bar"])


@pytest.mark.parametrize("cfg", ["1", "2"])
def test_bnb_configs(cfg):
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        ref = json.load(fh)["configs"][cfg]
    b = synth.config_window(int(cfg))
    assert b.n == ref["n"]
    r, stats = sol.solve_window(b, evd.SolverParams())
    assert _same(r, ref["result"])
    assert stats.bound_evals == 1 + 2 * (r.iterations - 1) or stats.bound_evals <= 2 * r.iterations + 1


def test_bnb_config3_if_golden():
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        ref = json.load(fh)["configs"].get("3")
    if ref is None:
        pytest.skip("config-3 golden not generated")
    b = synth.config_window(3)
    r = evd.maximise_contrast_bnb(b, evd.SolverParams())
    assert _same(r, ref["result"])


def test_bnb_config5_vs_reference():
    """Config 5 (1280x720, 5.33 M events; 768-thread CTAs): the reference's own
    result, measured once in this container (BASELINE.md, 1,791 s on one
    core): nu_hat, C(nu_hat) and the gap bit for bit, 144 iterations."""
    b = synth.config_window(5)
    r = evd.maximise_contrast_bnb(b, evd.SolverParams())
    assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (
        -0.4000001722040176, 753.9103765755924, 0.015945095486131322, 144)


def test_sequence_windows(bnb_golden):
    meta, _ = bnb_golden
    for s in meta["sequence"]:
        b = synth.sequence_window(s["k"])
        assert b.n == s["n"]
        assert _same(evd.maximise_contrast_bnb(b, evd.SolverParams()), s["result"])


def test_grid_search(bnb_golden):
    meta, windows = bnb_golden
    for g in meta["grid"]:
        nu, c = evd.grid_search_oracle(windows[g["window"]][1], evd.SolverParams(), g["n_points"])
        assert (nu, c) == (f64(g["nu"]), f64(g["c"]))


def test_iteration_limit(bnb_golden):
    meta, windows = bnb_golden
    lim = meta["iteration_limit"]
    with pytest.raises(evd.IterationLimitError) as err:
        evd.maximise_contrast_bnb(windows[lim["window"]][1],
                                  evd.SolverParams(max_iterations=lim["max_iterations"]))
    e = err.value
    assert (e.nu, e.contrast, e.iterations) == (f64(lim["nu"]), f64(lim["contrast"]),
                                                lim["iterations"])


def test_errors():
    g = SensorGeometry(8, 8)
    empty = EventBatch(np.empty(0), np.empty(0), np.empty(0), 0.5, g)
    with pytest.raises(evd.NoEventsError):
        evd.maximise_contrast_bnb(empty, evd.SolverParams())
    one = EventBatch(np.array([3.0]), np.array([3.0]), np.array([0.1]), 0.5, g)
    with pytest.raises(evd.CheiralityError):
        evd.maximise_contrast_bnb(one, evd.SolverParams(epsilon=0.0))
    with pytest.raises(evd.CheiralityError):
        evd.radial_warp(1.0, 1.0, 0.0, nu=-2.0, tau=0.5, geometry=SensorGeometry(100, 100))
    with pytest.raises(evd.CheiralityError):
        evd.bound_terms(one, VelocityInterval(-2.5, 0.0))


def test_stream_driver_gaps(rng):
    n = 400
    t = np.sort(np.concatenate([rng.uniform(0, 0.5, n), rng.uniform(2.5, 3.0, n)]))
    s = evd.EventStream(rng.uniform(0, 64, 2 * n), rng.uniform(0, 64, 2 * n), t,
                        np.ones(2 * n, dtype=np.int8), SensorGeometry(64, 64))
    samples = evd.estimate_stream_divergence(evd.batch_stream(s, 0.5), evd.SolverParams())
    assert [x.t for x in samples] == [0.5, 3.0]
    for x, b in zip(samples, [b for b in evd.batch_stream(s, 0.5) if b.n]):
        r = orc.maximise_contrast_bnb(b)
        assert (x.contrast, x.iterations) == (r.contrast, r.iterations)
        assert x.divergence == evd.divergence_from_velocity(r.nu, 0.5)


# ------------------------------------------------------------------ properties at full size
@pytest.mark.parametrize("cfg", [2])
def test_bound_validity_properties_full_size(cfg):
    """Size-independent properties at BASELINE sizes: H_bar >= H for nu in the
    interval, monotone refinement, singleton equality, marks == sum(H_bar)."""
    b = synth.config_window(cfg)
    r = np.random.default_rng(cfg)
    dom = velocity_domain(b.tau)
    for _ in range(4):
        lo, hi = np.sort(r.uniform(dom.lo, dom.hi, 2))
        ilo, ihi = np.sort(r.uniform(lo, hi, 2))
        nu = float(r.uniform(ilo, ihi))
        _, fi, marks, ims = con.bound_terms_many(b, [lo, ilo, nu], [hi, ihi, nu], images=True)
        ins, _, pim = con.point_terms(b, [nu], images=True, with_contrast=False)
        assert (ims[1] <= ims[0]).all() and (pim[0] <= ims[1]).all()
        assert np.array_equal(ims[2], pim[0])
        assert [int(ims[j].sum(dtype=np.uint64)) for j in range(3)] == [int(m) for m in marks]
        assert fi[2] == ins[0]


@pytest.mark.parametrize("k", ["1", "4"])
@pytest.mark.parametrize("cert", ["on", "off"])
def test_root_certificate(bnb_golden, monkeypatch, cert, k, rng):
    """The speculative solve certifies the root bound (S >= (sum of per-event
    cell lower bounds)^2 / M) instead of rasterising it; a window whose
    certificate fails (few events: the bound is not provably above c_hat +
    gamma) is rerun with the root rasterised.  Results equal the reference's
    either way, in both solve kernels, including iteration limits at the root
    and a root narrower than min_interval_width (whose exact bound is the
    reported bound_gap); grouped many-window solves too."""
    if cert == "off":
        monkeypatch.setenv("EVD_NO_ROOT_CERT", "1")
    monkeypatch.setenv("EVD_SPEC_K", k)  # 1: k_solve, 4: k_solve_spec
    meta, windows = bnb_golden
    for w, batch in windows:
        assert _same(evd.maximise_contrast_bnb(batch, evd.SolverParams()), w["result"])
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        gold = json.load(fh)
    for cfg in ("1", "2"):
        r, st = sol.solve_window(synth.config_window(int(cfg)), evd.SolverParams())
        assert _same(r, gold["configs"][cfg]["result"])
    # certificate failures: 1-6 events, and a dense tiny frame
    for n in (1, 2, 3, 6):
        b = random_batch(rng, 16, 12, n)
        o = orc.maximise_contrast_bnb(b)
        r = evd.maximise_contrast_bnb(b, evd.SolverParams())
        assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (o.nu, o.contrast, o.bound_gap,
                                                                 o.iterations)
    b = synth.config_window(1)
    with pytest.raises(evd.IterationLimitError) as err:
        evd.maximise_contrast_bnb(b, evd.SolverParams(max_iterations=1))
    o = orc.maximise_contrast_bnb(b, max_iterations=1)
    assert (err.value.nu, err.value.contrast, err.value.iterations) == (o.nu, o.contrast, 1)
    seq = gold["sequence"]
    wins = [synth.sequence_window(q["k"]) for q in seq]
    w0 = wins[0]
    tiny = EventBatch(w0.x[:2], w0.y[:2], w0.t[:2], w0.tau, w0.geometry)  # certificate fails
    res, _, _ = sol.solve_windows(wins + [tiny], evd.SolverParams(), groups=3)
    for r, q in zip(res, seq):
        assert r.status == 0 and _same(r, q["result"])
    o = orc.maximise_contrast_bnb(tiny)
    assert (res[-1].nu, res[-1].contrast, res[-1].iterations) == (o.nu, o.contrast, o.iterations)
    small = windows[0][1]
    r = evd.maximise_contrast_bnb(small, evd.SolverParams(min_interval_width=3.0))
    o = orc.maximise_contrast_bnb(small, min_interval_width=3.0)
    assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (o.nu, o.contrast, o.bound_gap, 1)


def test_node_terms_vs_oracle(rng):
    """evd_eval_nodes (the solve kernel's rounds without the search): the
    centre contrast and both children's c_bar of k nodes, bit-identical to the
    reference's contrast_at / bound_terms, for k = 1, 3, 4, 9 (several rounds
    of slots) on a golden-sized window and a random one; inadmissible
    endpoints raise like the reference."""
    from paper_2209_13168_b200.geometry import CheiralityError
    for b in (synth.config_window(1), random_batch(rng, 40, 30, 700)):
        dom = velocity_domain(b.tau)
        for k in (1, 3, 4, 9):
            lo = rng.uniform(dom.lo, dom.hi, k)
            hi = np.minimum(lo + rng.choice([1e-6, 1e-3, 0.1, 1.0], k), dom.hi)
            con_, ca, cb = con.node_terms(b, lo, hi)
            for j in range(k):
                c = 0.5 * (lo[j] + hi[j])
                assert con_[j] == orc.contrast_at(b, c)
                assert ca[j] == orc.bound_terms(b, lo[j], c)[2]
                assert cb[j] == orc.bound_terms(b, c, hi[j])[2]
    with pytest.raises(CheiralityError):
        con.node_terms(b, [-2.5], [-0.1])


def test_solve_events_sources(bnb_golden):
    """evd_solve_events (maximise_contrast_bnb's one-call path) from pageable
    host, pinned host and device arrays gives the reference's result, leaves
    the window resident for the per-call entry points, and reports an empty
    window like the reference."""
    import ctypes
    import torch
    with open(os.path.join(GOLDEN, "bnb.json")) as fh:
        ref = json.load(fh)["configs"]["1"]["result"]
    b = synth.config_window(1)
    g = b.geometry
    ctx = _lib.context()
    p = evd.SolverParams()
    r, _ = sol.solve_events(ctx, b, p)  # pageable numpy arrays
    assert _same(r, ref)
    sp = _lib.SolveParams(p.gamma, p.epsilon, p.min_interval_width, p.max_iterations)
    ptr = lambda v: ctypes.cast(v.data_ptr(), ctypes.POINTER(ctypes.c_double))
    for kind in ("pinned", "device"):
        ts = {k: torch.from_numpy(np.ascontiguousarray(getattr(b, k))) for k in "xyt"}
        ts = {k: (v.pin_memory() if kind == "pinned" else v.cuda()) for k, v in ts.items()}
        torch.cuda.synchronize()
        res = _lib.SolveResult()
        rc = ctx.lib.evd_solve_events(ctx.h, ptr(ts["x"]), ptr(ts["y"]), ptr(ts["t"]), b.n,
                                      g.width, g.height, b.tau, sp, res)
        assert rc == 0 and _same(res, ref), kind
    # the window stays resident: a per-call bound on it needs no upload
    dom = velocity_domain(b.tau)
    sb, fi, _ = con.frontier_terms(b, [dom.lo], [dom.center], ctx=ctx, loaded=True)
    o = orc.bound_terms(b, dom.lo, dom.center)
    assert float(sb[0]) == o[0] and int(fi[0]) == o[3]
    empty = EventBatch(np.empty(0), np.empty(0), np.empty(0), 0.5, SensorGeometry(8, 8))
    with pytest.raises(evd.NoEventsError):
        evd.maximise_contrast_bnb(empty, p)
