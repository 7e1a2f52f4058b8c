"""Batched frontier (one launch for many intervals) == per-interval bounds (GPU)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

from oracle import oracle as orc
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import contrast as con, frontier as fr, synth
from paper_2209_13168_b200.geometry import VelocityInterval, velocity_domain

pytestmark = pytest.mark.gpu


def _check_same(b, lo, hi):
    s, fi, mk = con.frontier_terms(b, lo, hi)
    s1, fi1, mk1, _ = con.bound_terms_many(b, lo, hi)
    assert np.array_equal(s, s1) and np.array_equal(fi, fi1) and np.array_equal(mk, mk1)
    return s, fi, mk


def test_uniform_frontier_matches_split():
    dom = velocity_domain(0.5)
    lo, hi = fr.uniform_frontier(dom, 5)
    ivs = [dom]
    for _ in range(5):
        ivs = [c for iv in ivs for c in iv.split()]
    assert np.array_equal(lo, [iv.lo for iv in ivs]) and np.array_equal(hi, [iv.hi for iv in ivs])
    assert np.array_equal(lo[1:], hi[:-1])


def test_frontier_equals_single_bounds_cfg1():
    b = synth.config_window(1)
    dom = velocity_domain(b.tau)
    lo, hi = fr.uniform_frontier(dom, 7)                 # 128 adjacent leaves
    r = np.random.default_rng(5)
    rl, rh = np.sort(r.uniform(dom.lo, dom.hi, (2, 45)), axis=0)
    lo = np.concatenate([lo, rl, [dom.lo, -0.4]])       # + disjoint, root, singleton
    hi = np.concatenate([hi, rh, [dom.hi, -0.4]])
    _check_same(b, lo, hi)


def test_frontier_bounds_assembly_bits():
    b = synth.config_window(1)
    lo, hi = fr.uniform_frontier(velocity_domain(b.tau), 6)
    cb = fr.frontier_bounds(b, lo, hi)
    for j in range(0, 64, 7):
        assert cb[j] == evd.bound_terms(b, VelocityInterval(lo[j], hi[j])).c_bar


@pytest.fixture
def frontier_path():
    """Set the context's frontier path for one test; back to auto afterwards."""
    from paper_2209_13168_b200 import _lib
    ctx = _lib.context()
    yield ctx
    ctx.set_option("frontier_path", _lib.FRONTIER_AUTO)
    ctx.set_option("frontier_image_budget", 8 << 30)


@pytest.fixture(scope="module")
def cfg3():
    b = synth.config_window(3)
    assert b.n == 999557
    lo, hi = fr.uniform_frontier(velocity_domain(b.tau), 12)
    g = np.load(os.path.join(GOLDEN, "frontier_cfg3.npz"))
    assert np.array_equal(lo, g["lo"]) and np.array_equal(hi, g["hi"])
    return b, lo, hi, g


@pytest.mark.parametrize("path,budget", [("tiles", None), ("global", None),
                                         ("global_exact", None), ("global", 1000 * 307200 * 4)])
def test_cfg3_frontier_all_leaves_vs_reference(cfg3, frontier_path, path, budget):
    """BASELINE configs[2]: all 4096 depth-12 leaves of the 999,557-event
    640x480 window in one evd_eval_frontier call, every leaf's (S_bar,
    fully_inside, marks) equal to the reference's own bound_terms
    (tests/golden/frontier_cfg3.npz, numba kernel per leaf).  Every path: the
    on-chip tiles, the global-image filtered kernel, its exact-only variant,
    and the global path chunked (image budget of 1000 intervals -> 4 launches)."""
    from paper_2209_13168_b200 import _lib
    b, lo, hi, g = cfg3
    ctx = frontier_path
    code = {"tiles": _lib.FRONTIER_TILES, "global": _lib.FRONTIER_GLOBAL,
            "global_exact": _lib.FRONTIER_GLOBAL_EXACT}[path]
    ctx.set_option("frontier_path", code)
    if budget:
        ctx.set_option("frontier_image_budget", budget)
    s, fi, mk = con.frontier_terms(b, lo, hi, ctx=ctx)
    assert ctx.frontier_info()["last_path"] == code
    assert np.array_equal(fi, g["fully_inside"])
    assert np.array_equal(mk, g["marks"])
    assert np.array_equal(s, g["s_bar"])
    assert int(mk.sum()) == 1787442891


def test_cfg3_bound_images_all_leaves_vs_reference(cfg3):
    """The per-interval kernel (k_bound_image, evd_bound_images) on all 4096
    leaves against the same reference golden: an independent second device
    path for every leaf."""
    b, lo, hi, g = cfg3
    s, fi, mk, _ = con.bound_terms_many(b, lo, hi)
    assert np.array_equal(fi, g["fully_inside"]) and np.array_equal(mk, g["marks"])
    assert np.array_equal(s, g["s_bar"])


def _paths_agree(ctx, b, lo, hi):
    from paper_2209_13168_b200 import _lib
    out = {}
    for code in (_lib.FRONTIER_TILES, _lib.FRONTIER_GLOBAL):
        ctx.set_option("frontier_path", code)
        out[code] = con.frontier_terms(b, lo, hi, ctx=ctx)
        assert ctx.frontier_info()["last_path"] == code
    for a, c in zip(out[_lib.FRONTIER_TILES], out[_lib.FRONTIER_GLOBAL]):
        assert np.array_equal(a, c)
    return out[_lib.FRONTIER_TILES]


@pytest.mark.parametrize("w,h,n", [(64, 48, 3000), (65, 49, 5000), (240, 180, 20000),
                                   (347, 261, 60000), (31, 7, 800), (1280, 720, 200000)])
def test_tiled_frontier_equals_global_random(frontier_path, w, h, n):
    """Tiled (shared-memory) frontier == global-image frontier on uniform
    windows: odd / even frames (FOE on a pixel centre or corner), frames
    smaller than one tile, random intervals of every width in the domain,
    the root, adjacent leaves and singletons."""
    r = np.random.default_rng(w * 1000 + h)
    b = synth.random_window(r, w, h, n)
    dom = velocity_domain(b.tau)
    llo, lhi = fr.uniform_frontier(dom, 6)
    rl, rh = np.sort(r.uniform(dom.lo, dom.hi, (2, 70)), axis=0)
    sing = r.uniform(dom.lo, dom.hi, 5)
    lo = np.concatenate([llo, rl, [dom.lo], sing, [0.0]])
    hi = np.concatenate([lhi, rh, [dom.hi], sing, [0.0]])
    s, fi, mk = _paths_agree(frontier_path, b, lo, hi)
    assert int(mk.sum()) > 0


def test_tiled_frontier_landing_windows(frontier_path):
    """Structured windows (radial trajectories, events at the FOE, t = tau):
    cfg 1 and the cfg-2 window against the global path on a depth-8 frontier."""
    for cfg in (1, 2):
        b = synth.config_window(cfg)
        lo, hi = fr.uniform_frontier(velocity_domain(b.tau), 8)
        _paths_agree(frontier_path, b, lo, hi)
    # events exactly at the FOE and on the FOE's row / column, t = 0 and t = tau
    w, h = 64, 48
    x = np.array([32.0, 32.0, 0.0, 63.9, 32.0, 31.5, 32.5, 10.0, 32.0])
    y = np.array([24.0, 24.0, 24.0, 24.0, 0.0, 24.0, 24.0, 10.0, 47.99])
    t = np.array([0.0, 0.5, 0.1, 0.2, 0.3, 0.25, 0.5, 0.5, 0.4])
    b = evd.EventBatch(x, y, t, 0.5, evd.SensorGeometry(w, h))
    lo, hi = fr.uniform_frontier(velocity_domain(0.5), 7)
    _paths_agree(frontier_path, b, lo, hi)


def test_tiled_frontier_fallbacks(frontier_path):
    """Auto takes the global path where tiles do not apply (nu > 0, non-finite
    events) and more than 32 intervals are asked for; forcing tiles there
    fails loudly."""
    from paper_2209_13168_b200 import _lib
    ctx = frontier_path
    r = np.random.default_rng(3)
    b = synth.random_window(r, 64, 48, 2000)
    edges = np.linspace(-0.5, 0.3, 41)
    lo, hi = edges[:-1], edges[1:]   # 40 intervals, the last ones with nu > 0
    a = con.frontier_terms(b, lo, hi, ctx=ctx)
    assert ctx.frontier_info()["last_path"] == _lib.FRONTIER_GLOBAL
    c = con.bound_terms_many(b, lo, hi, ctx=ctx)
    assert all(np.array_equal(u, v) for u, v in zip(a, c[:3]))
    ctx.set_option("frontier_path", _lib.FRONTIER_TILES)
    with pytest.raises(_lib.EvdError):
        con.frontier_terms(b, lo, hi, ctx=ctx)
    x = b.x.copy()
    x[7] = np.nan
    bn = evd.EventBatch(x, b.y, b.t, b.tau, b.geometry)
    with pytest.raises(_lib.EvdError):
        con.frontier_terms(bn, [-0.5], [-0.1], ctx=ctx)
    ctx.set_option("frontier_path", _lib.FRONTIER_AUTO)
    edges = np.linspace(-1.0, -0.1, 41)
    a = con.frontier_terms(bn, edges[:-1], edges[1:], ctx=ctx)
    assert ctx.frontier_info()["last_path"] == _lib.FRONTIER_GLOBAL
    c = con.bound_terms_many(bn, edges[:-1], edges[1:], ctx=ctx)
    assert all(np.array_equal(u, v) for u, v in zip(a, c[:3]))


@pytest.mark.parametrize("k", [1, 5, 32, 33])
def test_frontier_small_k_per_interval(frontier_path, k):
    """Auto evaluates up to 32 intervals one k_bound_image pass each and more
    on the tiled kernel; both give the integers of the tiled and global paths."""
    from paper_2209_13168_b200 import _lib
    ctx = frontier_path
    r = np.random.default_rng(40 + k)
    b = synth.random_window(r, 96, 64, 5000)
    edges = np.sort(r.uniform(-1.5, 0.0, k + 1))
    lo, hi = edges[:-1], edges[1:]
    auto = con.frontier_terms(b, lo, hi, ctx=ctx)
    want = _lib.FRONTIER_PER_INTERVAL if k <= 32 else _lib.FRONTIER_TILES
    assert ctx.frontier_info()["last_path"] == want
    for code in (_lib.FRONTIER_TILES, _lib.FRONTIER_GLOBAL, _lib.FRONTIER_PER_INTERVAL):
        ctx.set_option("frontier_path", code)
        got = con.frontier_terms(b, lo, hi, ctx=ctx)
        assert ctx.frontier_info()["last_path"] == code
        assert all(np.array_equal(u, v) for u, v in zip(auto, got))
    with pytest.raises(_lib.EvdError):
        ctx.set_option("frontier_path", 5)


def test_cfg3_frontier_sample_vs_oracle():
    """Config 3 (640x480, ~1M events): the 4096-leaf frontier in one call; a
    sample of leaves checked against the pinned CPU oracle."""
    b = synth.config_window(3)
    assert b.n == 999557
    lo, hi = fr.uniform_frontier(velocity_domain(b.tau), 12)
    s, fi, mk = con.frontier_terms(b, lo, hi)
    orc.THREADS = 8
    try:
        for j in (0, 1, 1500, 2047, 2048, 2600, 3276, 4095):
            oc, ofi = orc.bound_image(b, lo[j], hi[j])
            assert int(fi[j]) == ofi and int(mk[j]) == int(oc.sum())
            assert int(s[j]) == int((oc.astype(np.uint64) ** 2).sum())
    finally:
        orc.THREADS = 1
    # size-independent property: adjacent-leaf unions bound each leaf (marks >= 0,
    # fully_inside <= events)
    assert (fi <= b.n).all()


@pytest.mark.parametrize("k", [1, 2, 30, 31, 32, 33, 62, 63, 64, 65, 97])
def test_tiled_frontier_group_edges(frontier_path, k):
    """Group boundaries of the tiled kernel (31 contiguous / 32 general
    intervals per warp): contiguous frontiers of every awkward size, the same
    intervals shuffled (non-contiguous), and zero-width intervals inside a
    contiguous run, all against the per-interval kernel."""
    from paper_2209_13168_b200 import _lib
    b = synth.random_window(np.random.default_rng(k), 96, 72, 6000)
    dom = velocity_domain(b.tau)
    edges = np.linspace(dom.lo, -0.05, k + 1)
    edges[k // 2] = edges[k // 2 + 1] if k > 2 else edges[k // 2]  # a zero-width interval
    lo, hi = edges[:-1].copy(), edges[1:].copy()
    perm = np.random.default_rng(k + 1).permutation(k)
    frontier_path.set_option("frontier_path", _lib.FRONTIER_TILES)
    for l, h in ((lo, hi), (lo[perm], hi[perm])):
        got = con.frontier_terms(b, l, h, ctx=frontier_path)
        want = con.bound_terms_many(b, l, h, ctx=frontier_path)
        assert all(np.array_equal(u, v) for u, v in zip(got, want[:3]))
