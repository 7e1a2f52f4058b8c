"""Batched frontier (one launch for many intervals) == per-interval bounds (GPU)."""

import numpy as np
import pytest

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
