"""Randomised parity stress of the whole solve (GPU) against the pinned oracle:
sensor sizes, window sizes, solver parameters and adversarial coordinates
(integer and half-integer positions, duplicates, t at 0 and tau, events off
the frame) drawn from fixed seeds.  Bar: every BnbResult field identical
(runtime excepted), and the same bound images for random intervals."""

import numpy as np
import pytest

from oracle import oracle as orc
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import contrast as con, synth
from paper_2209_13168_b200.events import EventBatch, SensorGeometry
from paper_2209_13168_b200.geometry import velocity_domain

pytestmark = pytest.mark.gpu


def _window(r: np.random.Generator, case: int) -> EventBatch:
    w, h = int(r.integers(3, 160)), int(r.integers(3, 120))
    tau = float(r.choice([0.25, 0.5, 1.0]))
    n = int(r.integers(1, 4000))
    kind = case % 5
    if kind == 0:    # uniform
        x, y = r.uniform(0, w, n), r.uniform(0, h, n)
    elif kind == 1:  # integer and half-integer positions (pixel edges, corners)
        x = r.integers(0, w + 1, n) + r.choice([0.0, 0.5], n)
        y = r.integers(0, h + 1, n) + r.choice([0.0, 0.5], n)
    elif kind == 2:  # heavy duplicates
        k = max(1, n // 20)
        idx = r.integers(0, k, n)
        x, y = r.uniform(0, w, k)[idx], r.uniform(0, h, k)[idx]
    elif kind == 3:  # partly off the frame
        x, y = r.uniform(-0.3 * w, 1.3 * w, n), r.uniform(-0.3 * h, 1.3 * h, n)
    else:            # a small radial-flow descent
        d = synth.Descent(w, h, int(r.integers(20, 300)), nu=float(r.uniform(-0.8, -0.1)),
                          duration=tau, seed=int(r.integers(0, 1 << 30)))
        s = synth.landing_stream(d)
        keep = s.t <= tau
        x, y, t = s.x[keep], s.y[keep], s.t[keep]
        if t.size == 0:
            x, y, t = np.array([w / 2.0 + 0.3]), np.array([h / 2.0 + 0.3]), np.array([0.0])
        return EventBatch(np.ascontiguousarray(x), np.ascontiguousarray(y),
                          np.ascontiguousarray(t), tau, SensorGeometry(w, h))
    t = np.sort(r.uniform(0, tau, n))
    t[: max(1, n // 50)] = 0.0
    t[-max(1, n // 50):] = tau
    return EventBatch(x.astype(np.float64), y.astype(np.float64), t, tau, SensorGeometry(w, h))


@pytest.mark.parametrize("seed", range(12))
def test_random_windows_solve_like_the_oracle(seed):
    r = np.random.default_rng(777 + seed)
    for case in range(20):
        b = _window(r, case)
        gamma = float(r.choice([0.001, 0.025, 0.2]))
        p = evd.SolverParams(gamma=gamma)
        got = evd.maximise_contrast_bnb(b, p)
        ref = orc.maximise_contrast_bnb(b, gamma=gamma)
        assert (got.nu, got.contrast, got.bound_gap, got.iterations) == (
            ref.nu, ref.contrast, ref.bound_gap, ref.iterations), (seed, case, b.n)


@pytest.mark.parametrize("seed", range(3))
def test_random_bound_images_like_the_oracle(seed):
    r = np.random.default_rng(4242 + seed)
    for case in range(10):
        b = _window(r, case)
        dom = velocity_domain(b.tau)
        lo, hi = np.sort(r.uniform(dom.lo, dom.hi, (8, 2)), axis=1).T
        lo[0], hi[0] = dom.lo, dom.hi           # the root
        hi[1] = lo[1]                           # a singleton
        _, fi, marks, ims = con.bound_terms_many(b, lo, hi, images=True)
        for j in range(lo.size):
            ref_counts, ref_fi = orc.bound_image(b, float(lo[j]), float(hi[j]))
            assert np.array_equal(ims[j], ref_counts), (seed, case, j)
            assert fi[j] == ref_fi and marks[j] == ref_counts.sum(dtype=np.uint64)


@pytest.mark.parametrize("seed", range(3))
def test_random_frontiers_like_the_oracle(seed):
    """The batched frontier (filtered first pass: off-frame / one-cell /
    edge-adjacent certification, exact path for the rest) on adversarial
    windows and uniform leaves of depth 3-9, against the oracle's integers."""
    from paper_2209_13168_b200 import frontier as fr
    r = np.random.default_rng(9090 + seed)
    for case in range(10):
        b = _window(r, case)
        depth = int(r.integers(3, 10))
        lo, hi = fr.uniform_frontier(velocity_domain(b.tau), depth)
        pick = np.sort(r.choice(lo.size, min(lo.size, 40), replace=False))
        lo, hi = lo[pick], hi[pick]
        s_bar, fi, marks = con.frontier_terms(b, lo, hi)
        for j in range(lo.size):
            counts, ref_fi = orc.bound_image(b, float(lo[j]), float(hi[j]))
            c64 = counts.astype(np.uint64)
            assert (int(s_bar[j]), int(fi[j]), int(marks[j])) == (
                int((c64 * c64).sum()), ref_fi, int(c64.sum())), (seed, case, j)
