"""Edge geometries and solver settings against the CPU oracle (GPU).

Degenerate and skinny sensors (1x1, 1xN, Nx1, tiny primes), events exactly on
pixel edges and on the frame border, other window lengths and solver
parameters: images, contrast bits, bound integers and BnB results must equal
the oracle's (which is pinned to the reference, tests/test_oracle.py)."""

import numpy as np
import pytest

from oracle import oracle as orc
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200 import contrast as con, solver as sol
from paper_2209_13168_b200.events import EventBatch, SensorGeometry
from paper_2209_13168_b200.geometry import velocity_domain

pytestmark = pytest.mark.gpu

GEOMS = [(1, 1), (1, 37), (53, 1), (7, 5), (127, 3), (2, 128), (64, 64)]


def _batch(rng, w, h, n=400, tau=0.5):
    x = rng.uniform(0, w, n)
    y = rng.uniform(0, h, n)
    # a quarter of the events on pixel edges / the frame border
    k = n // 4
    x[:k] = rng.integers(0, w + 1, k).astype(np.float64)
    y[k:2 * k] = rng.integers(0, h + 1, k).astype(np.float64)
    x = np.minimum(x, np.nextafter(float(w), 0.0))
    y = np.minimum(y, np.nextafter(float(h), 0.0))
    t = np.sort(rng.uniform(0, tau, n))
    t[:3] = 0.0
    t[-3:] = tau
    return EventBatch(x, y, t, tau, SensorGeometry(w, h))


@pytest.mark.parametrize("w,h", GEOMS)
def test_images_and_bounds_vs_oracle(w, h):
    rng = np.random.default_rng(w * 1000 + h)
    b = _batch(rng, w, h)
    dom = velocity_domain(b.tau)
    nus = [dom.center, -0.4, 0.0, dom.lo, -1.0]
    inside, contrast, counts = con.point_terms(b, nus, images=True)
    for j, nu in enumerate(nus):
        oc, oin = orc.point_image(b, nu)
        assert np.array_equal(counts[j], oc) and int(inside[j]) == oin
        assert contrast[j] == orc.image_contrast(oc, oin)
    ivs = [(dom.lo, dom.hi), (dom.lo, dom.center), (-0.5, -0.3), (-0.4, -0.4 + 1e-7),
           (-1.0, -0.99)]
    s, fi, marks, cnt = con.bound_terms_many(b, [a for a, _ in ivs], [c for _, c in ivs],
                                             images=True)
    for j, (lo, hi) in enumerate(ivs):
        oc, ofi = orc.bound_image(b, lo, hi)
        assert np.array_equal(cnt[j], oc), (w, h, lo, hi)
        assert int(fi[j]) == ofi and int(marks[j]) == int(oc.sum())
        assert int(s[j]) == int((oc.astype(np.uint64) ** 2).sum())


@pytest.mark.parametrize("w,h", GEOMS)
def test_bnb_vs_oracle(w, h):
    rng = np.random.default_rng(7 + w * 31 + h)
    b = _batch(rng, w, h, n=300)
    r = evd.maximise_contrast_bnb(b, evd.SolverParams())
    o = orc.maximise_contrast_bnb(b)
    assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (o.nu, o.contrast, o.bound_gap,
                                                             o.iterations)


@pytest.mark.parametrize("gamma,tau,mw", [(0.1, 0.5, 1e-9), (0.001, 0.5, 1e-9), (0.025, 0.25, 1e-9),
                                          (0.025, 1.0, 1e-9), (0.001, 0.5, 1e-3)])
def test_solver_parameters_vs_oracle(gamma, tau, mw):
    rng = np.random.default_rng(int(gamma * 1e4) + int(tau * 100))
    b = _batch(rng, 48, 36, n=600, tau=tau)
    p = evd.SolverParams(gamma=gamma, tau=tau, min_interval_width=mw)
    r = evd.maximise_contrast_bnb(b, p)
    o = orc.maximise_contrast_bnb(b, gamma=gamma, min_interval_width=mw)
    assert (r.nu, r.contrast, r.bound_gap, r.iterations) == (o.nu, o.contrast, o.bound_gap,
                                                             o.iterations)


def test_windows_mixed_sizes_vs_single():
    """One grouped launch over windows from 1 to ~20k events equals per-window solves."""
    rng = np.random.default_rng(3)
    bs = [_batch(rng, 60, 45, n=n) for n in (1, 2, 5, 50, 700, 5000, 20000)]
    res, _, _ = sol.solve_windows(bs, evd.SolverParams(), groups=3)
    for b, r in zip(bs, res):
        one = evd.maximise_contrast_bnb(b, evd.SolverParams())
        assert r.status == 0
        assert (r.nu, r.contrast, r.bound_gap, int(r.iterations)) == (
            one.nu, one.contrast, one.bound_gap, one.iterations)
