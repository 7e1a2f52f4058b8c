"""The reference's own known-answer and property checks on this path
(pkg/tests/test_contrast.py, test_solver.py and acceptance
criterion 1), restated against the CUDA path (GPU).

Each case cites the reference test it mirrors; the assertions are the
reference's, with the exact integer comparisons it uses."""

import numpy as np
import pytest

from conftest import random_batch
from oracle import oracle as orc
import paper_2209_13168_b200 as evd
from paper_2209_13168_b200.events import EventBatch, SensorGeometry
from paper_2209_13168_b200.geometry import VelocityInterval, velocity_domain

pytestmark = pytest.mark.gpu


def _batch(x, y, t, w=16, h=16, tau=0.5):
    f = lambda a: np.asarray(a, dtype=np.float64)
    return EventBatch(f(x), f(y), f(t), tau, SensorGeometry(w, h))


def test_single_event_lands_in_its_pixel():
    """test_contrast.py:47-53: one event at rest bins to counts[row, col]."""
    img = evd.accumulate_image(_batch([3.4], [5.6], [0.2]), 0.0)
    assert img.counts[5, 3] == 1 and img.counts.sum() == 1 and img.in_image_events == 1


def test_contrast_known_answer_and_brute_force():
    """test_contrast.py:86-90 and brute_force_variance (:38-43): the contrast of
    a known image is its population variance."""
    # four events on one pixel, none elsewhere, of a 2x2 sensor: H = [4, 0, 0, 0],
    # mean 1, variance (9 + 1 + 1 + 1) / 4 = 3
    img = evd.accumulate_image(_batch([0.5] * 4, [0.5] * 4, [0.1] * 4, 2, 2), 0.0)
    assert evd.image_contrast(img) == 3.0
    r = np.random.default_rng(7)
    b = random_batch(r, 16, 16, 300)
    img = evd.accumulate_image(b, -0.3)
    h = img.counts.astype(np.float64)
    assert abs(evd.image_contrast(img) - np.mean((h - h.mean()) ** 2)) < 1e-12
    assert evd.image_contrast(img) == orc.contrast_at(b, -0.3)


def test_singleton_interval_bound_equals_point_image():
    """test_contrast.py:145-150: for lo == hi the upper-bound image is the point
    image, exactly."""
    b = random_batch(np.random.default_rng(11), 32, 32, 800)
    for nu in (-1.2, -0.4, 0.0):
        ub = evd.upper_bound_image(b, VelocityInterval(nu, nu))
        assert np.array_equal(ub.counts, evd.accumulate_image(b, nu).counts)


def test_long_segment_marks_each_pixel_once():
    """test_contrast.py:152-165: one event sweeping many pixels marks each at
    most once (the per-event dedup)."""
    b = _batch([15.3], [14.7], [0.0], 32, 32)
    ub = evd.upper_bound_image(b, velocity_domain(0.5))
    assert ub.counts.max() == 1 and ub.counts.sum() > 10


def test_refinement_is_monotone():
    """test_contrast.py:172-180: a sub-interval's bound image is pointwise <=."""
    b = random_batch(np.random.default_rng(12), 48, 40, 1500)
    outer = VelocityInterval(-1.5, -0.1)
    inner = VelocityInterval(-1.0, -0.6)
    assert (evd.upper_bound_image(b, inner).counts <= evd.upper_bound_image(b, outer).counts).all()
    assert evd.bound_terms(b, inner).c_bar <= evd.bound_terms(b, outer).c_bar + 1e-12


def test_all_inside_mu_lower():
    """test_contrast.py:192-200: events that stay inside the frame over the
    interval give mu_lower = N / M."""
    r = np.random.default_rng(13)
    n = 200
    b = _batch(r.uniform(28, 36, n), r.uniform(28, 36, n), r.uniform(0, 0.5, n), 64, 64)
    cb = evd.bound_terms(b, VelocityInterval(-0.2, 0.0))
    assert cb.mu_lower == n / (64 * 64)


def test_flat_objective_stops_at_the_root():
    """test_solver.py:21-29: events at t = tau do not move with nu, so the
    contrast is flat, the root's gap is 0 and the solve stops at once with the
    domain centre."""
    r = np.random.default_rng(14)
    b = _batch(r.uniform(0, 32, 400), r.uniform(0, 32, 400), np.full(400, 0.5), 32, 32)
    res = evd.maximise_contrast_bnb(b, evd.SolverParams())
    dom = velocity_domain(0.5)
    assert res.iterations == 1 and res.nu == dom.center


def test_solver_is_deterministic():
    """test_solver.py:52-58."""
    b = random_batch(np.random.default_rng(15), 64, 64, 2000)
    a1 = evd.maximise_contrast_bnb(b, evd.SolverParams())
    a2 = evd.maximise_contrast_bnb(b, evd.SolverParams())
    assert (a1.nu, a1.contrast, a1.iterations) == (a2.nu, a2.contrast, a2.iterations)


def test_acceptance_criterion_1_bound_validity():
    """test_acceptance.py:49-81: 1,000 random (batch, interval, nu) cases at
    64x64, N in [50, 2000]: H_bar >= H as int64, mu_lower <= mu + 1e-12,
    c_bar >= C - 1e-9."""
    r = np.random.default_rng(20230)
    dom = velocity_domain(0.5)
    viol = 0
    for _ in range(1000):
        b = random_batch(r, 64, 64, int(r.integers(50, 2001)))
        lo, hi = np.sort(r.uniform(dom.lo, dom.hi, 2))
        nu = float(r.uniform(lo, hi))
        iv = VelocityInterval(float(lo), float(hi))
        ub = evd.upper_bound_image(b, iv).counts.astype(np.int64)
        pt = evd.accumulate_image(b, nu)
        cb = evd.bound_terms(b, iv)
        ok = ((ub >= pt.counts.astype(np.int64)).all()
              and cb.mu_lower <= pt.in_image_events / (64 * 64) + 1e-12
              and cb.c_bar >= evd.image_contrast(pt) - 1e-9)
        viol += not ok
    assert viol == 0
