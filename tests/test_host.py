"""Host-side logic: input contract, windowing, interval arithmetic, synth (CPU)."""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2209_13168_b200 import events as ev
from paper_2209_13168_b200 import geometry as geo
from paper_2209_13168_b200 import synth
from paper_2209_13168_b200.solver import SolverParams


def test_synth_matches_reference_simulator():
    with open(os.path.join(GOLDEN, "synth.json")) as fh:
        ref = json.load(fh)
    for cfg, want in ref.items():
        b = synth.config_window(int(cfg))
        h = hashlib.sha256(b.x.tobytes() + b.y.tobytes() + b.t.tobytes()).hexdigest()
        assert b.n == want["n"] and h == want["sha256"], cfg


def test_config_sizes():
    assert synth.config_window(1).n == 20219
    assert synth.sequence_window(0).n == 23539 and synth.sequence_window(1999).n == 15495


def test_batch_stream_windows_and_gaps(rng):
    t = np.sort(np.concatenate([rng.uniform(0, 0.5, 50), rng.uniform(2.5, 3.0, 50)]))
    s = ev.EventStream(rng.uniform(0, 8, 100), rng.uniform(0, 8, 100), t,
                       np.ones(100, dtype=np.int8), ev.SensorGeometry(8, 8))
    bs = ev.batch_stream(s, 0.5)
    assert len(bs) == 6 and [b.n for b in bs] == [50, 0, 0, 0, 0, 50]
    assert bs[-1].t_start == 2.5 and bs[-1].t_end == 3.0
    assert all((b.t >= 0).all() and (b.t <= 0.5).all() for b in bs)


def test_stream_validation():
    g = ev.SensorGeometry(4, 4)
    with pytest.raises(ev.EventValidationError):
        ev.EventStream(np.array([1.0]), np.array([5.0]), np.array([0.0]),
                       np.array([1], dtype=np.int8), g)
    with pytest.raises(ev.EventValidationError):
        ev.EventStream(np.array([1.0, 1.0]), np.array([1.0, 1.0]), np.array([0.2, 0.1]),
                       np.array([1, 1], dtype=np.int8), g)
    with pytest.raises(ev.EventValidationError):
        ev.EventBatch(np.array([1.0]), np.array([1.0]), np.array([0.7]), 0.5, g)
    with pytest.raises(ev.EventValidationError):
        ev.SensorGeometry(0, 3)


def test_velocity_interval():
    lo, hi = geo.VelocityInterval(-1.0, 0.0).split()
    assert lo == geo.VelocityInterval(-1.0, -0.5) and hi == geo.VelocityInterval(-0.5, 0.0)
    with pytest.raises(ValueError):
        geo.VelocityInterval(0.0, -1.0)
    assert geo.velocity_domain(0.5).lo == -(1.0 - 1e-6) / 0.5
    assert geo.velocity_domain(1.0, 0.0).lo == -1.0
    with pytest.raises(ValueError):
        geo.velocity_domain(0.0)
    with pytest.raises(ValueError):
        geo.velocity_domain(0.5, 1.0)


def test_divergence_formulas(rng):
    assert geo.divergence_from_velocity(0.0, 0.5) == 0.0
    assert geo.divergence_from_velocity(-0.9, 1.0) == pytest.approx(-9.0)
    nus = np.sort(rng.uniform(-1.9, 0, 50))
    ds = [geo.divergence_from_velocity(float(n), 0.5) for n in nus]
    assert np.all(np.diff(ds) > 0)
    with pytest.raises(geo.CheiralityError):
        geo.divergence_from_velocity(-2.0, 0.5)
    assert geo.continuous_divergence(-0.2, 2.0, 5.0) == pytest.approx(-0.2)
    with pytest.raises(geo.CheiralityError):
        geo.continuous_divergence(-0.5, 1.0, 3.0)


def test_solver_params_validation():
    with pytest.raises(ValueError):
        SolverParams(gamma=0.0)
    with pytest.raises(ValueError):
        SolverParams(tau=-1.0)
