"""Synthetic ventral-descent event windows for benchmarks and parity tests.

Host-side input generator, NOT part of the product hot path.  It restates the
reference simulator's trajectory model (``pkg/src/eventdiv/simulator.py:74-145``)
with the per-scene-point Python loop vectorised; every floating-point
operation is the same elementwise IEEE operation in the same order, so the
generated streams are bit-identical to ``generate_landing_events`` for the
noise-free configurations used here (checked by ``tests/test_host.py`` against
fixtures produced by the reference itself).

Configurations follow SURVEY.md §8(d).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .events import EventBatch, EventStream, SensorGeometry, window_bounds


@dataclass(frozen=True)
class Descent:
    """Constant-velocity descent over a textured plane (``simulator.py:23-50``)."""

    width: int
    height: int
    n_points: int
    nu: float = -0.4
    z0: float = 1.0
    duration: float = 2.0
    spacing_px: float = 1.0
    seed: int = 0


def landing_stream(d: Descent) -> EventStream:
    """Events of every scene point crossing each ``spacing_px`` radial step.

    Restates ``simulator.py:74-107`` (trajectories, out-of-frame truncation)
    and ``:112-140`` (time sort, polarity draw) for the noise-free case.
    """
    rng = np.random.default_rng(d.seed)
    g = SensorGeometry(d.width, d.height)
    cx, cy = d.width / 2.0, d.height / 2.0
    px0 = rng.uniform(-cx, cx, size=d.n_points)
    py0 = rng.uniform(-cy, cy, size=d.n_points)
    r0 = np.hypot(px0, py0)
    if d.nu == 0:
        x = y = t = np.empty(0)
    else:
        z_end = d.z0 + d.nu * d.duration
        grow = d.z0 / z_end
        # steps per point; a point at the FOE (r0 == 0) never emits
        safe_r0 = np.where(r0 == 0.0, 1.0, r0)
        kmax = np.floor((safe_r0 * grow - safe_r0) / d.spacing_px).astype(np.int64)
        kmax[(r0 == 0.0) | (kmax < 1)] = 0
        owner = np.repeat(np.arange(d.n_points), kmax)
        first = np.cumsum(kmax) - kmax
        step = (np.arange(owner.size) - np.repeat(first, kmax) + 1).astype(np.float64)
        r0e = r0[owner]
        rk = r0e + d.spacing_px * step
        tk = (d.z0 / d.nu) * (r0e - rk) / rk
        scale = rk / r0e
        ex = cx + px0[owner] * scale
        ey = cy + py0[owner] * scale
        inside = (ex >= 0) & (ex < d.width) & (ey >= 0) & (ey < d.height)
        # radius grows monotonically: keep each point's prefix up to its first exit
        bad = np.concatenate([[0], np.cumsum(~inside)])
        keep = (bad[1:] - bad[first][owner]) == 0
        x, y, t = ex[keep], ey[keep], tk[keep]
    pol = rng.choice(np.array([-1, 1], dtype=np.int8), size=len(x))
    order = np.argsort(t, kind="stable")
    return EventStream(x[order], y[order], t[order], pol[order], g)


def concat_streams(streams: list[EventStream], period: float) -> EventStream:
    """One time-sorted stream from several, stream i shifted by i * period
    (a long landing sequence for the stream pipeline; each part must end
    before ``period``)."""
    g = streams[0].geometry
    parts = [(s.x, s.y, s.t + i * period, s.polarity) for i, s in enumerate(streams)]
    cat = lambda k: np.concatenate([p[k] for p in parts])
    return EventStream(cat(0), cat(1), cat(2), cat(3), g)


def stream_windows(stream: EventStream, tau: float = 0.5) -> list[EventBatch]:
    """All windows of a stream (including empty ones), as ``batch_stream``."""
    k0, bounds = window_bounds(stream.t, tau)
    out = []
    for j, (lo, hi) in enumerate(bounds):
        start = (k0 + j) * tau
        out.append(EventBatch(stream.x[lo:hi].copy(), stream.y[lo:hi].copy(),
                              np.minimum(stream.t[lo:hi] - start, tau), tau,
                              stream.geometry, t_start=start))
    return out


# SURVEY.md §8(d) recipes: window 0 of batch_stream(stream, 0.5)
CONFIGS = {
    1: Descent(240, 180, 1450, spacing_px=1.0),
    2: Descent(346, 260, 10000, spacing_px=1.0),
    3: Descent(640, 480, 13000, spacing_px=0.5),
    5: Descent(1280, 720, 38000, spacing_px=0.5),
}


def config_window(cfg: int, tau: float = 0.5) -> EventBatch:
    """Window 0 of the named configuration (N = 20,219 / 204,203 / 999,557 / 5,327,641)."""
    return stream_windows(landing_stream(CONFIGS[cfg]), tau)[0]


def sequence_descent(k: int, n_windows: int = 2000) -> Descent:
    """Window k of the cfg-4 landing sequence (SURVEY.md §8(d) cfg 4)."""
    nu_k = -0.1 - 0.6 * k / (n_windows - 1)
    n_points = int(round(1450 * 0.25 / (1.0 / (1.0 + nu_k * 0.5) - 1.0)))
    return Descent(240, 180, n_points, nu=nu_k, duration=0.5, seed=1000 + k)


def sequence_window(k: int, n_windows: int = 2000) -> EventBatch:
    return stream_windows(landing_stream(sequence_descent(k, n_windows)))[0]


def random_window(rng: np.random.Generator, width=64, height=64, n=500, tau=0.5) -> EventBatch:
    """Uniform events with no scene structure (reference ``tests/conftest.py:21-26``)."""
    x = rng.uniform(0, width, n)
    y = rng.uniform(0, height, n)
    t = np.sort(rng.uniform(0, tau, n))
    return EventBatch(x, y, t, tau, SensorGeometry(width, height))
