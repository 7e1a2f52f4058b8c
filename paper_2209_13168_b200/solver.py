"""Best-first branch and bound over the velocity interval, run on the device.

Drop-in for ``pkg/src/eventdiv/solver.py``.  ``maximise_contrast_bnb`` makes a
single ``evd_solve`` call: the whole best-first loop (solver.py:79-123) --
centre contrast, both child bounds, incumbent update with ``>=``, pruning with
``>=``, FIFO tie-break on equal bounds, the gamma / minimum-width stop and the
iteration cap -- executes inside one persistent cooperative kernel, so the
result (nu, contrast, bound_gap, iterations) is the reference's, bit for bit.
"""

from __future__ import annotations

import ctypes
import logging
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .contrast import load_window, point_terms
from .events import EventBatch
from .geometry import (CheiralityError, DivergenceSample, divergence_from_velocity,
                       velocity_domain)

LOG = logging.getLogger(__name__)


class NoEventsError(ValueError):
    """The batch has no events (solver.py:32-33)."""


class IterationLimitError(RuntimeError):
    """Iteration cap hit; carries the incumbent (solver.py:36-46)."""

    def __init__(self, nu: float, contrast: float, iterations: int):
        super().__init__(
            f"iteration limit reached after {iterations} iterations "
            f"(best nu={nu}, contrast={contrast})")
        self.nu = nu
        self.contrast = contrast
        self.iterations = iterations


@dataclass(frozen=True)
class SolverParams:
    """Solver settings (solver.py:49-62)."""

    gamma: float = 0.025
    tau: float = 0.5
    epsilon: float = 1e-6
    max_iterations: int = 1_000_000
    min_interval_width: float = 1e-9

    def __post_init__(self):
        if self.gamma <= 0:
            raise ValueError("gamma must be positive")
        if self.tau <= 0:
            raise ValueError("tau must be positive")


@dataclass(frozen=True)
class BnbResult:
    nu: float
    contrast: float
    bound_gap: float
    iterations: int
    runtime: float


@dataclass(frozen=True)
class SolveStats:
    """Explored-node counts of one solve (reported beside the reference's iterations)."""

    iterations: int
    bound_evals: int
    point_evals: int
    max_frontier: int
    device_ms: float
    kernel_launches: int


def contrast_at(batch: EventBatch, nu: float) -> float:
    """Contrast of the motion-compensated image at one velocity (solver.py:74-76)."""
    _, c, _ = point_terms(batch, [float(nu)])
    return float(c[0])


def _raise(ctx, rc, res=None):
    if rc == _lib.EVD_ERR_ITER_LIMIT:
        raise IterationLimitError(res.nu, res.contrast, int(res.iterations))
    if rc == _lib.EVD_ERR_CHEIRALITY:
        raise CheiralityError(ctx.error_text())
    if rc == _lib.EVD_ERR_NO_EVENTS:
        raise NoEventsError("no events in batch")
    if rc == _lib.EVD_ERR_ARG:
        raise ValueError(ctx.error_text())
    raise _lib.EvdError(rc, ctx.error_text())


def solve_loaded(ctx, params: SolverParams):
    """evd_solve on the window already resident in ``ctx``; returns (SolveResult, launches)."""
    p = _lib.SolveParams(float(params.gamma), float(params.epsilon),
                         float(params.min_interval_width), int(params.max_iterations))
    res = _lib.SolveResult()
    before = ctx.launches
    rc = ctx.lib.evd_solve(ctx.h, p, res)
    if rc:
        _raise(ctx, rc, res)
    return res, ctx.launches - before


def solve_events(ctx, batch: EventBatch, params: SolverParams):
    """evd_solve_events: upload the window and solve it in one call, the
    events arriving while the solve already runs; returns (SolveResult,
    launches).  The window stays resident in ``ctx``."""
    g = batch.geometry
    x, y, t = _lib.f64(batch.x), _lib.f64(batch.y), _lib.f64(batch.t)
    p = _lib.SolveParams(float(params.gamma), float(params.epsilon),
                         float(params.min_interval_width), int(params.max_iterations))
    if os.environ.get("EVD_LIB") and not hasattr(ctx.lib, "evd_solve_events"):
        return solve_loaded(load_window(batch, ctx, cache=False), params)  # older build (A/B)
    res = _lib.SolveResult()
    ctx._resident = None
    before = ctx.launches
    rc = ctx.lib.evd_solve_events(ctx.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t), t.size, g.width,
                                  g.height, float(batch.tau), p, res)
    if rc:
        _raise(ctx, rc, res)
    return res, ctx.launches - before


def solve_window(batch: EventBatch, params: SolverParams, ctx=None) -> tuple[BnbResult, SolveStats]:
    """maximise_contrast_bnb plus explored-node statistics."""
    if batch.n == 0:
        raise NoEventsError("no events in batch")
    start = time.perf_counter()
    velocity_domain(batch.tau, params.epsilon)  # ValueError on bad tau / epsilon (geometry.py:63-66)
    res, launches = solve_events(ctx or _lib.context(), batch, params)
    runtime = time.perf_counter() - start
    return (BnbResult(res.nu, res.contrast, res.bound_gap, int(res.iterations), runtime),
            SolveStats(int(res.iterations), int(res.bound_evals), int(res.point_evals),
                       int(res.max_frontier), float(res.device_ms), int(launches)))


def maximise_contrast_bnb(batch: EventBatch, params: SolverParams) -> BnbResult:
    """Exactly maximise contrast over the admissible velocity interval (solver.py:79-123)."""
    return solve_window(batch, params)[0]


def grid_search_oracle(batch: EventBatch, params: SolverParams, n_points: int
                       ) -> tuple[float, float]:
    """Contrast maximum over a uniform velocity grid (solver.py:126-136)."""
    if n_points < 2:
        raise ValueError("n_points must be >= 2")
    domain = velocity_domain(batch.tau, params.epsilon)
    nus = np.linspace(domain.lo, domain.hi, n_points)
    _, contrasts, _ = point_terms(batch, nus)
    best = int(np.argmax(contrasts))
    return float(nus[best]), float(contrasts[best])


def solve_windows(batches: list[EventBatch], params: SolverParams, groups: int = 0, ctx=None
                  ) -> tuple[list, float, int]:
    """Solve many windows in one device launch (evd_solve_windows).

    All windows must share sensor geometry and tau (as batch_stream's do).
    Returns ([WindowResult per window], device seconds, solver groups used).
    Empty windows get status EVD_ERR_NO_EVENTS.
    """
    if not batches:
        return [], 0.0, 0
    g0, tau = batches[0].geometry, float(batches[0].tau)
    if any(b.geometry.width != g0.width or b.geometry.height != g0.height or float(b.tau) != tau
           for b in batches):
        raise ValueError("solve_windows needs windows of one geometry and tau")
    velocity_domain(tau, params.epsilon)
    sizes = np.array([b.n for b in batches], dtype=np.int64)
    ctx = ctx or _lib.context()
    # every window's arrays straight to the device while the solve runs
    # (evd_solve_windows_list: pinned staging, no host concatenation, each
    # window's solver group starts once its events have arrived)
    cols = [[_lib.f64(getattr(b, k)) for b in batches] for k in ("x", "y", "t")]
    ptrs = [(_lib._d * len(batches))(*[_lib.ptr(a) for a in col]) for col in cols]
    p = _lib.SolveParams(float(params.gamma), float(params.epsilon),
                         float(params.min_interval_width), int(params.max_iterations))
    res = (_lib.WindowResult * len(batches))()
    ms = (ctypes.c_double * 1)()
    ctx._resident = None
    rc = ctx.lib.evd_solve_windows_list(ctx.h, ptrs[0], ptrs[1], ptrs[2],
                                        _lib.ptr(sizes, _lib._i64p), len(batches), g0.width,
                                        g0.height, tau, int(groups), p, res, ms)
    if rc:
        _raise(ctx, rc)
    return list(res), ms[0] / 1e3, (res[0].groups if len(batches) else 0)


def estimate_stream_divergence(batches: list[EventBatch], params: SolverParams
                               ) -> list[DivergenceSample]:
    """BnB per window; empty windows leave a gap (solver.py:139-162).

    All non-empty windows are solved in one device launch (evd_solve_windows)
    when they share geometry and tau; each result equals maximise_contrast_bnb's.
    ``runtime`` is the launch's wall time divided evenly over its windows.
    """
    live = [b for b in batches if b.n]
    if not live:
        return []
    same = all(b.geometry.width == live[0].geometry.width and
               b.geometry.height == live[0].geometry.height and b.tau == live[0].tau
               for b in live)
    if not same:
        return _estimate_each(batches, params)
    start = time.perf_counter()
    results, _, _ = solve_windows(live, params)
    per = (time.perf_counter() - start) / len(live)
    samples = []
    for batch, r in zip(live, results):
        if r.status == _lib.EVD_ERR_ITER_LIMIT:
            LOG.warning("batch at t=%.3f s: %s", batch.t_start,
                        IterationLimitError(r.nu, r.contrast, int(r.iterations)))
            continue
        if r.status != _lib.EVD_OK:
            raise _lib.EvdError(r.status, f"window at t={batch.t_start}: status {r.status}")
        samples.append(DivergenceSample(
            t=batch.t_end,
            divergence=divergence_from_velocity(r.nu, batch.tau),
            contrast=r.contrast,
            bound_gap=r.bound_gap,
            iterations=int(r.iterations),
            runtime=per))
    return samples


def stream_divergence(stream, params: SolverParams, tau: float | None = None, groups: int = 0,
                      ctx=None) -> list[DivergenceSample]:
    """``estimate_stream_divergence(batch_stream(stream, tau), params)`` in one
    device call (evd_solve_stream): windowing (events.py:330-359) on the device,
    then every window solved in one launch.  ``tau`` defaults to ``params.tau``.

    The samples equal the host pipeline's (t = window end, divergence, contrast,
    bound_gap, iterations); empty windows leave a gap and an iteration-limited
    window is logged and skipped, as solver.py:148-160 does.  ``runtime`` is
    the call's wall time divided evenly over the solved windows.
    """
    tau = float(params.tau if tau is None else tau)
    if tau <= 0:
        raise ValueError("tau must be positive")
    n = len(stream.t)
    if n == 0:
        return []
    velocity_domain(tau, params.epsilon)
    x, y, t = _lib.f64(stream.x), _lib.f64(stream.y), _lib.f64(stream.t)
    k0 = int(np.floor(t[0] / tau))
    cap = int(np.floor(t[-1] / tau)) - k0 + 1
    ctx = ctx or _lib.context()
    g = stream.geometry
    p = _lib.SolveParams(float(params.gamma), float(params.epsilon),
                         float(params.min_interval_width), int(params.max_iterations))
    res = (_lib.WindowResult * cap)()
    nw = ctypes.c_int32()
    k0_dev = ctypes.c_int64()
    ms = (ctypes.c_double * 1)()
    start = time.perf_counter()
    rc = ctx.lib.evd_solve_stream(ctx.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t), n, g.width,
                                  g.height, tau, int(groups), p, res, cap, ctypes.byref(nw),
                                  ctypes.byref(k0_dev), ms)
    if rc:
        _raise(ctx, rc)
    return _samples(res, nw.value, k0_dev.value, tau, time.perf_counter() - start)


def stream_divergence_bin(data: bytes, params: SolverParams, tau: float | None = None,
                          groups: int = 0, hot_pixel_k: float | None = None,
                          rescale_to=None, ctx=None) -> list[DivergenceSample]:
    """EVD1 file body -> divergence samples without a host parse: the records
    are decoded on the device (evd_load_bin), optionally cleaned of hot pixels
    (``hot_pixel_k``) and rescaled (``rescale_to``, a SensorGeometry) in place,
    and the resident stream is windowed and solved there
    (evd_solve_loaded_stream).  Equals ``estimate_stream_divergence(
    batch_stream(rescale_events(remove_hot_pixels(parse_event_bin(data), k),
    target), tau), params)``."""
    from .events import load_bin_resident
    tau = float(params.tau if tau is None else tau)
    if tau <= 0:
        raise ValueError("tau must be positive")
    if hot_pixel_k is not None and hot_pixel_k <= 0:
        raise ValueError("k must be positive")
    velocity_domain(tau, params.epsilon)
    start = time.perf_counter()
    ctx, _, n = load_bin_resident(data, ctx)
    if n and hot_pixel_k is not None:
        kept, thr = ctypes.c_int64(), ctypes.c_double()
        rc = ctx.lib.evd_stream_remove_hot_pixels(ctx.h, float(hot_pixel_k), ctypes.byref(kept),
                                                  ctypes.byref(thr))
        if rc:
            _raise(ctx, rc)
        n = kept.value
    if rescale_to is not None:
        rc = ctx.lib.evd_stream_rescale(ctx.h, rescale_to.width, rescale_to.height)
        if rc:
            _raise(ctx, rc)
    if n == 0:
        return []
    return _solve_resident(ctx, tau, params, groups, start)


def _solve_resident(ctx, tau, params, groups, start):
    p = _lib.SolveParams(float(params.gamma), float(params.epsilon),
                         float(params.min_interval_width), int(params.max_iterations))
    nw = ctypes.c_int32()
    k0 = ctypes.c_int64()
    ms = (ctypes.c_double * 1)()
    cap = 64
    while True:
        res = (_lib.WindowResult * cap)()
        rc = ctx.lib.evd_solve_loaded_stream(ctx.h, tau, int(groups), p, res, cap,
                                             ctypes.byref(nw), ctypes.byref(k0), ms)
        if rc == _lib.EVD_ERR_ARG and nw.value > cap:
            cap = nw.value
            continue
        if rc:
            _raise(ctx, rc)
        break
    return _samples(res, nw.value, k0.value, tau, time.perf_counter() - start)


def _samples(res, nw, k0, tau, wall):
    solved = sum(1 for r in res[:nw] if r.status == _lib.EVD_OK)
    per = wall / max(solved, 1)
    samples = []
    for w in range(nw):
        r = res[w]
        t_start = (k0 + w) * tau  # events.py:345
        if r.status == _lib.EVD_ERR_NO_EVENTS:
            continue
        if r.status == _lib.EVD_ERR_ITER_LIMIT:
            LOG.warning("batch at t=%.3f s: %s", t_start,
                        IterationLimitError(r.nu, r.contrast, int(r.iterations)))
            continue
        if r.status != _lib.EVD_OK:
            raise _lib.EvdError(r.status, f"window at t={t_start}: status {r.status}")
        samples.append(DivergenceSample(
            t=t_start + tau, divergence=divergence_from_velocity(r.nu, tau),
            contrast=r.contrast, bound_gap=r.bound_gap, iterations=int(r.iterations),
            runtime=per))
    return samples


def _estimate_each(batches: list[EventBatch], params: SolverParams) -> list[DivergenceSample]:
    samples = []
    for batch in batches:
        if batch.n == 0:
            continue
        try:
            result = maximise_contrast_bnb(batch, params)
        except IterationLimitError as exc:
            LOG.warning("batch at t=%.3f s: %s", batch.t_start, exc)
            continue
        samples.append(DivergenceSample(
            t=batch.t_end,
            divergence=divergence_from_velocity(result.nu, batch.tau),
            contrast=result.contrast,
            bound_gap=result.bound_gap,
            iterations=result.iterations,
            runtime=result.runtime))
    return samples
