"""Best-first branch and bound over the velocity interval, run on the device.

Drop-in for ``pkg/src/eventdiv/solver.py``.  ``maximise_contrast_bnb`` makes a
single ``evd_solve`` call: the whole best-first loop (solver.py:79-123) --
centre contrast, both child bounds, incumbent update with ``>=``, pruning with
``>=``, FIFO tie-break on equal bounds, the gamma / minimum-width stop and the
iteration cap -- executes inside one persistent cooperative kernel, so the
result (nu, contrast, bound_gap, iterations) is the reference's, bit for bit.
"""

from __future__ import annotations

import logging
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


def solve_window(batch: EventBatch, params: SolverParams, ctx=None) -> tuple[BnbResult, SolveStats]:
    """maximise_contrast_bnb plus explored-node statistics."""
    if batch.n == 0:
        raise NoEventsError("no events in batch")
    start = time.perf_counter()
    velocity_domain(batch.tau, params.epsilon)  # ValueError on bad tau / epsilon (geometry.py:63-66)
    ctx = load_window(batch, ctx)
    res, launches = solve_loaded(ctx, params)
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


def estimate_stream_divergence(batches: list[EventBatch], params: SolverParams
                               ) -> list[DivergenceSample]:
    """BnB per window; empty windows leave a gap (solver.py:139-162)."""
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
