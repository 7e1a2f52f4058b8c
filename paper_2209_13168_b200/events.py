"""Input contract of the bound-evaluation hot path: sensor grid, event window, stream.

Mirrors the reference's data types so a caller holding ``eventdiv`` objects can
pass them unchanged (every entry point in this package duck-types on the fields
``x, y, t, tau, geometry.width, geometry.height``):

* ``SensorGeometry``  -- ``pkg/src/eventdiv/events.py:29-44``
* ``EventStream``     -- ``pkg/src/eventdiv/events.py:47-90`` (validation rules kept)
* ``EventBatch``      -- ``pkg/src/eventdiv/events.py:93-120``
* ``batch_stream``    -- ``pkg/src/eventdiv/events.py:330-359`` (windowing)

File parsing, hot-pixel removal, rescaling and subsampling are outside the hot
path and are not provided here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class EventValidationError(ValueError):
    """Event data violates a stream/batch invariant (``events.py:25-26``)."""


@dataclass(frozen=True)
class SensorGeometry:
    width: int
    height: int

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise EventValidationError(
                f"sensor dimensions must be positive, got {self.width}x{self.height}")

    @property
    def n_pixels(self) -> int:
        return self.width * self.height


@dataclass(frozen=True)
class EventStream:
    """Time-sorted SoA events on a sensor; invariants as ``events.py:61-81``."""

    x: np.ndarray
    y: np.ndarray
    t: np.ndarray
    polarity: np.ndarray
    geometry: SensorGeometry

    def __post_init__(self):
        n = len(self.t)
        if len(self.x) != n or len(self.y) != n or len(self.polarity) != n:
            raise EventValidationError("event arrays must have equal length")
        if n == 0:
            return
        g = self.geometry
        if not (np.isfinite(self.x).all() and np.isfinite(self.y).all()):
            raise EventValidationError("event coordinates must be finite")
        if (self.t < 0).any():
            raise EventValidationError("timestamps must be non-negative")
        if (np.diff(self.t) < 0).any():
            raise EventValidationError("events must be sorted by timestamp")
        if ((self.x < 0) | (self.x >= g.width) | (self.y < 0) | (self.y >= g.height)).any():
            raise EventValidationError("event coordinates outside sensor geometry")
        if not np.isin(self.polarity, (-1, 1)).all():
            raise EventValidationError("polarity must be +1 or -1")

    @property
    def n(self) -> int:
        return len(self.t)


@dataclass(frozen=True)
class EventBatch:
    """One window of events, batch-local t in [0, tau] (``events.py:93-120``)."""

    x: np.ndarray
    y: np.ndarray
    t: np.ndarray
    tau: float
    geometry: SensorGeometry
    t_start: float = 0.0

    def __post_init__(self):
        if self.tau <= 0:
            raise EventValidationError("batch duration tau must be positive")
        if len(self.t) and ((self.t < 0).any() or (self.t > self.tau).any()):
            raise EventValidationError("batch timestamps must lie in [0, tau]")

    @property
    def n(self) -> int:
        return len(self.t)

    @property
    def t_end(self) -> float:
        return self.t_start + self.tau


def window_bounds(t: np.ndarray, tau: float) -> tuple[int, np.ndarray]:
    """First window index k0 and an (n_windows, 2) array of [lo, hi) offsets.

    Window k covers [k*tau, k*tau + tau) on the absolute clock; both bounds are
    left-searchsorted as ``events.py:341-347`` does.
    """
    k0 = int(np.floor(t[0] / tau))
    k1 = int(np.floor(t[-1] / tau))
    starts = np.array([k * tau for k in range(k0, k1 + 1)], dtype=np.float64)
    lo = np.searchsorted(t, starts, side="left")
    hi = np.searchsorted(t, starts + tau, side="left")
    return k0, np.stack([lo, hi], axis=1)


def batch_stream(stream: EventStream, tau: float) -> list[EventBatch]:
    """Split a stream into windows [k*tau, (k+1)*tau) (``events.py:330-359``).

    Empty windows inside the stream span are kept as empty batches.
    """
    if tau <= 0:
        raise ValueError("tau must be positive")
    if stream.n == 0:
        return []
    k0, bounds = window_bounds(stream.t, tau)
    out = []
    for j, (lo, hi) in enumerate(bounds):
        start = (k0 + j) * tau
        out.append(EventBatch(
            stream.x[lo:hi].copy(), stream.y[lo:hi].copy(),
            np.minimum(stream.t[lo:hi] - start, tau), tau, stream.geometry,
            t_start=start))
    return out
