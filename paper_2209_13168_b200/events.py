"""Input contract of the bound-evaluation hot path: sensor grid, event window, stream.

Mirrors the reference's data types so a caller holding ``eventdiv`` objects can
pass them unchanged (every entry point in this package duck-types on the fields
``x, y, t, tau, geometry.width, geometry.height``):

* ``SensorGeometry``  -- ``pkg/src/eventdiv/events.py:29-44``
* ``EventStream``     -- ``pkg/src/eventdiv/events.py:47-90`` (validation rules kept)
* ``EventBatch``      -- ``pkg/src/eventdiv/events.py:93-120``
* ``batch_stream``    -- ``pkg/src/eventdiv/events.py:330-359`` (windowing)
* ``parse_event_bin`` -- ``pkg/src/eventdiv/events.py:186-206`` (EVD1 decoded on the
  device); ``write_event_bin`` (``:236-246``) for round trips

* ``pixel_counts`` / ``remove_hot_pixels`` / ``rescale_events`` -- ``events.py:273-313``
  on the device

CSV parsing and subsampling (numpy PCG64 stream parity) stay outside the hot
path and are not provided here.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

BIN_MAGIC = b"EVD1"
_BIN_RECORD = np.dtype([("t_us", "<u8"), ("x", "<f4"), ("y", "<f4"), ("p", "i1")])


class EventValidationError(ValueError):
    """Event data violates a stream/batch invariant (``events.py:25-26``)."""


class EventFormatError(ValueError):
    """Malformed event file (``events.py:21-22``)."""


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


def load_bin_resident(data: bytes, ctx=None):
    """Decode an EVD1 body on the device (evd_load_bin); the stream stays
    resident in the context.  Returns (ctx, geometry, n)."""
    import ctypes

    from . import _lib
    ctx = ctx or _lib.context()
    data = bytes(data)
    w, h, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    rc = ctx.lib.evd_load_bin(ctx.h, data, len(data), ctypes.byref(w), ctypes.byref(h),
                              ctypes.byref(n))
    if rc == _lib.EVD_ERR_FORMAT:
        raise EventFormatError(ctx.error_text())
    if rc == _lib.EVD_ERR_VALIDATION:
        raise EventValidationError(ctx.error_text())
    if rc:
        raise _lib.EvdError(rc, ctx.error_text())
    return ctx, SensorGeometry(w.value, h.value), n.value


def parse_event_bin(data: bytes, ctx=None) -> EventStream:
    """Parse the BIN event format (``events.py:186-206``): decoded, sorted and
    validated on the device, then copied back as an EventStream."""
    import ctypes

    from . import _lib
    ctx, geometry, n = load_bin_resident(data, ctx)
    x, y, t = (np.empty(n, dtype=np.float64) for _ in range(3))
    p = np.empty(n, dtype=np.int8)
    if n:
        rc = ctx.lib.evd_stream_copy(ctx.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t),
                                     p.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
        if rc:
            raise _lib.EvdError(rc, ctx.error_text())
    return EventStream(x, y, t, p, geometry)


def write_event_bin(stream: EventStream, path) -> None:
    """Write the BIN event format (``events.py:236-246``)."""
    g = stream.geometry
    body = np.empty(stream.n, dtype=_BIN_RECORD)
    body["t_us"] = np.round(stream.t * 1e6).astype(np.uint64)
    body["x"] = stream.x
    body["y"] = stream.y
    body["p"] = stream.polarity
    with open(Path(path), "wb") as fh:
        fh.write(struct.pack("<4sIIQ", BIN_MAGIC, g.width, g.height, stream.n))
        fh.write(body.tobytes())


def _stream_ctx(stream, ctx=None):
    """Upload ``stream`` as the context's resident stream (evd_load_stream)."""
    import ctypes

    from . import _lib
    ctx = ctx or _lib.context()
    x, y, t = _lib.f64(stream.x), _lib.f64(stream.y), _lib.f64(stream.t)
    p = np.ascontiguousarray(stream.polarity, dtype=np.int8)
    g = stream.geometry
    rc = ctx.lib.evd_load_stream(ctx.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t),
                                 p.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)), len(t),
                                 g.width, g.height)
    if rc:
        raise _lib.EvdError(rc, ctx.error_text())
    return ctx


def _resident_stream(ctx, n: int, geometry: SensorGeometry) -> EventStream:
    import ctypes

    from . import _lib
    x, y, t = (np.empty(n, dtype=np.float64) for _ in range(3))
    p = np.empty(n, dtype=np.int8)
    if n:
        rc = ctx.lib.evd_stream_copy(ctx.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t),
                                     p.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
        if rc:
            raise _lib.EvdError(rc, ctx.error_text())
    return EventStream(x, y, t, p, geometry)


def pixel_counts(stream: EventStream, ctx=None) -> np.ndarray:
    """Per-pixel event counts (height x width), floor-binned (``events.py:273-281``)."""
    from . import _lib
    ctx = _stream_ctx(stream, ctx)
    g = stream.geometry
    counts = np.empty((g.height, g.width), dtype=np.int64)
    rc = ctx.lib.evd_pixel_counts(ctx.h, _lib.ptr(counts, _lib._i64p))
    if rc:
        raise _lib.EvdError(rc, ctx.error_text())
    return counts


def remove_hot_pixels(stream: EventStream, k: float = 10.0, ctx=None) -> EventStream:
    """Drop all events on pixels whose count exceeds median + k*MAD of the
    nonzero counts (``events.py:284-300``), on the device."""
    import ctypes

    from . import _lib
    if k <= 0:
        raise ValueError("k must be positive")
    if stream.n == 0:
        return stream
    ctx = _stream_ctx(stream, ctx)
    n = ctypes.c_int64()
    thr = ctypes.c_double()
    rc = ctx.lib.evd_stream_remove_hot_pixels(ctx.h, float(k), ctypes.byref(n), ctypes.byref(thr))
    if rc:
        raise _lib.EvdError(rc, ctx.error_text())
    return _resident_stream(ctx, n.value, stream.geometry)


def rescale_events(stream: EventStream, target: SensorGeometry, ctx=None) -> EventStream:
    """Scale event coordinates onto a new sensor grid (``events.py:303-313``)."""
    from . import _lib
    ctx = _stream_ctx(stream, ctx)
    rc = ctx.lib.evd_stream_rescale(ctx.h, target.width, target.height)
    if rc:
        raise _lib.EvdError(rc, ctx.error_text())
    return _resident_stream(ctx, stream.n, target)
