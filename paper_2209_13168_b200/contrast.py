"""Motion-compensated event images, the contrast objective and its interval bound.

Drop-in for ``pkg/src/eventdiv/contrast.py``.  Every image is built on the
B200 (libevd.so, include/evd.h); the host only assembles the scalar bound
``c_bar = s_bar/M - mu_lower**2`` exactly as ``contrast.py:248-251`` does, from
the exact integers the device returns.

Beyond the reference API this module adds batched forms used by the batched
frontier and the grid oracle: ``point_terms`` (k velocities) and
``bound_terms_many`` (k intervals) over one resident window.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .events import EventBatch, SensorGeometry
from .geometry import CheiralityError, VelocityInterval


@dataclass(frozen=True)
class EventImage:
    """Per-pixel counts (height x width) and in-image event count (contrast.py:23-36)."""

    counts: np.ndarray
    in_image_events: int

    @property
    def n_pixels(self) -> int:
        return self.counts.size

    @property
    def mean(self) -> float:
        return self.in_image_events / self.counts.size


@dataclass(frozen=True)
class ContrastBound:
    """c_bar = s_bar/M - mu_lower^2 (contrast.py:39-45)."""

    s_bar: float
    mu_lower: float
    c_bar: float


def _raise(ctx, rc):
    if rc == _lib.EVD_ERR_CHEIRALITY:
        raise CheiralityError(ctx.error_text())
    if rc == _lib.EVD_ERR_ARG:
        raise ValueError(ctx.error_text())
    raise _lib.EvdError(rc, ctx.error_text())


WINDOW_CACHE = True  # keep one window resident across per-call entry points


def _same_window(ctx, key, arrays) -> bool:
    """The window resident in ctx is exactly these arrays' current contents:
    same arrays, frame and tau, the context's window untouched since
    (evd_window_generation), and -- unless all three arrays are read-only --
    bit-identical contents to the host copy taken at upload (exact compare of
    the uint64 views, ~0.6 ms at 200 k events, against a ~1.5 ms re-upload)."""
    res = getattr(ctx, "_resident", None)
    if not WINDOW_CACHE or res is None or res[0] != key or res[1] != ctx.window_generation:
        return False
    if all(not a.flags.writeable for a in arrays):
        return all(a is c for a, c in zip(arrays, res[2]))
    return all(np.array_equal(a.view(np.uint64), c.view(np.uint64))
               for a, c in zip(arrays, res[2]))


def load_window(batch: EventBatch, ctx=None, cache: bool = True):
    """Make the window resident on the device (evd_set_events); returns the
    context.  The per-call entry points (accumulate_image, contrast_at,
    upper_bound_image, bound_terms, ...) call it every time, as the reference
    recomputes from the batch every time; a window already resident with
    identical contents is not uploaded again (_same_window).  ``cache=False``
    (one-shot callers such as a whole solve) uploads without keeping the host
    copy the content check needs."""
    ctx = ctx or _lib.context()
    g = batch.geometry
    x, y, t = _lib.f64(batch.x), _lib.f64(batch.y), _lib.f64(batch.t)
    key = (x.ctypes.data, y.ctypes.data, t.ctypes.data, t.size, g.width, g.height,
           float(batch.tau))
    cache = cache and WINDOW_CACHE
    if cache and _same_window(ctx, key, (x, y, t)):
        return ctx
    ctx._resident = None
    rc = ctx.lib.evd_set_events(ctx.h, _lib.ptr(x), _lib.ptr(y), _lib.ptr(t), t.size,
                                g.width, g.height, float(batch.tau))
    if rc:
        _raise(ctx, rc)
    # read-only arrays: held (so their buffers cannot be freed and reused at
    # the same address); writeable ones: a copy to compare against
    if cache:
        frozen = all(not a.flags.writeable for a in (x, y, t))
        ctx._resident = (key, ctx.window_generation,
                         (x, y, t) if frozen else (x.copy(), y.copy(), t.copy()))
    return ctx


def load_window_device(x, y, t, tau: float, geometry, ctx=None):
    """evd_set_events from device arrays on the context's GPU (torch CUDA
    tensors of float64, contiguous), e.g. a window broadcast over NCCL.

    The context is the tensors' own device's.  libevd copies on its own
    stream, so the producer's stream (torch's current stream: the NCCL
    broadcast that filled the tensors is ordered before it) is synchronised
    first -- otherwise the copy could read the buffer before it is filled."""
    import ctypes

    import torch
    dev = t.device.index if t.is_cuda else None
    if ctx is None:
        ctx = _lib.context(dev)
    elif dev is not None and ctx.device != dev:
        raise ValueError(f"events on cuda:{dev} but the libevd context is on cuda:{ctx.device}")
    if t.is_cuda:
        torch.cuda.current_stream(t.device).synchronize()
    n = int(t.numel())
    ptr = lambda v: ctypes.cast(ctypes.c_void_p(v.data_ptr()), _lib._d)
    rc = ctx.lib.evd_set_events(ctx.h, ptr(x), ptr(y), ptr(t), n, geometry.width,
                                geometry.height, float(tau))
    if rc:
        _raise(ctx, rc)
    return ctx


def point_terms(batch: EventBatch, nus, images: bool = False, ctx=None, loaded=False,
                with_contrast: bool = True):
    """accumulate_image + image_contrast at every nu in ``nus`` on the device.

    Returns (in_image int64[k], contrast float64[k], counts uint32[k, H, W] | None).
    """
    g = batch.geometry
    nu = _lib.f64(np.atleast_1d(nus))
    ctx = ctx if loaded else load_window(batch, ctx)
    k = nu.size
    inside = np.empty(k, dtype=np.int64)
    con = np.empty(k, dtype=np.float64)
    counts = np.empty((k, g.height, g.width), dtype=np.uint32) if images else None
    rc = ctx.lib.evd_point_images(ctx.h, _lib.ptr(nu), k, _lib.ptr(inside, _lib._i64p),
                                  _lib.ptr(con) if with_contrast else None,
                                  _lib.ptr(counts, _lib._u32p) if images else None)
    if rc:
        _raise(ctx, rc)
    return inside, con, counts


def bound_terms_many(batch: EventBatch, lo, hi, images: bool = False, ctx=None, loaded=False):
    """Exact bound integers for k intervals [lo_j, hi_j] on the device.

    Returns (s_bar uint64[k], fully_inside int64[k], marks uint64[k],
    counts uint32[k, H, W] | None).
    """
    g = batch.geometry
    lo, hi = _lib.f64(np.atleast_1d(lo)), _lib.f64(np.atleast_1d(hi))
    ctx = ctx if loaded else load_window(batch, ctx)
    k = lo.size
    s_bar = np.empty(k, dtype=np.uint64)
    fi = np.empty(k, dtype=np.int64)
    marks = np.empty(k, dtype=np.uint64)
    counts = np.empty((k, g.height, g.width), dtype=np.uint32) if images else None
    rc = ctx.lib.evd_bound_images(ctx.h, _lib.ptr(lo), _lib.ptr(hi), k,
                                  _lib.ptr(s_bar, _lib._u64p), _lib.ptr(fi, _lib._i64p),
                                  _lib.ptr(marks, _lib._u64p),
                                  _lib.ptr(counts, _lib._u32p) if images else None)
    if rc:
        _raise(ctx, rc)
    return s_bar, fi, marks, counts


def assemble_bound(s_bar_int: int, fully_inside: int, m: int) -> ContrastBound:
    """contrast.py:248-251 on the exact device integers (host CPython floats)."""
    s_bar = float(s_bar_int)
    mu_lower = fully_inside / m
    return ContrastBound(s_bar, mu_lower, s_bar / m - mu_lower**2)


def accumulate_image(batch: EventBatch, nu: float) -> EventImage:
    """Warp every event to the batch end and bin by floor (contrast.py:48-58)."""
    inside, _, counts = point_terms(batch, [float(nu)], images=True, with_contrast=False)
    return EventImage(counts[0].astype(np.float64), int(inside[0]))


def _device_contrast(counts: np.ndarray, in_image: int) -> float:
    c = _lib.f64(counts.ravel())
    out = np.empty(1, dtype=np.float64)
    ctx = _lib.context()
    rc = ctx.lib.evd_image_contrast(ctx.h, _lib.ptr(c), c.size, int(in_image), _lib.ptr(out))
    if rc:
        _raise(ctx, rc)
    return float(out[0])


def image_contrast(image: EventImage) -> float:
    """Variance of the counts about the in-image mean (contrast.py:61-64), with
    numpy's pairwise summation order reproduced on the device."""
    return _device_contrast(np.asarray(image.counts), image.in_image_events)


def image_contrast_expanded(image: EventImage) -> float:
    """(1/M) * sum(H^2) - mean^2 (contrast.py:67-70)."""
    mu = image.mean
    return float(_device_contrast(np.asarray(image.counts), 0) - mu * mu)


def rasterize_segment(p0: tuple[float, float], p1: tuple[float, float],
                      geometry: SensorGeometry) -> set[tuple[int, int]]:
    """Pixels whose closed squares meet the closed segment p0->p1 (contrast.py:206-222)."""
    return rasterize_segments([(p0[0], p0[1], p1[0], p1[1])], geometry)[0]


def rasterize_segments(segments, geometry: SensorGeometry, chunk: int = 0
                       ) -> list[set[tuple[int, int]]]:
    """Batched rasterize_segment: one device launch for all segments.

    ``chunk`` sets how many crossings one sampling chunk holds (0: default);
    the pixels do not depend on it."""
    segs = _lib.f64(np.asarray(segments, dtype=np.float64).reshape(-1, 4))
    k = segs.shape[0]
    if k == 0:
        return []
    counts = np.empty((k, geometry.height, geometry.width), dtype=np.uint32)
    ctx = _lib.context()
    rc = ctx.lib.evd_rasterize_segments(ctx.h, _lib.ptr(segs), k, geometry.width,
                                        geometry.height, int(chunk),
                                        _lib.ptr(counts, _lib._u32p))
    if rc:
        _raise(ctx, rc)
    if counts.max(initial=0) > 1:
        raise _lib.EvdError(_lib.EVD_ERR_CUDA, "supercover marked a pixel twice for one segment")
    out = []
    for j in range(k):
        ys, xs = np.nonzero(counts[j])
        out.append({(int(a), int(b)) for a, b in zip(xs, ys)})
    return out


def upper_bound_image(batch: EventBatch, interval: VelocityInterval) -> EventImage:
    """Per-pixel count of events whose endpoint segment touches the pixel (contrast.py:231-238)."""
    _, _, marks, counts = bound_terms_many(batch, [interval.lo], [interval.hi], images=True)
    return EventImage(counts[0].astype(np.float64), int(marks[0]))


def bound_terms(batch: EventBatch, interval: VelocityInterval) -> ContrastBound:
    """Contrast upper bound over the interval (contrast.py:241-251)."""
    s_bar, fi, _, _ = bound_terms_many(batch, [interval.lo], [interval.hi])
    return assemble_bound(int(s_bar[0]), int(fi[0]), batch.geometry.n_pixels)


def node_terms(batch: EventBatch, lo, hi, ctx=None, loaded=False):
    """The per-node work of maximise_contrast_bnb (solver.py:109-117) for the
    nodes [lo[i], hi[i]]: contrast_at(center) and both children's c_bar
    (evd_eval_nodes: the solve kernel's rounds, several nodes per event pass).

    Returns (contrast float64[k], cbar_lo float64[k], cbar_hi float64[k]).
    """
    lo = _lib.f64(np.atleast_1d(lo))
    hi = _lib.f64(np.atleast_1d(hi))
    if lo.shape != hi.shape:
        raise ValueError("lo and hi differ in length")
    ctx = ctx if loaded else load_window(batch, ctx)
    k = lo.size
    con, ca, cb = (np.empty(k, dtype=np.float64) for _ in range(3))
    rc = ctx.lib.evd_eval_nodes(ctx.h, _lib.ptr(lo), _lib.ptr(hi), k, _lib.ptr(con),
                                _lib.ptr(ca), _lib.ptr(cb))
    if rc:
        _raise(ctx, rc)
    return con, ca, cb


def frontier_terms(batch: EventBatch, lo, hi, ctx=None, loaded=False):
    """Batched frontier: exact bound integers for k intervals in one pass.

    Same values as ``bound_terms_many`` (s_bar uint64[k], fully_inside int64[k],
    marks uint64[k]); the whole frontier is evaluated by one evd_eval_frontier
    call (SURVEY §8(a) part 4).
    """
    lo, hi = _lib.f64(np.atleast_1d(lo)), _lib.f64(np.atleast_1d(hi))
    ctx = ctx if loaded else load_window(batch, ctx)
    k = lo.size
    s_bar = np.empty(k, dtype=np.uint64)
    fi = np.empty(k, dtype=np.int64)
    marks = np.empty(k, dtype=np.uint64)
    rc = ctx.lib.evd_eval_frontier(ctx.h, _lib.ptr(lo), _lib.ptr(hi), k,
                                   _lib.ptr(s_bar, _lib._u64p), _lib.ptr(fi, _lib._i64p),
                                   _lib.ptr(marks, _lib._u64p))
    if rc:
        _raise(ctx, rc)
    return s_bar, fi, marks
