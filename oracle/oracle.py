"""CPU oracle for the bound-evaluation hot path (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
may import this module; the product package never does.  It restates the
reference algorithm:

* per-event work (warp, point image, supercover raster)  -> ``evd_oracle.c``
  (C restatement of ``contrast.py:48-58,73-203`` / ``geometry.py:70-87``)
* contrast and bound assembly                           -> numpy, literally the
  reference expressions (``contrast.py:61-64,241-251``): numpy IS the
  reference's arithmetic for these reductions (pairwise ``np.sum``)
* branch-and-bound / grid oracle / stream driver         -> ``solver.py:74-162``
  restated with ``heapq``

Pinned by ``tests/test_oracle.py`` against ``tests/golden/*`` which were
produced by importing the reference package itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import heapq
import itertools
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_d = ctypes.POINTER(ctypes.c_double)
_u32 = ctypes.POINTER(ctypes.c_uint32)
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return os.path.join(HERE, "liboracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.orc_warp.argtypes = [_d, _d, _d, _i64, ctypes.c_double, ctypes.c_double, _i32, _i32, _d, _d]
        L.orc_point_image_mt.argtypes = [_d, _d, _d, _i64, ctypes.c_double, ctypes.c_double,
                                         _i32, _i32, _u32, ctypes.c_int]
        L.orc_point_image_mt.restype = _i64
        L.orc_bound_image_mt.argtypes = [_d, _d, _d, _i64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, _i32, _i32, _u32, ctypes.c_int]
        L.orc_bound_image_mt.restype = _i64
        L.orc_bound_image_endpoints.argtypes = [_d, _d, _d, _d, _i64, _i32, _i32, _u32]
        L.orc_bound_image_endpoints.restype = _i64
        L.orc_rasterize_segment.argtypes = [ctypes.c_double] * 4 + [_i32, _i32, _u32]
        _LIB = L
    return _LIB


def _p(a, ptr=_d):
    return a.ctypes.data_as(ptr)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


THREADS = 1  # bench.py's CPU-baseline leg raises this to the host core count


# ---------------------------------------------------------------- geometry.py
def warp(x, y, t, nu, tau, width, height):
    """geometry.py:70-87 (radial_warp) for arrays."""
    x, y, t = _f64(x), _f64(y), _f64(t)
    xo, yo = np.empty_like(x), np.empty_like(y)
    lib().orc_warp(_p(x), _p(y), _p(t), x.size, nu, tau, width, height, _p(xo), _p(yo))
    return xo, yo


# ---------------------------------------------------------------- contrast.py
def point_image(batch, nu):
    """accumulate_image (contrast.py:48-58) -> (uint32 (H, W) counts, in_image)."""
    g = batch.geometry
    x, y, t = _f64(batch.x), _f64(batch.y), _f64(batch.t)
    counts = np.zeros((g.height, g.width), dtype=np.uint32)
    inside = lib().orc_point_image_mt(_p(x), _p(y), _p(t), x.size, nu, batch.tau,
                                      g.width, g.height, _p(counts, _u32), THREADS)
    return counts, int(inside)


def image_contrast(counts, in_image):
    """image_contrast (contrast.py:61-64), the reference numpy expression."""
    c = np.asarray(counts, dtype=np.float64)
    mu = in_image / c.size
    return float(np.sum((c - mu) ** 2) / c.size)


def contrast_at(batch, nu):
    """solver.py:74-76"""
    return image_contrast(*point_image(batch, nu))


def bound_image(batch, lo, hi):
    """_bound_image_kernel over warps at lo/hi -> (uint32 counts, fully_inside)."""
    g = batch.geometry
    x, y, t = _f64(batch.x), _f64(batch.y), _f64(batch.t)
    counts = np.zeros((g.height, g.width), dtype=np.uint32)
    fi = lib().orc_bound_image_mt(_p(x), _p(y), _p(t), x.size, lo, hi, batch.tau,
                                  g.width, g.height, _p(counts, _u32), THREADS)
    return counts, int(fi)


def bound_terms(batch, lo, hi):
    """bound_terms (contrast.py:241-251) -> (s_bar, mu_lower, c_bar, fully_inside, counts)."""
    counts, fi = bound_image(batch, lo, hi)
    m = counts.size
    s_bar = float(np.sum(counts.astype(np.float64) ** 2))
    mu_lower = fi / m
    return s_bar, mu_lower, s_bar / m - mu_lower ** 2, fi, counts


def rasterize_segment(p0, p1, width, height):
    """rasterize_segment (contrast.py:206-222) -> set of (ix, iy)."""
    counts = np.zeros((height, width), dtype=np.uint32)
    lib().orc_rasterize_segment(float(p0[0]), float(p0[1]), float(p1[0]), float(p1[1]),
                                width, height, _p(counts, _u32))
    ys, xs = np.nonzero(counts)
    return {(int(a), int(b)) for a, b in zip(xs, ys)}


def pairwise_sum(a) -> float:
    """numpy's float64 pairwise summation (numpy/_core/src/umath/loops_utils.h.src),
    restated for a contiguous 1-D array and started from 0.0 as ``np.sum`` does.
    Used to pin the device's fixed reduction tree."""
    a = np.asarray(a, dtype=np.float64).ravel()

    def pw(lo, n):
        if n < 8:
            r = 0.0
            for i in range(n):
                r += float(a[lo + i])
            return r
        if n <= 128:
            r = [float(v) for v in a[lo:lo + 8]]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += float(a[lo + i + j])
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += float(a[lo + i])
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return pw(lo, n2) + pw(lo + n2, n - n2)

    return 0.0 + pw(0, a.size)


# ---------------------------------------------------------------- solver.py
@dataclass(frozen=True)
class Result:
    nu: float
    contrast: float
    bound_gap: float
    iterations: int
    runtime: float
    bound_evals: int = 0
    status: str = "ok"


def velocity_domain(tau, epsilon=1e-6):
    """geometry.py:61-67"""
    return -(1.0 - epsilon) / tau, 0.0


def maximise_contrast_bnb(batch, gamma=0.025, epsilon=1e-6, max_iterations=1_000_000,
                          min_interval_width=1e-9):
    """Best-first BnB, solver.py:79-123 (heap key (-c_bar, FIFO counter))."""
    if batch.n == 0:
        raise ValueError("no events in batch")
    start = time.perf_counter()
    lo0, hi0 = velocity_domain(batch.tau, epsilon)
    nu_hat = 0.5 * (lo0 + hi0)
    c_hat = contrast_at(batch, nu_hat)
    counter = itertools.count()
    heap = [(-bound_terms(batch, lo0, hi0)[2], next(counter), lo0, hi0)]
    evals = 1
    iterations = 0
    bound_gap = 0.0
    while heap:
        neg, _, lo, hi = heapq.heappop(heap)
        iterations += 1
        gap = -neg - c_hat
        if gap <= gamma or (hi - lo) < min_interval_width:
            bound_gap = max(gap, 0.0)
            break
        c = 0.5 * (lo + hi)
        c_c = contrast_at(batch, c)
        if c_c >= c_hat:
            nu_hat, c_hat = c, c_c
        for clo, chi in ((lo, c), (c, hi)):
            cb = bound_terms(batch, clo, chi)[2]
            evals += 1
            if cb >= c_hat:
                heapq.heappush(heap, (-cb, next(counter), clo, chi))
        if iterations >= max_iterations:
            return Result(nu_hat, c_hat, bound_gap, iterations,
                          time.perf_counter() - start, evals, "iteration_limit")
    return Result(nu_hat, c_hat, bound_gap, iterations, time.perf_counter() - start, evals)


def grid_search(batch, n_points, epsilon=1e-6):
    """grid_search_oracle, solver.py:126-136"""
    lo, hi = velocity_domain(batch.tau, epsilon)
    nus = np.linspace(lo, hi, n_points)
    cs = np.array([contrast_at(batch, float(nu)) for nu in nus])
    best = int(np.argmax(cs))
    return float(nus[best]), float(cs[best])


# ------------------------------------------------------------------ EVD1 files
class FormatError(ValueError):
    pass


class ValidationError(ValueError):
    pass


def parse_bin(data: bytes):
    """parse_event_bin (events.py:186-206) + _from_columns (:128-134) + the
    EventStream invariants (:61-81), restated with numpy/struct.  Returns
    (x, y, t, p, (width, height)); raises FormatError / ValidationError with
    the reference's messages."""
    import struct
    if len(data) < 20:
        raise FormatError("truncated BIN header")
    magic, width, height, count = struct.unpack_from("<4sIIQ", data, 0)
    if magic != b"EVD1":
        raise FormatError(f"bad magic {magic!r}")
    rec = np.dtype([("t_us", "<u8"), ("x", "<f4"), ("y", "<f4"), ("p", "i1")])
    if len(data) < 20 + count * rec.itemsize:
        raise FormatError(f"truncated BIN body: expected {count} records")
    r = np.frombuffer(data, dtype=rec, count=count, offset=20)
    if width < 1 or height < 1:
        raise ValidationError(f"sensor dimensions must be positive, got {width}x{height}")
    t = np.asarray(r["t_us"], dtype=np.float64) * 1e-6
    order = np.argsort(t, kind="stable")
    x = np.asarray(r["x"], np.float64)[order]
    y = np.asarray(r["y"], np.float64)[order]
    t = t[order]
    p = np.asarray(r["p"], np.int8)[order]
    if len(t):
        if not (np.isfinite(x).all() and np.isfinite(y).all()):
            raise ValidationError("event coordinates must be finite")
        if ((x < 0) | (x >= width) | (y < 0) | (y >= height)).any():
            raise ValidationError("event coordinates outside sensor geometry")
        if not np.isin(p, (-1, 1)).all():
            raise ValidationError("polarity must be +1 or -1")
    return x, y, t, p, (int(width), int(height))


# ------------------------------------------------------------------ preprocessing
def pixel_counts(x, y, width, height):
    """events.py:273-281 restated."""
    counts = np.zeros((height, width), dtype=np.int64)
    if len(x):
        np.add.at(counts, (np.floor(y).astype(np.intp), np.floor(x).astype(np.intp)), 1)
    return counts


def remove_hot_pixels(x, y, t, p, width, height, k=10.0):
    """events.py:284-300 restated: returns (x, y, t, p, threshold)."""
    if k <= 0:
        raise ValueError("k must be positive")
    if len(x) == 0:
        return x, y, t, p, 0.0
    counts = pixel_counts(x, y, width, height)
    nz = counts[counts > 0].astype(np.float64)
    med = np.median(nz)
    mad = np.median(np.abs(nz - med))
    threshold = med + k * mad
    keep = ~(counts > threshold)[np.floor(y).astype(np.intp), np.floor(x).astype(np.intp)]
    return x[keep], y[keep], t[keep], p[keep], float(threshold)


def rescale(x, y, width, height, width2, height2):
    """events.py:303-313 restated: returns (x, y)."""
    sx, sy = width2 / width, height2 / height
    return (np.minimum(x * sx, np.nextafter(float(width2), 0.0)),
            np.minimum(y * sy, np.nextafter(float(height2), 0.0)))
