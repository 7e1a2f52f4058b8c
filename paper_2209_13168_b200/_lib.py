"""ctypes binding of libevd.so (the C ABI in include/evd.h).

There is no fallback: if the shared library is missing or no CUDA device is
usable, every entry point raises ``EvdUnavailable``.  One device context is
kept per (host thread, device).
"""

from __future__ import annotations

import ctypes
import os
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EVD_LIB") or os.path.join(HERE, "libevd.so")

EVD_OK, EVD_ERR_CUDA, EVD_ERR_ARG, EVD_ERR_NO_EVENTS = 0, 1, 2, 3
EVD_ERR_CHEIRALITY, EVD_ERR_ITER_LIMIT, EVD_ERR_STATE = 4, 5, 6
EVD_ERR_FORMAT, EVD_ERR_VALIDATION = 7, 8
FRONTIER_AUTO, FRONTIER_TILES, FRONTIER_GLOBAL, FRONTIER_GLOBAL_EXACT = 0, 1, 2, 3
FRONTIER_PER_INTERVAL = 4

# every symbol include/evd.h declares (checked by tests/test_abi.py)
SYMBOLS = (
    "evd_create", "evd_destroy", "evd_last_error", "evd_set_stream", "evd_kernel_launches",
    "evd_window_generation",
    "evd_device_sms", "evd_set_events", "evd_set_events_list", "evd_radial_warp",
    "evd_warp_scale",
    "evd_point_images", "evd_bound_images", "evd_eval_frontier", "evd_set_option",
    "evd_frontier_info", "evd_image_contrast",
    "evd_rasterize_segments",
    "evd_eval_nodes", "evd_solve", "evd_solve_events", "evd_solve_windows", "evd_solve_windows_list", "evd_solve_trace", "evd_solve_block_trace",
    "evd_probe_events", "evd_solve_stream", "evd_solve_loaded_stream", "evd_load_bin",
    "evd_stream_copy", "evd_load_stream", "evd_pixel_counts", "evd_stream_remove_hot_pixels",
    "evd_stream_rescale",
    "evd_pow2_table",
)


class EvdUnavailable(RuntimeError):
    """libevd.so could not be loaded or no CUDA device is usable."""


class EvdError(RuntimeError):
    """A CUDA-side failure reported by libevd."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class SolveParams(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("epsilon", ctypes.c_double),
                ("min_interval_width", ctypes.c_double), ("max_iterations", ctypes.c_int64)]


class SolveResult(ctypes.Structure):
    _fields_ = [("nu", ctypes.c_double), ("contrast", ctypes.c_double),
                ("bound_gap", ctypes.c_double), ("iterations", ctypes.c_int64),
                ("bound_evals", ctypes.c_int64), ("point_evals", ctypes.c_int64),
                ("max_frontier", ctypes.c_int64), ("device_ms", ctypes.c_double),
                ("marks", ctypes.c_uint64), ("exact_events", ctypes.c_uint64),
                ("rounds", ctypes.c_int64)]


class WindowResult(ctypes.Structure):
    _fields_ = [("nu", ctypes.c_double), ("contrast", ctypes.c_double),
                ("bound_gap", ctypes.c_double), ("iterations", ctypes.c_int64),
                ("bound_evals", ctypes.c_int64), ("point_evals", ctypes.c_int64),
                ("max_frontier", ctypes.c_int64), ("marks", ctypes.c_uint64),
                ("exact_events", ctypes.c_uint64),
                ("status", ctypes.c_int32), ("groups", ctypes.c_int32),
                ("rounds", ctypes.c_int64)]


_d = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double

_SIGS = {
    "evd_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "evd_destroy": (None, [_vp]),
    "evd_last_error": (ctypes.c_char_p, [_vp]),
    "evd_set_stream": (ctypes.c_int, [_vp, _vp]),
    "evd_kernel_launches": (_i64, [_vp]),
    "evd_window_generation": (_i64, [_vp]),
    "evd_device_sms": (ctypes.c_int, [_vp]),
    "evd_set_events": (ctypes.c_int, [_vp, _d, _d, _d, _i64, _i32, _i32, _f64]),
    "evd_set_events_list": (ctypes.c_int, [_vp, ctypes.POINTER(_d), ctypes.POINTER(_d),
                                           ctypes.POINTER(_d), _i64p, _i32, _i32, _i32, _f64]),
    "evd_radial_warp": (ctypes.c_int, [_vp, _d, _d, _d, _i64, _f64, _f64, _i32, _i32, _d, _d]),
    "evd_warp_scale": (ctypes.c_int, [_vp, _d, _i64, _f64, _f64, _d]),
    "evd_point_images": (ctypes.c_int, [_vp, _d, _i32, _i64p, _d, _u32p]),
    "evd_bound_images": (ctypes.c_int, [_vp, _d, _d, _i32, _u64p, _i64p, _u64p, _u32p]),
    "evd_eval_frontier": (ctypes.c_int, [_vp, _d, _d, _i32, _u64p, _i64p, _u64p]),
    "evd_set_option": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64]),
    "evd_frontier_info": (ctypes.c_int, [_vp, _i64p]),
    "evd_image_contrast": (ctypes.c_int, [_vp, _d, _i64, _i64, _d]),
    "evd_rasterize_segments": (ctypes.c_int, [_vp, _d, _i32, _i32, _i32, _i32, _u32p]),
    "evd_eval_nodes": (ctypes.c_int, [_vp, _d, _d, _i64, _d, _d, _d]),
    "evd_solve": (ctypes.c_int, [_vp, ctypes.POINTER(SolveParams), ctypes.POINTER(SolveResult)]),
    "evd_solve_events": (ctypes.c_int, [_vp, _d, _d, _d, _i64, _i32, _i32, _f64,
                                        ctypes.POINTER(SolveParams), ctypes.POINTER(SolveResult)]),
    "evd_solve_windows": (ctypes.c_int, [_vp, _i64p, _i32, _i32, ctypes.POINTER(SolveParams),
                                         ctypes.POINTER(WindowResult), _d]),
    "evd_solve_windows_list": (ctypes.c_int, [_vp, ctypes.POINTER(_d), ctypes.POINTER(_d),
                                              ctypes.POINTER(_d), _i64p, _i32, _i32, _i32, _f64,
                                              _i32, ctypes.POINTER(SolveParams),
                                              ctypes.POINTER(WindowResult), _d]),
    "evd_solve_trace": (ctypes.c_int, [_vp, _i64p, _i64, _i64p]),
    "evd_solve_block_trace": (ctypes.c_int, [_vp, _i64p, _i64, ctypes.POINTER(_i32)]),
    "evd_probe_events": (ctypes.c_int, [_vp, _f64, _f64, _i32, _d]),
    "evd_solve_stream": (ctypes.c_int, [_vp, _d, _d, _d, _i64, _i32, _i32, _f64, _i32,
                                        ctypes.POINTER(SolveParams), ctypes.POINTER(WindowResult),
                                        _i32, ctypes.POINTER(_i32), _i64p, _d]),
    "evd_solve_loaded_stream": (ctypes.c_int, [_vp, _f64, _i32, ctypes.POINTER(SolveParams),
                                               ctypes.POINTER(WindowResult), _i32,
                                               ctypes.POINTER(_i32), _i64p, _d]),
    "evd_load_bin": (ctypes.c_int, [_vp, ctypes.c_char_p, _i64, ctypes.POINTER(_i32),
                                    ctypes.POINTER(_i32), _i64p]),
    "evd_stream_copy": (ctypes.c_int, [_vp, _d, _d, _d, ctypes.POINTER(ctypes.c_int8)]),
    "evd_load_stream": (ctypes.c_int, [_vp, _d, _d, _d, ctypes.POINTER(ctypes.c_int8), _i64, _i32,
                                       _i32]),
    "evd_pixel_counts": (ctypes.c_int, [_vp, _i64p]),
    "evd_stream_remove_hot_pixels": (ctypes.c_int, [_vp, _f64, _i64p, _d]),
    "evd_stream_rescale": (ctypes.c_int, [_vp, _i32, _i32]),
    "evd_pow2_table": (ctypes.c_int, [_i64, _i64, _d]),
}

_lib = None
_lib_lock = threading.Lock()
_tls = threading.local()
_default_device = int(os.environ.get("EVD_DEVICE", "0"))
_explicit_device: int | None = None


def load():
    """Load libevd.so and declare its signatures (no device is touched)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise EvdUnavailable(
                    f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (make -C paper_2209_13168_b200/csrc)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                if os.environ.get("EVD_LIB") and not hasattr(lib, name):
                    continue  # an older build under A/B (tools/ab_libs.sh)
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def set_device(device: int) -> None:
    """Device used by contexts created afterwards in this process."""
    global _explicit_device
    _explicit_device = int(device)


class Context:
    """One libevd context (device buffers, stream) for the calling thread."""

    _resident = None  # contrast.load_window's record of the resident window

    def __init__(self, device: int):
        self.lib = load()
        h = _vp()
        rc = self.lib.evd_create(device, ctypes.byref(h))
        if rc != EVD_OK:
            msg = self.lib.evd_last_error(None).decode()
            raise EvdUnavailable(f"evd_create(device={device}) failed: {msg}")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.evd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def window_generation(self) -> int:
        return int(self.lib.evd_window_generation(self.h))

    def error_text(self) -> str:
        return self.lib.evd_last_error(self.h).decode()

    @property
    def launches(self) -> int:
        return int(self.lib.evd_kernel_launches(self.h))

    @property
    def sms(self) -> int:
        return int(self.lib.evd_device_sms(self.h))

    def set_option(self, name: str, value: int) -> None:
        rc = self.lib.evd_set_option(self.h, name.encode(), int(value))
        if rc:
            raise EvdError(rc, self.error_text())

    def frontier_info(self) -> dict:
        out = np.zeros(5, dtype=np.int64)
        rc = self.lib.evd_frontier_info(self.h, out.ctypes.data_as(_i64p))
        if rc:
            raise EvdError(rc, self.error_text())
        return {"tiles": int(out[0]), "tile_pixels": int(out[1]), "listed_events": int(out[2]),
                "tiles_with_work": int(out[3]), "last_path": int(out[4])}


def _current_device() -> int:
    """set_device's choice; else torch's current device once torch has
    initialised CUDA in this process (one rank per GPU under torch.distributed
    calls torch.cuda.set_device(local_rank)); else EVD_DEVICE / 0."""
    if _explicit_device is not None:
        return _explicit_device
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_initialized():
                return int(torch.cuda.current_device())
        except Exception:
            pass
    return _default_device


def context(device: int | None = None) -> Context:
    """The calling thread's context for `device` (default: set_device, else
    torch's current CUDA device, else EVD_DEVICE / 0)."""
    dev = _current_device() if device is None else int(device)
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    ctx = cache.get(dev)
    if ctx is None:
        ctx = cache[dev] = Context(dev)
    return ctx


def ptr(a: np.ndarray, kind=_d):
    return a.ctypes.data_as(kind)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)
