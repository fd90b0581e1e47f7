"""ctypes binding of the C ABI (include/gsr.h) -> _build/libgsr.so.

There is no CPU fallback: if the library is missing or no CUDA device is
present, every render/metric call raises RenderError (loudly), it never
silently computes on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
# GSR_LIB_PATH: a tuning variant built with `build.py --out ... -D ...`
LIB_PATH = Path(os.environ.get("GSR_LIB_PATH") or PKG / "_build" / "libgsr.so")
HEADER = PKG.parent / "include" / "gsr.h"

GSR_OK = 0
GSR_E_INVALID = -1
GSR_E_CUDA = -2
GSR_E_OOM = -3
GSR_E_DIM_MISMATCH = -4
GSR_E_TOO_SMALL = -5
GSR_E_NO_DEVICE = -6
GSR_E_PLY_HEADER = -7
GSR_E_PLY_PROPERTY = -8
GSR_E_PLY_TRUNCATED = -9
GSR_E_NONFINITE = -10
GSR_PLY_NCOLS = 59


class RenderError(Exception):
    """render.py:52-53."""


class GsrCamera(ctypes.Structure):
    _fields_ = [("w2c", ctypes.c_double * 12), ("campos", ctypes.c_double * 3),
                ("fx", ctypes.c_double), ("fy", ctypes.c_double), ("cx", ctypes.c_double),
                ("cy", ctypes.c_double), ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class GsrStats(ctypes.Structure):
    _fields_ = [("splats_drawn", ctypes.c_int64), ("splats_culled", ctypes.c_int64),
                ("tile_keys", ctypes.c_int64), ("depth_passes", ctypes.c_int32),
                ("retries", ctypes.c_int32), ("ms_device", ctypes.c_float),
                ("ms_preprocess", ctypes.c_float), ("ms_depth_sort", ctypes.c_float),
                ("ms_binning", ctypes.c_float), ("ms_tile_sort", ctypes.c_float),
                ("ms_blend", ctypes.c_float), ("kernel_launches", ctypes.c_int32),
                ("overflow_frames", ctypes.c_int32), ("pairs", ctypes.c_int64),
                ("composited", ctypes.c_int64), ("row_evals_blend", ctypes.c_int64),
                ("row_evals_binning", ctypes.c_int64), ("long_run_frames", ctypes.c_int32),
                ("ms_slice_b", ctypes.c_float)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class GsrPlyInfo(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int64), ("body_offset", ctypes.c_int64),
                ("body_bytes", ctypes.c_int64), ("n_props", ctypes.c_int32),
                ("has_rest", ctypes.c_int32), ("col", ctypes.c_int32 * GSR_PLY_NCOLS),
                ("ms_slice_b", ctypes.c_float)]


class GsrPlyStats(ctypes.Structure):
    _fields_ = [("h2d_ms", ctypes.c_double), ("kernel_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("body_bytes", ctypes.c_int64),
                ("scene_bytes", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# (name, restype, argtypes); every symbol declared in include/gsr.h
_vp, _i32, _i64, _dbl, _sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
_P = ctypes.POINTER
SIGNATURES = [
    ("gsr_abi_version", _i32, []),
    ("gsr_tile_size", _i32, [_P(ctypes.c_int), _P(ctypes.c_int)]),
    ("gsr_last_error", ctypes.c_char_p, []),
    ("gsr_device_count", _i32, [_P(_i32)]),
    ("gsr_scene_create", _i32, [_P(_vp), _i32, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    ("gsr_scene_destroy", _i32, [_vp]),
    ("gsr_scene_count", _i64, [_vp]),
    ("gsr_scene_device_bytes", _i64, [_vp]),
    ("gsr_scene_sh_is_f32", _i32, [_vp]),
    ("gsr_ply_parse_header", _i32, [_vp, _i64, _P(GsrPlyInfo)]),
    ("gsr_scene_create_ply", _i32, [_P(_vp), _i32, _vp, _i64, _P(GsrPlyStats)]),
    ("gsr_scene_read", _i32, [_vp, _i32, _vp]),
    ("gsr_ctx_create", _i32, [_P(_vp), _i32]),
    ("gsr_ctx_destroy", _i32, [_vp]),
    ("gsr_ctx_device_bytes", _i64, [_vp]),
    ("gsr_ctx_frame_u8", _vp, [_vp]),
    ("gsr_ctx_stream", _vp, [_vp]),
    ("gsr_ctx_set_kernel_timing", _i32, [_vp, _i32]),
    ("gsr_ctx_set_slicing", _i32, [_vp, _i64, ctypes.c_float]),
    ("gsr_ctx_kernel_times", _i32, [_vp, _i32, _vp, _vp, _P(_i32)]),
    ("gsr_render", _i32, [_vp, _vp, _P(GsrCamera), _vp, _i32, _i32, _vp, _vp, _vp, _P(GsrStats)]),
    ("gsr_render_async", _i32, [_vp, _vp, _P(GsrCamera), _vp, _i32, _i32]),
    ("gsr_ctx_finish", _i32, [_vp, _vp, _P(GsrStats)]),
    ("gsr_render_enqueue", _i32, [_vp, _vp, _P(GsrCamera), _vp, _i32, _i32, _vp]),
    ("gsr_debug_preprocess", _i32, [_vp, _vp, _P(GsrCamera), _i32, _i32, _vp, _vp, _vp,
                                    _P(GsrStats)]),
    ("gsr_debug_tile_lists", _i32, [_vp, _vp, _vp, _vp, _P(GsrStats)]),
    ("gsr_debug_frame_counters", _i32, [_vp, _vp, _i32]),
    ("gsr_debug_blend_items", _i32, [_vp, _vp, _i64]),
    ("gsr_debug_contract_tiles", _i32, [_vp, _i32, _P(_i64), _vp, _vp, _vp,
                                        _P(ctypes.c_float)]),
    ("gsr_resample_bilinear_u8", _i32, [_vp, _vp, _i32, _i32, _vp, _i32, _i32]),
    ("gsr_ssim_u8", _i32, [_vp, _vp, _vp, _i32, _i32, _P(_dbl)]),
    ("gsr_ssim_luma_f64", _i32, [_vp, _vp, _vp, _i32, _i32, _P(_dbl)]),
    ("gsr_encode_jpeg", _i32, [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _sz, _P(_sz)]),
    ("gsr_sse_u8", _i32, [_vp, _vp, _vp, _i64, _P(ctypes.c_uint64)]),
    ("gsr_eval_frame", _i32, [_vp, _vp, _P(GsrCamera), _vp, _i32, _vp, _i32, _i32, _vp,
                              _P(_dbl), _P(ctypes.c_uint64)]),
    ("gsr_host_alloc", _i32, [_P(_vp), _sz]),
    ("gsr_host_free", _i32, [_vp]),
    ("gsr_ladder_ssim", _i32, [_vp, _vp, _P(GsrCamera), _vp, _i32, _i32, _P(GsrCamera),
                               _P(_dbl), _P(GsrStats)]),
]

_lib = None
_lock = threading.Lock()


def load():
    """Load libgsr.so (raises RenderError if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RenderError(f"CUDA library {LIB_PATH} is not built; run "
                                  "`python -m paper_2605_08699_b200.build` (no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().gsr_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map GSR_E_* to the reference's exception types."""
    if rc == GSR_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == GSR_E_INVALID:
        raise ValueError(msg)
    if rc == GSR_E_DIM_MISMATCH:
        from .metrics import DimensionMismatch
        raise DimensionMismatch(msg)
    if rc == GSR_E_TOO_SMALL:
        from .metrics import TooSmall
        raise TooSmall(msg)
    if GSR_E_NONFINITE <= rc <= GSR_E_PLY_HEADER:  # model.py:40-57, reference messages
        from . import model
        cls = {GSR_E_PLY_HEADER: model.MalformedHeader, GSR_E_PLY_PROPERTY: model.MissingProperty,
               GSR_E_PLY_TRUNCATED: model.TruncatedBody,
               GSR_E_NONFINITE: model.NonFiniteAttribute}[rc]
        raise cls(last_error())
    raise RenderError(msg or f"gsr error {rc}")


def device_count() -> int:
    n = ctypes.c_int(0)
    load().gsr_device_count(ctypes.byref(n))
    return int(n.value)


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class Context:
    """One gsr_ctx: a CUDA stream + workspace, owned by one thread."""

    def __init__(self, device: int = 0):
        self.lib = load()
        self.device = device
        h = ctypes.c_void_p()
        check(self.lib.gsr_ctx_create(ctypes.byref(h), int(device)), "gsr_ctx_create")
        self.handle = h
        self._pinned = {}

    def pinned(self, key: str, shape, dtype) -> np.ndarray:
        """A page-locked host array (reused per key) for fast readback.  The
        memory belongs to a PinnedBlock that every returned view references
        (through numpy's base chain), so it is freed only when the context
        has dropped it (close, or a larger request for the key) AND the last
        view is gone: arrays returned from here never dangle."""
        nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        blk = self._pinned.get(key)
        if blk is None or blk.nbytes < nbytes:
            blk = PinnedBlock(self.lib, max(nbytes, 1))
            self._pinned[key] = blk  # the old block lives on in its views, if any
        return np.asarray(blk)[:nbytes].view(dtype).reshape(shape)

    def close(self):
        if getattr(self, "handle", None) is not None:
            self._pinned = {}
            self.lib.gsr_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


class PinnedBlock:
    """cudaHostAlloc'd bytes (gsr_host_alloc) freed when the block object
    dies; numpy arrays made from it keep it alive via __array_interface__."""

    def __init__(self, lib, nbytes: int):
        self.lib = lib
        self.nbytes = int(nbytes)
        p = ctypes.c_void_p()
        check(lib.gsr_host_alloc(ctypes.byref(p), self.nbytes), "gsr_host_alloc")
        self.ptr = p

    @property
    def __array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr.value, False),
                "version": 3}

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            if self.ptr is not None and self.ptr.value:
                self.lib.gsr_host_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


_tls = threading.local()


def context(device: int = 0) -> Context:
    """The calling thread's context for `device` (server.py:99-100 threads)."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    c = ctxs.get(device)
    if c is None:
        c = ctxs[device] = Context(device)
    return c
