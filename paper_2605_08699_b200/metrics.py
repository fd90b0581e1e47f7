"""Quality hooks on the GPU: ``ssim`` and ``upscale_to`` (mirror of
splatstream/metrics.py:57-130), plus the fused ladder evaluation.

``upscale_to`` is Pillow's BILINEAR resize restated in the sm_100a resample
kernels (bit-exact, integer fixed point); ``ssim`` is metrics.ssim restated
in f64 on the device (|delta| ~1e-16 against scipy).  ``psnr`` stays the
reference's numpy expression (not on the north-star path).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .render import _bg, device_scene, make_camera

PSNR_CAP_DB = 100.0
SSIM_WINDOW = 11
LUMA_WEIGHTS = np.array([0.299, 0.587, 0.114])


class MetricError(Exception):
    pass


class DimensionMismatch(MetricError):
    pass


class TooSmall(MetricError):
    pass


class EmptyInput(MetricError):
    pass


class IndexOutOfRange(MetricError):
    pass


def psnr(a, b) -> float:
    """metrics.py:57-66."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise DimensionMismatch(f"shapes differ: {a.shape} vs {b.shape}")
    mse = np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2)
    if mse == 0:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, 10.0 * math.log10(255.0 ** 2 / mse))


def _luma(img: np.ndarray) -> np.ndarray:
    img = np.asarray(img, dtype=np.float64)
    if img.ndim == 3:
        return np.ascontiguousarray(img @ LUMA_WEIGHTS)
    return np.ascontiguousarray(img)


def ssim(a, b, *, device: int | None = None) -> float:
    """metrics.py:76-114 on the GPU (RGB u8 fast path; other inputs are
    reduced to luma planes first, as the reference's _luma does)."""
    from .render import _default_device
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise DimensionMismatch(f"shapes differ: {a.shape} vs {b.shape}")
    if min(a.shape[0], a.shape[1]) < SSIM_WINDOW:
        raise TooSmall(f"images must be at least {SSIM_WINDOW}x{SSIM_WINDOW}")
    ctx = _lib.context(_default_device if device is None else device)
    h, w = int(a.shape[0]), int(a.shape[1])
    out = ctypes.c_double(0.0)
    if a.dtype == np.uint8 and a.ndim == 3 and a.shape[2] == 3:
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        _lib.check(ctx.lib.gsr_ssim_u8(ctx.handle, _lib.ptr(a), _lib.ptr(b), w, h,
                                       ctypes.byref(out)), "gsr_ssim_u8")
    else:
        x, y = _luma(a), _luma(b)
        _lib.check(ctx.lib.gsr_ssim_luma_f64(ctx.handle, _lib.ptr(x), _lib.ptr(y), w, h,
                                             ctypes.byref(out)), "gsr_ssim_luma_f64")
    return float(out.value)


def upscale_to(img: np.ndarray, width: int, height: int, *, device: int | None = None):
    """metrics.py:125-130: identity when the size matches, else Pillow
    BILINEAR, bit-exact, on the GPU."""
    from .render import _default_device
    if img.shape[1] == width and img.shape[0] == height:
        return img
    src = np.ascontiguousarray(img, dtype=np.uint8)
    if src.ndim != 3 or src.shape[2] != 3:
        raise ValueError("upscale_to expects an (H, W, 3) uint8 image")
    ctx = _lib.context(_default_device if device is None else device)
    out = np.empty((int(height), int(width), 3), dtype=np.uint8)
    _lib.check(ctx.lib.gsr_resample_bilinear_u8(ctx.handle, _lib.ptr(src), src.shape[1],
                                                src.shape[0], _lib.ptr(out), int(width),
                                                int(height)), "gsr_resample_bilinear_u8")
    return out


def ladder_ssim(prims, pose, base_intr, rungs, background=(0.0, 0.0, 0.0), sh_degree: int = 0,
                *, device: int | None = None):
    """Config-3 quality loop fully on the device: render at base_intr, render
    each rung (width, height) with scale_intrinsics (render.py:537), upscale to
    the base size (metrics.py:208) and score SSIM against the base render
    (metrics.py:161-162).  Returns (list of SSIM per rung, base GsrStats)."""
    from .camera import scale_intrinsics
    from .render import _default_device
    dev = _default_device if device is None else device
    sc = device_scene(prims, dev)
    ctx = _lib.context(dev)
    base_cam = make_camera(pose, base_intr)
    cams = (_lib.GsrCamera * max(len(rungs), 1))()
    for i, (w, h) in enumerate(rungs):
        cams[i] = make_camera(pose, scale_intrinsics(base_intr, int(w), int(h)))
    out = (ctypes.c_double * max(len(rungs), 1))()
    st = _lib.GsrStats()
    _lib.check(ctx.lib.gsr_ladder_ssim(ctx.handle, sc.handle, ctypes.byref(base_cam),
                                       _bg(background), int(sh_degree), len(rungs), cams, out,
                                       ctypes.byref(st)), "gsr_ladder_ssim")
    return [float(out[i]) for i in range(len(rungs))], st


__all__ = ["psnr", "ssim", "upscale_to", "ladder_ssim", "MetricError", "DimensionMismatch",
           "TooSmall", "EmptyInput", "IndexOutOfRange"]
