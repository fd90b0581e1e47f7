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
from dataclasses import dataclass

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


def _psnr_from_mse(mse: float) -> float:
    if mse == 0:
        return PSNR_CAP_DB
    return min(PSNR_CAP_DB, 10.0 * math.log10(255.0 ** 2 / mse))


def psnr(a, b, *, device: int | None = None) -> float:
    """metrics.py:57-66.  u8 images: the sum of squared differences on the GPU
    (an integer, so the mean -- one f64 division, as numpy's -- and the dB
    value are the reference's exactly); other dtypes: the reference's numpy."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        raise DimensionMismatch(f"shapes differ: {a.shape} vs {b.shape}")
    if a.dtype == np.uint8 and b.dtype == np.uint8 and a.size > 0:
        from .render import _default_device
        ctx = _lib.context(_default_device if device is None else device)
        sse = ctypes.c_uint64(0)
        a = np.ascontiguousarray(a)
        b = np.ascontiguousarray(b)
        _lib.check(ctx.lib.gsr_sse_u8(ctx.handle, _lib.ptr(a), _lib.ptr(b), a.size,
                                      ctypes.byref(sse)), "gsr_sse_u8")
        return _psnr_from_mse(float(sse.value) / a.size)
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


# ---------------------------------------------- session evaluation (8f row 3) --

@dataclass
class EvalTriplet:
    """metrics.py EvalTriplet: transmitted and ground-truth u8 frames."""

    transmitted: np.ndarray
    ground_truth: np.ndarray
    pose: object
    level: int


def materialize_ground_truth(prims, log, sample_indices, background=(0.0, 0.0, 0.0)):
    """metrics.py:133-150: re-render logged poses at base resolution (GPU) as
    lossless PNGs (Pillow, host)."""
    from .camera import pose_from_degrees
    from .render import encode_png, render_framebuffer
    pngs = []
    for idx in sample_indices:
        if not 0 <= idx < len(log.frames):
            raise IndexOutOfRange(f"sample index {idx} outside log of {len(log.frames)}")
        f = log.frames[idx]
        pose = pose_from_degrees(f.azimuth_deg, f.elevation_deg, (f.tx, f.ty, f.tz))
        pngs.append(encode_png(render_framebuffer(prims, pose, log.base_intrinsics, background)))
    return pngs


def _report(rows):
    """metrics.py:153-182's report from (psnr, ssim, level) rows."""
    psnrs = [r[0] for r in rows]
    ssims = [r[1] for r in rows]
    by_level: dict = {}
    for p, s_, lvl in rows:
        by_level.setdefault(lvl, []).append((p, s_))
    return {
        "frames": len(rows),
        "mean_psnr_db": float(np.mean(psnrs)),
        "min_psnr_db": float(np.min(psnrs)),
        "mean_ssim": float(np.mean(ssims)),
        "min_ssim": float(np.min(ssims)),
        "per_level": {
            str(level): {
                "frames": len(vals),
                "mean_psnr_db": float(np.mean([v[0] for v in vals])),
                "mean_ssim": float(np.mean([v[1] for v in vals])),
            }
            for level, vals in sorted(by_level.items())
        },
    }


def aggregate_session(triplets) -> dict:
    """metrics.py:153-182: mean/min PSNR and SSIM plus a per-level breakdown."""
    if not triplets:
        raise EmptyInput("no triplets to aggregate")
    return _report([(psnr(t.transmitted, t.ground_truth), ssim(t.transmitted, t.ground_truth),
                     t.level) for t in triplets])


def evaluate_session_dir(prims, session_dir, background=(0.0, 0.0, 0.0), sh_degree: int = 0,
                         *, device: int | None = None) -> dict:
    """metrics.py:185-214 with each triplet evaluated on the device in one call
    (gsr_eval_frame: GT render at base intrinsics, upscale_to of the decoded
    transmitted frame, SSIM and SSE); only the JPEG decode stays on the host."""
    import json
    from pathlib import Path

    from .camera import Intrinsics, pose_from_degrees
    from .render import _bg, _default_device, decode_image, device_scene, make_camera
    session_dir = Path(session_dir)
    sidecar_path = session_dir / "samples.json"
    if not sidecar_path.is_file():
        raise EmptyInput(f"no samples.json under {session_dir}")
    sidecar = json.loads(sidecar_path.read_text())
    samples = sidecar.get("samples", [])
    if not samples:
        raise EmptyInput("session has no sampled frames")
    base = sidecar["base_intrinsics"]
    base_intr = Intrinsics(fx=base["fx"], fy=base["fy"], cx=base["cx"], cy=base["cy"],
                           width=int(base["width"]), height=int(base["height"]))
    dev = _default_device if device is None else device
    sc = device_scene(prims, dev)
    ctx = _lib.context(dev)
    rows = []
    for sample in samples:
        pose = pose_from_degrees(sample["azimuth_deg"], sample["elevation_deg"],
                                 tuple(sample["translation"]))
        transmitted = np.ascontiguousarray(
            decode_image((session_dir / sample["file"]).read_bytes()), dtype=np.uint8)
        cam = make_camera(pose, base_intr)
        out_ssim = ctypes.c_double(0.0)
        sse = ctypes.c_uint64(0)
        _lib.check(ctx.lib.gsr_eval_frame(ctx.handle, sc.handle, ctypes.byref(cam),
                                          _bg(background), int(sh_degree),
                                          _lib.ptr(transmitted), transmitted.shape[1],
                                          transmitted.shape[0], None, ctypes.byref(out_ssim),
                                          ctypes.byref(sse)), "gsr_eval_frame")
        mse = float(sse.value) / (base_intr.width * base_intr.height * 3)
        rows.append((_psnr_from_mse(mse), float(out_ssim.value), int(sample["level"])))
    report = _report(rows)
    report["model_id"] = sidecar.get("model_id", "")
    return report


__all__ = ["psnr", "ssim", "upscale_to", "ladder_ssim", "MetricError", "DimensionMismatch",
           "TooSmall", "EmptyInput", "IndexOutOfRange", "EvalTriplet", "aggregate_session",
           "evaluate_session_dir", "materialize_ground_truth"]
