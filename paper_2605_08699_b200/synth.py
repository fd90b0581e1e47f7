"""Seeded synthetic scenes and pose traces for benchmarks and tests.

``make_synthetic_set`` restates splatstream/synth.py:12-39 draw for draw
(same numpy Generator calls in the same order), and ``synthetic_scene``
applies the PLY float32 round trip (synth.py:42-65 -> model.py:169-220) and
``activate`` (model.py:223-252), so a scene built here is bit-identical to the
one the reference serves from disk.  tests/golden pins this with hashes made
by the reference itself.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SH_COEFF_COUNT = 16           # model.py:27
SH_DC_COEFF = 0.28209479177   # model.py:25


@dataclass
class GaussianPrimitiveSet:
    """model.py:77-86: raw attributes as stored in the PLY."""

    count: int
    means: np.ndarray
    log_scales: np.ndarray
    quaternions: np.ndarray
    opacity_logits: np.ndarray
    sh_coeffs: np.ndarray


@dataclass
class ActivatedPrimitives:
    """model.py:89-102: the renderer's input type."""

    means: np.ndarray       # (N, 3)
    scales: np.ndarray      # (N, 3)
    rotations: np.ndarray   # (N, 4) unit wxyz
    opacities: np.ndarray   # (N,)
    colors_dc: np.ndarray   # (N, 3)
    sh_coeffs: np.ndarray   # (N, 16, 3)

    @property
    def count(self) -> int:
        return self.means.shape[0]


def make_synthetic_set(count=1000, seed=7, center=(0.0, 0.0, 4.0), extent=(3.0, 2.0, 2.0),
                       scale_range=(0.02, 0.12), include_rest=False) -> GaussianPrimitiveSet:
    """synth.py:12-39."""
    rng = np.random.default_rng(seed)
    center = np.asarray(center)
    extent = np.asarray(extent)
    means = center + (rng.random((count, 3)) - 0.5) * extent
    log_scales = np.log(rng.uniform(scale_range[0], scale_range[1], size=(count, 3)))
    quats = rng.normal(size=(count, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    opacity_logits = rng.uniform(-1.0, 3.0, size=count)
    sh = np.zeros((count, SH_COEFF_COUNT, 3))
    sh[:, 0, :] = rng.uniform(-1.8, 1.8, size=(count, 3))
    if include_rest:
        sh[:, 1:, :] = rng.normal(scale=0.2, size=(count, SH_COEFF_COUNT - 1, 3))
    return GaussianPrimitiveSet(count=count, means=means, log_scales=log_scales,
                                quaternions=quats, opacity_logits=opacity_logits,
                                sh_coeffs=sh)


def ply_round_trip(raw: GaussianPrimitiveSet) -> GaussianPrimitiveSet:
    """serialize_ply -> parse_ply: every attribute through float32."""
    f = lambda a: np.asarray(a).astype("<f4").astype(np.float64)
    return GaussianPrimitiveSet(count=raw.count, means=f(raw.means),
                                log_scales=f(raw.log_scales),
                                quaternions=f(raw.quaternions),
                                opacity_logits=f(raw.opacity_logits),
                                sh_coeffs=f(raw.sh_coeffs))


PLY_REQUIRED = ("x", "y", "z", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2",
                "rot_3", "opacity", "f_dc_0", "f_dc_1", "f_dc_2")   # model.py:31-36
PLY_REST = tuple(f"f_rest_{i}" for i in range(45))


def serialize_ply(prims: GaussianPrimitiveSet, include_rest: bool = True) -> bytes:
    """synth.py:40-64: binary little-endian splat PLY (f_rest channel-major)."""
    names = list(PLY_REQUIRED) + (list(PLY_REST) if include_rest else [])
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {prims.count}"]
    header += [f"property float {name}" for name in names] + ["end_header"]
    n = prims.count
    cols = [np.asarray(prims.means).reshape(n, 3), np.asarray(prims.log_scales).reshape(n, 3),
            np.asarray(prims.quaternions).reshape(n, 4),
            np.asarray(prims.opacity_logits).reshape(n, 1),
            np.asarray(prims.sh_coeffs)[:, 0, :].reshape(n, 3)]
    if include_rest:
        cols.append(np.asarray(prims.sh_coeffs)[:, 1:, :].transpose(0, 2, 1).reshape(n, -1))
    table = np.concatenate(cols, axis=1).astype("<f4")
    return ("\n".join(header) + "\n").encode("ascii") + table.tobytes()


def activate(prims: GaussianPrimitiveSet) -> ActivatedPrimitives:
    """model.py:223-252."""
    from scipy.special import expit
    with np.errstate(over="ignore"):
        scales = np.exp(prims.log_scales)
    opacities = expit(prims.opacity_logits)
    norms = np.linalg.norm(prims.quaternions, axis=1, keepdims=True)
    with np.errstate(invalid="ignore", divide="ignore"):
        rotations = prims.quaternions / norms
    colors_dc = np.clip(SH_DC_COEFF * prims.sh_coeffs[:, 0, :] + 0.5, 0.0, 1.0)
    return ActivatedPrimitives(means=prims.means.copy(), scales=scales, rotations=rotations,
                               opacities=opacities, colors_dc=colors_dc,
                               sh_coeffs=prims.sh_coeffs.copy())


def scale_range_for(count: int) -> tuple[float, float]:
    """R(N) = (0.02, 0.12) * (1e4 / N)^(1/3)."""
    f = (1e4 / count) ** (1.0 / 3.0)
    return (0.02 * f, 0.12 * f)


def synthetic_scene(count: int, seed: int = 7, sh_degree: int = 3,
                    scale_range=None) -> ActivatedPrimitives:
    """Benchmark scene: synth -> PLY round trip -> activate."""
    if scale_range is None:
        scale_range = scale_range_for(count)
    raw = make_synthetic_set(count=count, seed=seed, scale_range=scale_range,
                             include_rest=sh_degree > 0)
    return activate(ply_round_trip(raw))


@dataclass(frozen=True)
class TracePose:
    t_ms: float
    azimuth_deg: float
    elevation_deg: float
    translation: tuple


def pose_trace(n: int, seed: int = 0, hz: float = 30.0) -> list[TracePose]:
    """Seeded smooth EyeNavGS-style head-motion walk.

    Yaw/pitch follow a damped random walk (degrees), translation drifts
    slowly and is kept in front of the scene (tz <= 1.5).  Emits the harness
    movement CSV fields (harness.py:109-133).
    """
    rng = np.random.default_rng(seed)
    az, el = 0.0, 0.0
    vaz, vel = 0.0, 0.0
    pos = np.zeros(3)
    vpos = np.zeros(3)
    out = []
    for i in range(n):
        vaz = 0.9 * vaz + rng.normal(scale=0.35)
        vel = 0.9 * vel + rng.normal(scale=0.2)
        az = float(np.clip(az + vaz, -25.0, 25.0))
        el = float(np.clip(el + vel, -15.0, 15.0))
        vpos = 0.95 * vpos + rng.normal(scale=0.002, size=3)
        pos = pos + vpos
        pos[0] = float(np.clip(pos[0], -0.6, 0.6))
        pos[1] = float(np.clip(pos[1], -0.4, 0.4))
        pos[2] = float(np.clip(pos[2], -0.8, 1.5))
        out.append(TracePose(t_ms=1000.0 * i / hz, azimuth_deg=az, elevation_deg=el,
                             translation=(float(pos[0]), float(pos[1]), float(pos[2]))))
    return out


def trace_to_csv(trace) -> str:
    lines = ["t_ms,azimuth_deg,elevation_deg,tx,ty,tz"]
    for p in trace:
        lines.append(f"{p.t_ms:.3f},{p.azimuth_deg!r},{p.elevation_deg!r},"
                     f"{p.translation[0]!r},{p.translation[1]!r},{p.translation[2]!r}")
    return "\n".join(lines) + "\n"


def ladder_1080p():
    """Config 3 ladder 1080p/720p/540p/360p (abr.py:92-100 field names)."""
    return [dict(width=1920, height=1080, jpeg_quality=90, expected_kb=400),
            dict(width=1280, height=720, jpeg_quality=90, expected_kb=240),
            dict(width=960, height=540, jpeg_quality=65, expected_kb=55),
            dict(width=640, height=360, jpeg_quality=35, expected_kb=20)]


def base_intrinsics_1080p():
    """harness.py:33-35 DEFAULT_BASE_INTRINSICS rescaled to 1920x1080."""
    from .camera import Intrinsics, scale_intrinsics
    base = Intrinsics(fx=1108.512516844081, fy=1108.512516844081, cx=640.0, cy=360.0,
                      width=1280, height=720)
    return scale_intrinsics(base, 1920, 1080)


__all__ = ["ActivatedPrimitives", "GaussianPrimitiveSet", "make_synthetic_set",
           "ply_round_trip", "serialize_ply", "activate", "synthetic_scene", "scale_range_for",
           "pose_trace", "trace_to_csv", "ladder_1080p", "base_intrinsics_1080p"]
