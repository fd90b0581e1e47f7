"""Host-side camera types and view math (mirror of splatstream/camera.py).

The render boundary takes the world-to-camera matrix and camera position as
f64 values computed on the host, exactly as the reference computes them
(camera.py:84-108, render.py:276), so the 12 w2c doubles handed to the GPU
are bit-identical to the ones the reference kernel sees.  Any object with the
same attributes (the reference's own CameraPose/Intrinsics) is accepted by
the renderer; these classes exist so the package runs without the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

Z_NEAR = 0.01                                   # camera.py:17
ELEVATION_EPS = 1e-4                            # camera.py:21
ELEVATION_LIMIT = math.pi / 2 - ELEVATION_EPS   # camera.py:22


@dataclass(frozen=True)
class CameraPose:
    """camera.py:25-44: yaw/pitch + translation; elevation clamped."""

    azimuth: float
    elevation: float
    translation: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        values = (self.azimuth, self.elevation, *self.translation)
        if not all(math.isfinite(v) for v in values):
            raise ValueError("camera pose components must be finite")
        clamped = min(max(self.elevation, -ELEVATION_LIMIT), ELEVATION_LIMIT)
        object.__setattr__(self, "elevation", clamped)
        object.__setattr__(self, "translation", tuple(float(v) for v in self.translation))


def pose_from_degrees(azimuth_deg: float, elevation_deg: float,
                      translation=(0.0, 0.0, 0.0)) -> CameraPose:
    """camera.py:47-50."""
    return CameraPose(math.radians(azimuth_deg), math.radians(elevation_deg), translation)


@dataclass(frozen=True)
class Intrinsics:
    """camera.py:53-73: pinhole parameters with the reference's validation."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise ValueError("focal lengths must be positive")
        if self.width <= 0 or self.height <= 0:
            raise ValueError("image dimensions must be positive")
        if not (0 <= self.cx <= self.width) or not (0 <= self.cy <= self.height):
            raise ValueError("principal point must lie within the image")

    def horizontal_fov(self) -> float:
        return 2.0 * math.atan(self.width / (2.0 * self.fx))


@dataclass(frozen=True)
class ViewTransform:
    rotation: np.ndarray
    world_to_camera: np.ndarray


def rotation_from_angles(azimuth: float, elevation: float) -> np.ndarray:
    """camera.py:84-98: R = R_y(az) @ R_x(el), numpy matmul like the reference."""
    ca, sa = math.cos(azimuth), math.sin(azimuth)
    ce, se = math.cos(elevation), math.sin(elevation)
    r_y = np.array([[ca, 0.0, sa], [0.0, 1.0, 0.0], [-sa, 0.0, ca]])
    r_x = np.array([[1.0, 0.0, 0.0], [0.0, ce, -se], [0.0, se, ce]])
    return r_y @ r_x


def world_to_camera(pose) -> ViewTransform:
    """camera.py:101-108: 4x4 with R^T and -R^T t."""
    rot = rotation_from_angles(pose.azimuth, pose.elevation)
    t = np.asarray(pose.translation, dtype=np.float64)
    mat = np.eye(4)
    mat[:3, :3] = rot.T
    mat[:3, 3] = -rot.T @ t
    return ViewTransform(rotation=rot, world_to_camera=mat)


def camera_position(view: ViewTransform) -> np.ndarray:
    """render.py:276: cam_pos = -R @ w2c[:3, 3]."""
    return -view.rotation @ view.world_to_camera[:3, 3]


def scale_intrinsics(intr, new_width: int, new_height: int) -> Intrinsics:
    """camera.py:146-154: rescale keeping the field of view."""
    if new_width <= 0 or new_height <= 0:
        raise ValueError("new dimensions must be positive")
    sx = new_width / intr.width
    sy = new_height / intr.height
    return Intrinsics(fx=intr.fx * sx, fy=intr.fy * sy, cx=intr.cx * sx, cy=intr.cy * sy,
                      width=int(new_width), height=int(new_height))
