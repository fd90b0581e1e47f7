"""B200-native per-pose Gaussian-splat render path (TIGAS backend, arXiv 2605.08699).

Drop-in for splatstream's renderer API (render_framebuffer / render_view and
the SSIM hook ssim / upscale_to); the hot path runs in libgsr.so, hand-written
CUDA for sm_100a behind the C ABI in include/gsr.h.  See DESIGN.md.
"""

__version__ = "0.1.0"

from .camera import CameraPose, Intrinsics, pose_from_degrees, scale_intrinsics, world_to_camera
from .metrics import (DimensionMismatch, EmptyInput, EvalTriplet, IndexOutOfRange, TooSmall,
                      aggregate_session, evaluate_session_dir, ladder_ssim,
                      materialize_ground_truth, psnr, ssim, upscale_to)
from .render import (DeviceScene, EncodeFailure, Framebuffer, RenderError, RenderPipeline,
                     RenderStats,
                     decode_image, device_scene, encode_jpeg, encode_png, evict,
                     framebuffer_to_u8, render_framebuffer, render_u8, render_view, set_device)
from .model import (DeviceActivatedPrimitives, MalformedHeader, MissingProperty, ModelError,
                    NonFiniteAttribute, TruncatedBody, load_ply, parse_ply_header)
from .registry import DeviceRegistry
from .synth import ActivatedPrimitives

__all__ = [
    "ActivatedPrimitives", "CameraPose", "DeviceRegistry", "DeviceScene", "DimensionMismatch", "EmptyInput",
    "EncodeFailure", "EvalTriplet", "IndexOutOfRange", "aggregate_session", "evaluate_session_dir",
    "materialize_ground_truth",
    "Framebuffer", "Intrinsics", "RenderError", "RenderPipeline", "RenderStats", "TooSmall", "decode_image",
    "device_scene", "encode_jpeg", "encode_png", "evict", "framebuffer_to_u8", "ladder_ssim",
    "pose_from_degrees", "psnr", "render_framebuffer", "render_u8", "render_view",
    "scale_intrinsics", "set_device", "ssim", "upscale_to", "world_to_camera",
    "DeviceActivatedPrimitives", "MalformedHeader", "MissingProperty", "ModelError",
    "NonFiniteAttribute", "TruncatedBody", "load_ply", "parse_ply_header",
]
