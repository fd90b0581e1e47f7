"""CPU-side checks of the C-ABI library: it loads without a GPU, exports
every symbol include/gsr.h declares, and the product fails loudly (no CPU
fallback) when no device is present."""

from __future__ import annotations

import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    text = (ROOT / "include" / "gsr.h").read_text()
    return sorted(set(re.findall(r"GSR_API\s+[\w\s\*]*?\b(gsr_\w+)\s*\(", text)))


def test_header_declares_abi():
    syms = header_symbols()
    assert "gsr_render" in syms and "gsr_ssim_u8" in syms and "gsr_resample_bilinear_u8" in syms
    assert len(syms) >= 20


def test_library_exports_every_header_symbol():
    from paper_2605_08699_b200 import _lib
    from paper_2605_08699_b200.build import build
    build()
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    declared = {n for n, _, _ in _lib.SIGNATURES}
    assert declared == set(header_symbols())
    assert lib.gsr_abi_version() == 1


def test_no_cpu_fallback_without_device():
    from paper_2605_08699_b200 import _lib
    import paper_2605_08699_b200 as g
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    from paper_2605_08699_b200.synth import synthetic_scene
    prims = synthetic_scene(100, seed=1, sh_degree=0)
    intr = g.Intrinsics(fx=60.0, fy=60.0, cx=32.0, cy=32.0, width=64, height=64)
    with pytest.raises(g.RenderError):
        g.render_framebuffer(prims, g.CameraPose(0, 0), intr)
    with pytest.raises(g.RenderError):
        g.ssim(np.zeros((16, 16, 3), np.uint8), np.ones((16, 16, 3), np.uint8))
    with pytest.raises(g.RenderError):
        g.upscale_to(np.zeros((16, 16, 3), np.uint8), 32, 32)


def test_argument_validation_precedes_device_work():
    import paper_2605_08699_b200 as g
    with pytest.raises(g.TooSmall):
        g.ssim(np.zeros((8, 8, 3)), np.zeros((8, 8, 3)))
    with pytest.raises(g.DimensionMismatch):
        g.ssim(np.zeros((16, 16, 3)), np.zeros((16, 17, 3)))
    img = np.zeros((4, 5, 3), np.uint8)
    assert g.upscale_to(img, 5, 4) is img
