"""Shared pytest configuration.

Markers: ``gpu`` for tests that need a B200 (run on the GPU box with
``pytest -m gpu``); everything else runs on CPU (``-m "not gpu"``).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as o
    o.build()
    return o


def golden_scene(spec):
    """Rebuild a golden scene from its (count, seed, scale_range, rest) spec."""
    from paper_2605_08699_b200.synth import activate, make_synthetic_set, ply_round_trip
    count, seed, sr, rest = spec
    raw = make_synthetic_set(count=count, seed=seed, scale_range=tuple(sr),
                             include_rest=bool(rest))
    return activate(ply_round_trip(raw))


def sweep_scenes():
    """Yields (prims-like dict, pose tuple, golden rgb32, t32, u8) for sweep.npz."""
    from paper_2605_08699_b200.synth import ActivatedPrimitives
    g = np.load(GOLDEN / "sweep.npz")
    off = 0
    for i, c in enumerate(g["counts"]):
        sl = slice(off, off + int(c))
        off += int(c)
        prims = ActivatedPrimitives(means=g["means"][sl], scales=g["scales"][sl],
                                    rotations=g["rotations"][sl], opacities=g["opacities"][sl],
                                    colors_dc=g["colors"][sl],
                                    sh_coeffs=np.zeros((int(c), 16, 3)))
        p = g["poses"][i]
        yield prims, (float(p[0]), float(p[1]), (float(p[2]), float(p[3]), float(p[4]))), \
            g["rgb32"][i], g["t32"][i], g["u8"][i]


def textured(seed=0, h=96, w=128):
    """tests/test_metrics.py:16-22 of the reference."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 255, (h // 8, w // 8, 3), dtype=np.uint8)
    img = np.kron(base, np.ones((8, 8, 1), dtype=np.uint8))
    noise = rng.integers(-12, 13, img.shape)
    return np.clip(img.astype(int) + noise, 0, 255).astype(np.uint8)
