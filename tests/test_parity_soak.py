"""Randomised parity soak: seeded random scenes, SH degrees, resolutions
(odd sizes included), backgrounds and poses; every frame from the CUDA path
(render_framebuffer through the C ABI) must be float-bit-identical to the C
oracle (f32 rgb planes, transmittance, u8) with the same drawn count.

GSR_SOAK_CASES sets the number of cases (default 24, about a minute on a
B200 box); GSR_SOAK_SEED the base seed.  The summary line is printed so a
long run can be kept as evidence (profiles/r01_parity_soak.txt).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(g, synth, rng):
    n = int(rng.choice([1, 7, 500, 5_000, 40_000, 150_000]))
    sh = int(rng.integers(0, 4))
    sr = synth.scale_range_for(max(n, 1000)) if rng.random() < 0.7 else (0.001, 0.4)
    raw = synth.make_synthetic_set(count=n, seed=int(rng.integers(1 << 30)), scale_range=sr,
                                   include_rest=sh > 0)
    prims = synth.activate(synth.ply_round_trip(raw))
    w = int(rng.choice([16, 33, 256, 320, 641, 960, 1280]))
    h = int(rng.choice([9, 64, 180, 241, 540, 720]))
    hfov = float(rng.uniform(0.5, 1.6))
    fx = w / (2.0 * np.tan(hfov / 2.0))
    intr = g.Intrinsics(fx=fx, fy=fx * float(rng.uniform(0.8, 1.25)),
                        cx=float(np.clip(w / 2.0 + rng.normal(0, 3), 0.5, w - 0.5)),
                        cy=float(np.clip(h / 2.0 + rng.normal(0, 3), 0.5, h - 0.5)),
                        width=w, height=h)
    pose = g.pose_from_degrees(float(rng.uniform(-60, 60)), float(rng.uniform(-30, 30)),
                               tuple(float(x) for x in rng.uniform(-0.5, 0.5, 3)))
    bg = (0.0, 0.0, 0.0) if rng.random() < 0.6 else tuple(float(x) for x in rng.random(3))
    return prims, intr, pose, sh, bg


def test_random_frames_bit_exact(oracle):
    _soak(oracle, int(os.environ.get("GSR_SOAK_CASES", "24")),
          int(os.environ.get("GSR_SOAK_SEED", "20261017")))


def test_capacity_history_regression(oracle):
    """Seed 777's cases 0..109 rendered in a fresh process, then case 110
    (150k large splats, 7M tile keys at 320x241) compared with the oracle.
    With that history case 110's tile-key capacity grew inside an existing
    allocation (no new buffer generation), and its frame graph, keyed by the
    generation only, was replayed with the old capacity baked in: the lists
    overflowed again while the host saw the frame fit, and the frame came back
    empty.  The graph key now includes the capacities.  (A fresh process:
    the allocation history is what triggers it.)"""
    import subprocess
    import sys
    root = os.path.join(os.path.dirname(__file__), "..")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "debug_soak_case.py"),
                        "777", "110", "0"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def _soak(oracle, cases, seed):
    import paper_2605_08699_b200 as g
    from paper_2605_08699_b200 import _lib, synth
    if _lib.device_count() == 0:
        pytest.fail("no CUDA device visible to libgsr")
    rng = np.random.default_rng(seed)
    px = evals = 0
    only = os.environ.get("GSR_SOAK_ONLY")  # debugging: render just this case index
    for k in range(cases):
        prims, intr, pose, sh, bg = _case(g, synth, rng)
        if only is not None and k != int(only):
            continue
        if os.environ.get("GSR_SOAK_VERBOSE"):
            print("case", k, prims.count, sh, intr, pose, bg, flush=True)
        st = g.RenderStats()
        fb = g.render_framebuffer(prims, pose, intr, bg, sh, st)
        rot, w2c = oracle.world_to_camera(pose.azimuth, pose.elevation, pose.translation)
        ref = oracle.render(prims.means, prims.scales, prims.rotations, prims.opacities,
                            prims.colors_dc, prims.sh_coeffs, w2c, rot, intr.fx, intr.fy,
                            intr.cx, intr.cy, intr.width, intr.height, bg, sh)
        what = (k, prims.count, sh, intr.width, intr.height, bg)
        assert st.splats_drawn == ref.splats_drawn, what
        assert np.array_equal(fb.u8, ref.u8), what
        assert np.array_equal(fb._rgb32.view(np.uint32), ref.rgb32.view(np.uint32)), what
        assert np.array_equal(fb._t32.view(np.uint32), ref.trans32.view(np.uint32)), what
        px += intr.width * intr.height
        evals += st.splats_drawn
        g.evict(prims)
    print(f"soak: {cases} random frames bit-exact vs the oracle "
          f"({px / 1e6:.1f} Mpx, {evals} splats drawn)")


def test_pipeline_random_scenes_bit_exact(oracle):
    """RenderPipeline (3 frames in flight, contexts rotating) over a random
    mix of scenes -- small, large, and 150k large splats whose first frames
    overflow the tile-key buffers and re-render while other frames are in
    flight -- every returned frame bit-exact (u8) vs the oracle."""
    import paper_2605_08699_b200 as g
    from paper_2605_08699_b200 import synth
    rng = np.random.default_rng(31)
    intr = g.Intrinsics(fx=300.0, fy=320.0, cx=160.0, cy=120.5, width=320, height=241)
    specs = [(500, None), (2_000, None), (40_000, None), (150_000, (0.001, 0.4)),
             (80_000, None), (150_000, None)]
    scenes = []
    for k, (n, sr) in enumerate(specs):
        raw = synth.make_synthetic_set(count=n, seed=100 + k,
                                       scale_range=sr or synth.scale_range_for(n),
                                       include_rest=True)
        scenes.append(synth.activate(synth.ply_round_trip(raw)))
    jobs = {}
    pipe = g.RenderPipeline(intr, sh_degree=3, depth=3)

    def check(tag, frame):
        k, pose = jobs.pop(tag)
        p = scenes[k]
        rot, w2c = oracle.world_to_camera(pose.azimuth, pose.elevation, pose.translation)
        ref = oracle.render(p.means, p.scales, p.rotations, p.opacities, p.colors_dc,
                            p.sh_coeffs, w2c, rot, intr.fx, intr.fy, intr.cx, intr.cy,
                            intr.width, intr.height, (0.0, 0.0, 0.0), 3)
        assert np.array_equal(frame, ref.u8), (tag, k)

    try:
        for t in range(30):
            k = int(rng.integers(len(scenes)))
            pose = g.pose_from_degrees(float(rng.uniform(-40, 40)), float(rng.uniform(-20, 20)),
                                       tuple(float(x) for x in rng.uniform(-0.3, 0.3, 3)))
            jobs[t] = (k, pose)
            r = pipe.submit(scenes[k], pose, tag=t)
            if r is not None:
                check(r[0], r[1].copy())
        for tag, frame in pipe.drain():
            check(tag, frame.copy())
    finally:
        pipe.close()
    assert not jobs
