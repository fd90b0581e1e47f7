"""Full-scale golden digests produced by running the UNMODIFIED reference
(/root/reference/pkg/src/splatstream, numba + numpy + scipy + Pillow) in the
build container, at BASELINE configs 2 and 3 (VERDICT r1 "next" 1c/1b):

  config2_pose0   500k Gaussians, SH3, 1280x720, pose 0 of the config-2 test
                  trace (pose_trace(300, seed=2)[0])
  config3_pose0   3M Gaussians, SH3, 1920x1080, pose 0 of the bench trace
                  (pose_trace(n, seed=0)[0])
  config3_ladder  the same 3M scene and pose through the ABR ladder: each
                  rung (1280x720, 960x540, 640x360) rendered at
                  scale_intrinsics(base, w, h), upscaled to 1080p with
                  metrics.upscale_to and scored with metrics.ssim against the
                  1080p frame (metrics.py:76-130, render.py:527-541)

Per case: the scene arrays' digests (the reference's own make_synthetic_set
-> serialize_ply -> parse_ply -> activate), drawn/culled counts, and the
sha256 of the keep mask, the stable depth order (positions in the kept
list), the packed table captured from the reference's own rasterize, rgb /
T (f32) and the u8 frame.  The GPU box has no /root/reference: the tests
compare the device (and the C oracle) with these committed digests.

    python tests/golden/make_fullscale_golden.py      # ~3 min on 8 cores
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_golden")
sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent.parent))

import numpy as np  # noqa: E402

from make_golden import digest, ref_frame, scene  # noqa: E402  (reference imports)
import splatstream.render as R  # noqa: E402
from splatstream.camera import Intrinsics, pose_from_degrees, scale_intrinsics  # noqa: E402
from splatstream.metrics import ssim, upscale_to  # noqa: E402

from paper_2605_08699_b200.synth import pose_trace, scale_range_for  # noqa: E402


def base_1080p():
    base = Intrinsics(fx=1108.512516844081, fy=1108.512516844081, cx=640.0, cy=360.0,
                      width=1280, height=720)  # harness.py:33-35
    return scale_intrinsics(base, 1920, 1080)


def case_record(count, seed, sh, pose_deg, intr, prims, fr):
    kept = fr["kept"]
    return dict(
        scene=[count, seed, list(scale_range_for(count)), sh > 0], sh=sh,
        pose_deg=[pose_deg[0], pose_deg[1], list(pose_deg[2])],
        intr=[intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height],
        scene_digests={k: digest(getattr(prims, k)) for k in
                       ("means", "scales", "rotations", "opacities", "colors_dc", "sh_coeffs")},
        drawn=int(fr["stats"].splats_drawn), culled=int(fr["stats"].splats_culled),
        keep=digest(fr["keep"].astype(np.uint8)),
        order=digest(np.asarray(fr["order"], dtype=np.int64)),
        order_index=digest(kept[fr["order"]].astype(np.int64)),
        packed=digest(fr["packed"]), rgb32=digest(np.clip(fr["rgb32"], 0, 1)),
        t32=digest(fr["t32"]), u8=digest(fr["u8"]))


def main():
    out = {}
    # ---- config 2, pose 0 of the test trace
    t0 = time.time()
    n2 = 500_000
    prims2 = scene(n2, 7, scale_range_for(n2), True)
    intr2 = scale_intrinsics(base_1080p(), 1280, 720)
    tp = pose_trace(300, seed=2)[0]
    pd = (tp.azimuth_deg, tp.elevation_deg, tuple(tp.translation))
    fr = ref_frame(prims2, pose_from_degrees(*pd), intr2, (0.0, 0.0, 0.0), 3)
    out["config2_pose0"] = case_record(n2, 7, 3, pd, intr2, prims2, fr)
    print("config2", out["config2_pose0"]["drawn"], f"{time.time() - t0:.1f}s", flush=True)
    del prims2, fr

    # ---- config 3, pose 0 of the bench trace, + the ABR ladder
    t0 = time.time()
    n3 = 3_000_000
    prims3 = scene(n3, 7, scale_range_for(n3), True)
    intr3 = base_1080p()
    tp = pose_trace(8, seed=0)[0]
    pd = (tp.azimuth_deg, tp.elevation_deg, tuple(tp.translation))
    pose = pose_from_degrees(*pd)
    fr = ref_frame(prims3, pose, intr3, (0.0, 0.0, 0.0), 3)
    out["config3_pose0"] = case_record(n3, 7, 3, pd, intr3, prims3, fr)
    print("config3", out["config3_pose0"]["drawn"], f"{time.time() - t0:.1f}s", flush=True)
    gt = fr["u8"]
    ladder = {"pose_deg": [pd[0], pd[1], list(pd[2])], "rungs": []}
    for w, h in ((1280, 720), (960, 540), (640, 360)):
        ri = scale_intrinsics(intr3, w, h)
        st = R.RenderStats()
        fb = R.render_framebuffer(prims3, pose, ri, (0.0, 0.0, 0.0), 3, st)
        lo = R.framebuffer_to_u8(fb)
        up = upscale_to(lo, intr3.width, intr3.height)
        ladder["rungs"].append(dict(width=w, height=h, drawn=int(st.splats_drawn),
                                    intr=[ri.fx, ri.fy, ri.cx, ri.cy, ri.width, ri.height],
                                    u8=digest(lo), upscaled=digest(up),
                                    ssim=float(ssim(up, gt))))
        print("rung", w, h, ladder["rungs"][-1]["ssim"], flush=True)
    out["config3_ladder"] = ladder
    (HERE / "fullscale.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
