"""Generate golden parity vectors by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports splatstream from /root/reference/pkg/src unmodified and records, for
seeded inputs, its outputs as small fixtures (full arrays for tiny cases,
SHA-256 digests of the exact bytes for larger ones).  The fixtures travel with
the repo; /root/reference does not.  Tests compare the oracle (CPU) and the
CUDA path against these.

Recorded cases:
  camera.npz         world_to_camera / scale_intrinsics for 24 poses
  synth.json         digests of activated synthetic scenes (synth -> PLY -> activate)
  sweep.npz          50 random 64x64 scenes (test_render.py:343-356 generator):
                     reference rgb/alpha as f32 + u8
  frames.json/.npz   synthetic scenes through render_framebuffer: keep, stable
                     depth order, packed table (captured from the reference's
                     own rasterize), rgb/T and u8 digests; config-1 u8 frame
  tiles.json         tile-list contract computed by an
                     independent numpy-f32 restatement over the reference's
                     captured packed table
  resample.npz       Pillow BILINEAR via metrics.upscale_to
  ssim.json          metrics.ssim values
  sort.npz           sort_splats known answers
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import splatstream.render as R  # noqa: E402
from splatstream.camera import CameraPose, Intrinsics, scale_intrinsics, world_to_camera  # noqa: E402
from splatstream.metrics import ssim, upscale_to  # noqa: E402
from splatstream.model import ActivatedPrimitives, activate, parse_ply  # noqa: E402
from splatstream.synth import make_synthetic_set, serialize_ply  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def scene(count, seed, scale_range, include_rest):
    raw = make_synthetic_set(count=count, seed=seed, scale_range=scale_range,
                             include_rest=include_rest)
    return activate(parse_ply(serialize_ply(raw, include_rest=True)))


def random_scene(rng, count):
    """tests/test_render.py:33-42."""
    means = np.column_stack([rng.uniform(-1.2, 1.2, count), rng.uniform(-1.2, 1.2, count),
                             rng.uniform(1.5, 6.0, count)])
    scales = rng.uniform(0.02, 0.5, (count, 3))
    quats = rng.normal(size=(count, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    colors = rng.uniform(0, 1, (count, 3))
    opacities = rng.uniform(0.05, 1.0, count)
    return ActivatedPrimitives(means=means, scales=scales, rotations=quats,
                               opacities=opacities, colors_dc=colors,
                               sh_coeffs=np.zeros((count, 16, 3)))


class Capture:
    """Wraps the reference's _count_kernel to capture its packed table."""

    def __init__(self):
        self.packed = None
        self._orig = R._count_kernel

    def __enter__(self):
        def hook(packed, *a):
            self.packed = np.array(packed, copy=True)
            return self._orig(packed, *a)
        R._count_kernel = hook
        return self

    def __exit__(self, *exc):
        R._count_kernel = self._orig


def ref_frame(prims, pose, intr, bg=(0.0, 0.0, 0.0), sh_degree=0):
    stats = R.RenderStats()
    with Capture() as cap:
        fb = R.render_framebuffer(prims, pose, intr, bg, sh_degree, stats)
    view = world_to_camera(pose)
    batch = R.project_gaussians(prims, view, intr, sh_degree=sh_degree)
    u = np.empty(prims.count); v = np.empty(prims.count); z = np.empty(prims.count)
    cov = np.empty((prims.count, 3)); keep = np.empty(prims.count, dtype=np.bool_)
    if prims.count:
        R._project_kernel(prims.means, prims.rotations, prims.scales,
                          np.ascontiguousarray(view.world_to_camera[:3, :]),
                          intr.fx, intr.fy, intr.cx, intr.cy, float(intr.width),
                          float(intr.height), 0.01, R.COV2D_FLOOR, R.CUTOFF_SIGMA, True,
                          u, v, z, cov, keep)
    kept = np.flatnonzero(keep)
    order = np.argsort(z[kept], kind="stable")
    rgb32 = fb.rgb.astype(np.float32)
    t32 = (1.0 - fb.accumulated_alpha).astype(np.float32)
    assert len(batch) == len(kept) == stats.splats_drawn
    return dict(fb=fb, stats=stats, packed=cap.packed, keep=keep, kept=kept, order=order,
                rgb32=rgb32, t32=t32, u8=R.framebuffer_to_u8(fb))


def tile_contract(packed, width, height, tile=16):
    """Independent numpy-f32 restatement of SURVEY.md A.4 over the reference's
    packed table (render.py:329-333 row range, 384-397 interval)."""
    f32 = np.float32
    tiles_x = (width + tile - 1) // tile
    ents_t, ents_r = [], []
    for s in range(packed.shape[0]):
        u, v, ia, ib, ic, rsq = (f32(x) for x in packed[s, :6])
        ry = f32(packed[s, 10])
        lo = max(0, int(np.floor(f32(v - ry))))
        hi = min(height, int(np.ceil(f32(v + ry))) + 1)
        rowmin, rowmax = {}, {}
        for iy in range(lo, hi):
            dy = f32(f32(iy) + f32(0.5)) - v
            dy = f32(dy)
            disc = f32(f32(f32(ib * dy) * f32(ib * dy)) - f32(ia * f32(f32(f32(ic * dy) * dy) - rsq)))
            if not disc > 0:
                continue
            span = f32(np.sqrt(disc) / ia)
            mid = f32(u - f32(f32(ib * dy) / ia))
            x0 = max(0, int(np.floor(f32(mid - span))))
            x1 = min(width, int(np.ceil(f32(mid + span))) + 1)
            if x0 >= x1:
                continue
            ty = iy // tile
            rowmin[ty] = min(rowmin.get(ty, x0), x0)
            rowmax[ty] = max(rowmax.get(ty, x1), x1)
        for ty in sorted(rowmin):
            for tx in range(rowmin[ty] // tile, (rowmax[ty] - 1) // tile + 1):
                ents_t.append(ty * tiles_x + tx)
                ents_r.append(s)
    t = np.asarray(ents_t, dtype=np.int32)
    r = np.asarray(ents_r, dtype=np.int32)
    o = np.argsort(t, kind="stable")
    return t[o], r[o]


def textured(seed=0, h=96, w=128):
    """tests/test_metrics.py:16-22."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 255, (h // 8, w // 8, 3), dtype=np.uint8)
    img = np.kron(base, np.ones((8, 8, 1), dtype=np.uint8))
    noise = rng.integers(-12, 13, img.shape)
    return np.clip(img.astype(int) + noise, 0, 255).astype(np.uint8)


def main():
    # ---------------------------------------------------------------- camera
    rng = np.random.default_rng(2024)
    poses, w2cs, rots, intr_out = [], [], [], []
    for i in range(24):
        az, el = float(rng.uniform(-3.5, 3.5)), float(rng.uniform(-2.0, 2.0))
        t = tuple(float(x) for x in rng.uniform(-5, 5, 3))
        p = CameraPose(az, el, t)
        vt = world_to_camera(p)
        poses.append([az, el, *t]); w2cs.append(vt.world_to_camera); rots.append(vt.rotation)
    base = Intrinsics(fx=1108.512516844081, fy=1108.512516844081, cx=640.0, cy=360.0,
                      width=1280, height=720)
    sizes = [(1920, 1080), (1280, 720), (960, 540), (640, 360), (320, 180), (333, 777)]
    for w, h in sizes:
        s = scale_intrinsics(base, w, h)
        intr_out.append([s.fx, s.fy, s.cx, s.cy, s.width, s.height])
    np.savez_compressed(OUT / "camera.npz", poses=np.array(poses), w2c=np.array(w2cs),
                        rot=np.array(rots), sizes=np.array(sizes), intr=np.array(intr_out))

    # ----------------------------------------------------------------- synth
    synth = {}
    for count, seed, sr, rest in [(1000, 7, (0.02, 0.12), True), (10000, 7, (0.02, 0.12), False),
                                  (2000, 3, (0.01, 0.05), True), (500, 11, (0.02, 0.12), False)]:
        pr = scene(count, seed, sr, rest)
        synth[f"{count}_{seed}_{sr[0]}_{sr[1]}_{int(rest)}"] = {
            k: digest(getattr(pr, k)) for k in
            ("means", "scales", "rotations", "opacities", "colors_dc", "sh_coeffs")}
    (OUT / "synth.json").write_text(json.dumps(synth, indent=1))

    # ----------------------------------------------------------------- sweep
    intr64 = Intrinsics(fx=60.0, fy=60.0, cx=32.0, cy=32.0, width=64, height=64)
    rng = np.random.default_rng(123)
    sweep = {"counts": [], "poses": [], "means": [], "scales": [], "rotations": [],
             "opacities": [], "colors": [], "rgb32": [], "t32": [], "u8": []}
    for _ in range(50):
        count = int(rng.integers(1, 11))
        prims = random_scene(rng, count)
        pose = CameraPose(rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3),
                          tuple(rng.uniform(-0.5, 0.5, 3)))
        fr = ref_frame(prims, pose, intr64)
        sweep["counts"].append(count)
        sweep["poses"].append([pose.azimuth, pose.elevation, *pose.translation])
        for k, a in (("means", prims.means), ("scales", prims.scales),
                     ("rotations", prims.rotations), ("opacities", prims.opacities[:, None]),
                     ("colors", prims.colors_dc)):
            sweep[k].append(a)
        sweep["rgb32"].append(fr["rgb32"]); sweep["t32"].append(fr["t32"])
        sweep["u8"].append(fr["u8"])
    np.savez_compressed(
        OUT / "sweep.npz", counts=np.array(sweep["counts"]), poses=np.array(sweep["poses"]),
        means=np.concatenate(sweep["means"]), scales=np.concatenate(sweep["scales"]),
        rotations=np.concatenate(sweep["rotations"]),
        opacities=np.concatenate(sweep["opacities"])[:, 0],
        colors=np.concatenate(sweep["colors"]), rgb32=np.stack(sweep["rgb32"]),
        t32=np.stack(sweep["t32"]), u8=np.stack(sweep["u8"]))

    # ---------------------------------------------------------------- frames
    cases = [
        # name, (count, seed, scale_range, rest), pose, (W, H, fx), sh, bg
        ("c1_10k_sh0_256", (10000, 7, (0.02, 0.12), False), (0.0, 0.0, (0, 0, 0)),
         (256, 256, 221.70250336881622), 0, (0.0, 0.0, 0.0)),
        ("s1k_sh3_160x120", (1000, 7, (0.02, 0.12), True), (0.07, -0.04, (0.1, -0.05, 0.3)),
         (160, 120, 138.5640646055102), 3, (0.0, 0.0, 0.0)),
        ("s1k_sh1_160x120", (1000, 7, (0.02, 0.12), True), (-0.2, 0.1, (0.0, 0.1, 0.5)),
         (160, 120, 138.5640646055102), 1, (0.25, 0.5, 0.75)),
        ("s1k_sh2_97x61", (1000, 7, (0.02, 0.12), True), (0.3, 0.05, (-0.3, 0.0, 0.2)),
         (97, 61, 70.0), 2, (0.0, 0.0, 0.0)),
        ("s2k_sh3_320x180", (2000, 3, (0.01, 0.05), True), (0.0, 0.0, (0.0, 0.0, 1.0)),
         (320, 180, 277.12812921102034), 3, (0.1, 0.1, 0.1)),
        ("s2k_sh3_back", (2000, 3, (0.01, 0.05), True), (3.14159, 0.0, (0.0, 0.0, 0.0)),
         (320, 180, 277.12812921102034), 3, (0.0, 0.0, 0.0)),
    ]
    frames = {}
    arrays = {}
    tiles = {}
    for name, sc, (az, el, t), (w, h, f), sh, bg in cases:
        prims = scene(*sc)
        pose = CameraPose(az, el, t)
        intr = Intrinsics(fx=f, fy=f, cx=w / 2, cy=h / 2, width=w, height=h)
        fr = ref_frame(prims, pose, intr, bg, sh)
        colors = (R.eval_sh_colors(prims, -world_to_camera(pose).rotation
                                   @ world_to_camera(pose).world_to_camera[:3, 3], sh)
                  if sh else prims.colors_dc)
        frames[name] = dict(
            scene=[sc[0], sc[1], list(sc[2]), sc[3]], pose=[az, el, list(t)],
            intr=[f, f, w / 2, h / 2, w, h], sh=sh, bg=list(bg),
            drawn=fr["stats"].splats_drawn, culled=fr["stats"].splats_culled,
            keep=digest(fr["keep"].astype(np.uint8)), order=digest(fr["order"].astype(np.int64)),
            packed=digest(fr["packed"]), colors=digest(np.asarray(colors, dtype=np.float64)),
            rgb32=digest(fr["rgb32"]), t32=digest(fr["t32"]), u8=digest(fr["u8"]))
        tt, tr = tile_contract(fr["packed"], w, h)
        tiles[name] = dict(D=int(tt.shape[0]), tiles=digest(tt), ranks=digest(tr))
        if w * h <= 256 * 256:
            arrays[name + "_u8"] = fr["u8"]
        print(name, frames[name]["drawn"], tiles[name]["D"], flush=True)
    (OUT / "frames.json").write_text(json.dumps(frames, indent=1))
    (OUT / "tiles.json").write_text(json.dumps(tiles, indent=1))
    np.savez_compressed(OUT / "frames.npz", **arrays)

    # -------------------------------------------------------------- resample
    res = {}
    rs_cases = [((36, 64), (1080, 1920)), ((180, 320), (1080, 1920)), ((360, 640), (1080, 1920)),
                ((540, 960), (1080, 1920)), ((720, 1280), (1080, 1920)), ((1080, 1920), (180, 320)),
                ((61, 97), (200, 311)), ((200, 311), (61, 97)), ((50, 50), (50, 173)),
                ((77, 33), (31, 33))]
    rng = np.random.default_rng(77)
    for i, ((sh_, sw), (dh, dw)) in enumerate(rs_cases):
        src = rng.integers(0, 256, (sh_, sw, 3), dtype=np.uint8)
        out = upscale_to(src, dw, dh)
        res[f"src{i}"] = src if src.size <= 200_000 else np.zeros(0, np.uint8)
        res[f"seed{i}"] = np.array([sh_, sw, dh, dw])
        res[f"digest{i}"] = np.frombuffer(bytes.fromhex(digest(out)), dtype=np.uint8)
        if out.size <= 200_000:
            res[f"out{i}"] = out
    np.savez_compressed(OUT / "resample.npz", n=np.array(len(rs_cases)), **res)

    # ------------------------------------------------------------------ ssim
    ss = {}
    for i in range(6):
        a = textured(3 + i)
        b = np.clip(a.astype(int) + np.random.default_rng(4 + i).integers(-30, 31, a.shape),
                    0, 255).astype(np.uint8)
        ss[f"textured_{i}"] = repr(ssim(a, b))
    ss["identical"] = repr(ssim(textured(1), textured(1)))
    ss["inverted"] = repr(ssim(textured(2), 255 - textured(2)))
    r = np.random.default_rng(9)
    a = r.integers(0, 256, (11, 22, 3), dtype=np.uint8)
    b = r.integers(0, 256, (11, 22, 3), dtype=np.uint8)
    ss["small_11x22"] = repr(ssim(a, b))
    a = r.integers(0, 256, (37, 53, 3), dtype=np.uint8)
    ss["noise_37x53"] = repr(ssim(a, np.clip(a.astype(int) + 7, 0, 255).astype(np.uint8)))
    (OUT / "ssim.json").write_text(json.dumps(ss, indent=1))

    # ------------------------------------------------------------------ sort
    rng = np.random.default_rng(1)
    depths = rng.uniform(0, 100, 1000)
    ties = np.repeat(rng.uniform(0, 5, 50), 20)
    rng.shuffle(ties)
    np.savez_compressed(OUT / "sort.npz", depths=depths,
                        order=np.argsort(depths, kind="stable"), ties=ties,
                        ties_order=np.argsort(ties, kind="stable"))
    print("golden vectors written to", OUT)


if __name__ == "__main__":
    main()
