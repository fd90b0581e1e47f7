"""CPU parity oracle for the per-pose render path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this module; the product
(paper_2605_08699_b200) never imports, links or falls back to it.

It drives oracle/oracle.c (a float-exact C restatement of the reference) in
the reference's own stage order:

* ``world_to_camera``            camera.py:84-108 (restated here in numpy)
* ``project_gaussians``          render.py:240-290 -> orc_project + orc_eval_sh
* ``sort_splats``                render.py:293-302 -> orc_stable_argsort
* ``_cutoff_radius_sq``          render.py:476-481 (numpy, same expression)
* ``rasterize``                  render.py:430-473 -> orc_pack + orc_rasterize
* ``framebuffer_to_u8``          render.py:484-485 -> orc_to_u8
* tile-list contract             SURVEY.md A.4     -> orc_tile_keys
* ``upscale_to`` (Pillow)        metrics.py:125-130 -> orc_resample_bilinear
* ``ssim`` (scipy)               metrics.py:76-114 -> orc_ssim
* ``encode_jpeg`` (Pillow/libjpeg-turbo) render.py:488-498 -> orc_jpeg

Pinned by tests/test_oracle_golden.py against vectors produced by the
reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"

TILE = 16
TAIL_SAFETY = 32.0
CUTOFF_SIGMA = 4.5
ELEVATION_LIMIT = math.pi / 2 - 1e-4

_lib = None


def _cc() -> str:
    # a gcc with libgomp; some images put a toolchain without it first on PATH
    for cand in ("/usr/bin/gcc", "gcc"):
        if cand == "gcc" or os.path.exists(cand):
            return cand
    return "gcc"


def build(force: bool = False) -> Path:
    """Compile oracle.c (gcc, -ffp-contract=off, OpenMP) into _build/."""
    src = HERE / "oracle.c"
    if (not force and LIB_PATH.exists()
            and LIB_PATH.stat().st_mtime >= src.stat().st_mtime):
        return LIB_PATH
    LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
    cmd = [_cc(), "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-frounding-math",
           "-fopenmp",
           "-fPIC", "-shared", "-o", str(LIB_PATH), str(src), "-lm"]
    subprocess.run(cmd, check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(LIB_PATH))
        _declare(_lib)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _declare(L):
    vp, i64, dbl, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    L.orc_project.argtypes = [i64, vp, vp, vp, vp, dbl, dbl, dbl, dbl, dbl, dbl, i32,
                              vp, vp, vp, vp, vp]
    L.orc_eval_sh.argtypes = [i64, vp, vp, vp, i32, vp]
    L.orc_stable_argsort.argtypes = [i64, vp, vp]
    L.orc_pack.argtypes = [i64, vp, vp, vp, vp, vp, vp, vp]
    L.orc_rasterize.argtypes = [i64, vp, i64, i64, i64, vp, vp, vp]
    L.orc_to_u8.argtypes = [i64, vp, vp]
    L.orc_tile_keys.argtypes = [i64, vp, i64, i64, i64, vp, vp, vp]
    L.orc_resample_bilinear.argtypes = [vp, i32, i32, vp, i32, i32]
    L.orc_ssim.argtypes = [vp, vp, i32, i32]
    L.orc_ssim.restype = dbl
    L.orc_jpeg.argtypes = [vp, i32, i32, i32, i32, vp, i64]
    L.orc_jpeg.restype = i64
    L.orc_np_exp.argtypes = [i64, vp, vp]
    L.orc_glibc_exp.argtypes = [i64, vp, vp]
    L.orc_np_log.argtypes = [i64, vp, vp]
    L.orc_num_threads.restype = i32
    L.orc_set_num_threads.argtypes = [i32]


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


# --------------------------------------------------------------------------
# host camera math, camera.py:84-108 (numpy, same expression order)
# --------------------------------------------------------------------------

def world_to_camera(azimuth: float, elevation: float, translation=(0.0, 0.0, 0.0)):
    """Returns (R camera-to-world 3x3, world_to_camera 4x4), f64."""
    elevation = min(max(elevation, -ELEVATION_LIMIT), ELEVATION_LIMIT)
    ca, sa = math.cos(azimuth), math.sin(azimuth)
    ce, se = math.cos(elevation), math.sin(elevation)
    r_y = np.array([[ca, 0.0, sa], [0.0, 1.0, 0.0], [-sa, 0.0, ca]])
    r_x = np.array([[1.0, 0.0, 0.0], [0.0, ce, -se], [0.0, se, ce]])
    rot = r_y @ r_x
    t = np.asarray(tuple(float(v) for v in translation), dtype=np.float64)
    mat = np.eye(4)
    mat[:3, :3] = rot.T
    mat[:3, 3] = -rot.T @ t
    return rot, mat


def cutoff_radius_sq(opacities: np.ndarray) -> np.ndarray:
    """render.py:476-481."""
    floor = 1.0 / (255.0 * TAIL_SAFETY)
    with np.errstate(divide="ignore"):
        rsq = 2.0 * np.log(np.maximum(opacities, floor) / floor)
    return np.minimum(rsq, CUTOFF_SIGMA ** 2)


@dataclass
class OracleFrame:
    width: int
    height: int
    keep: np.ndarray        # (N,) bool
    kept: np.ndarray        # (K,) int64 original indices, index order
    order: np.ndarray       # (K,) int64 stable depth order over kept
    depths: np.ndarray      # (K,) f64 depth in sorted order
    packed: np.ndarray      # (K, 11) f32 packed table, sorted order
    rgb32: np.ndarray       # (H, W, 3) f32 before clipping
    trans32: np.ndarray     # (H, W) f32 transmittance
    u8: np.ndarray          # (H, W, 3) u8

    @property
    def splats_drawn(self) -> int:
        return int(self.kept.shape[0])


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def project(means, rotations, scales, w2c, fx, fy, cx, cy, width, height, do_cull=True):
    """render.py:163-237 via orc_project; returns u, v, z, cov(N,3), keep."""
    L = lib()
    n = means.shape[0]
    means, rotations, scales = _c(means, np.float64), _c(rotations, np.float64), _c(scales, np.float64)
    w = _c(np.asarray(w2c)[:3, :], np.float64)
    u = np.empty(n); v = np.empty(n); z = np.empty(n); cov = np.empty((n, 3))
    keep = np.empty(n, dtype=np.uint8)
    L.orc_project(n, _p(means), _p(rotations), _p(scales), _p(w), float(fx), float(fy),
                  float(cx), float(cy), float(width), float(height), int(bool(do_cull)),
                  _p(u), _p(v), _p(z), _p(cov), _p(keep))
    return u, v, z, cov, keep.astype(bool)


def eval_sh(means, sh_coeffs, campos, degree):
    """render.py:126-160 via orc_eval_sh (degree 1..3)."""
    if not 0 <= degree <= 3:
        raise ValueError("SH degree must be in 0..3")
    L = lib()
    n = means.shape[0]
    out = np.empty((n, 3))
    means = _c(means, np.float64)
    sh = _c(sh_coeffs, np.float64)
    cam = _c(campos, np.float64)
    L.orc_eval_sh(n, _p(means), _p(sh), _p(cam), int(degree), _p(out))
    return out


def stable_argsort(keys):
    keys = _c(keys, np.float64)
    order = np.empty(keys.shape[0], dtype=np.int64)
    lib().orc_stable_argsort(keys.shape[0], _p(keys), _p(order))
    return order


def rasterize(packed, width, height, background=(0.0, 0.0, 0.0), n_stripes=None):
    packed = _c(packed, np.float32)
    k = packed.shape[0]
    if n_stripes is None:
        n_stripes = min(max(1, height // 16), 8 * num_threads())
    rgb = np.empty((height, width, 3), dtype=np.float32)
    trans = np.empty((height, width), dtype=np.float32)
    bg = np.asarray(background, dtype=np.float32)
    lib().orc_rasterize(k, _p(packed), width, height, n_stripes, _p(bg), _p(rgb), _p(trans))
    return rgb, trans


def to_u8(rgb32):
    rgb32 = _c(rgb32, np.float32)
    out = np.empty(rgb32.shape, dtype=np.uint8)
    lib().orc_to_u8(rgb32.size, _p(rgb32), _p(out))
    return out


def render(means, scales, rotations, opacities, colors_dc, sh_coeffs, w2c, rot, fx, fy,
           cx, cy, width, height, background=(0.0, 0.0, 0.0), sh_degree=0,
           frustum_culling=True, rsq_all=None) -> OracleFrame:
    """render_framebuffer (render.py:516-524) restated stage by stage."""
    if not 0 <= sh_degree <= 3:
        raise ValueError("SH degree must be in 0..3")
    n = means.shape[0]
    u, v, z, cov, keep = project(means, rotations, scales, w2c, fx, fy, cx, cy, width,
                                 height, frustum_culling)
    if sh_degree == 0:
        colors = np.asarray(colors_dc, dtype=np.float64)
    else:
        cam_pos = -rot @ np.asarray(w2c)[:3, 3]
        colors = eval_sh(means, sh_coeffs, cam_pos, sh_degree)
    kept = np.flatnonzero(keep)
    depths = z[kept]
    order = stable_argsort(depths)
    sidx = kept[order]
    opac = np.asarray(opacities, dtype=np.float64)
    if rsq_all is None:
        rsq = cutoff_radius_sq(opac[sidx])
    else:
        rsq = np.asarray(rsq_all)[sidx]
    k = sidx.shape[0]
    packed = np.empty((k, 11), dtype=np.float32)
    lib().orc_pack(k, _p(_c(u[sidx], np.float64)), _p(_c(v[sidx], np.float64)),
                   _p(_c(cov[sidx], np.float64)), _p(_c(colors[sidx], np.float64)),
                   _p(_c(opac[sidx], np.float64)), _p(_c(rsq, np.float64)), _p(packed))
    rgb, trans = rasterize(packed, width, height, background)
    return OracleFrame(width=width, height=height, keep=keep, kept=kept, order=order,
                       depths=depths[order], packed=packed, rgb32=rgb, trans32=trans,
                       u8=to_u8(rgb))


def tile_lists(packed, width, height, tile=TILE):
    """Tile-list contract.

    Returns (tile_ids, ranks, ranges): entries sorted by (tile, depth rank);
    ranges is (n_tiles, 2) [start, end) into the entry arrays.
    """
    L = lib()
    packed = _c(packed, np.float32)
    k = packed.shape[0]
    counts = np.empty(k, dtype=np.int64)
    L.orc_tile_keys(k, _p(packed), width, height, tile, None, _p(counts), None)
    offsets = np.zeros(k + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    d = int(offsets[-1])
    tiles = np.empty(d, dtype=np.int32)
    L.orc_tile_keys(k, _p(packed), width, height, tile, _p(offsets), None, _p(tiles))
    ranks = np.repeat(np.arange(k, dtype=np.int32), counts)
    order = np.argsort(tiles, kind="stable")
    tiles_sorted = tiles[order]
    ranks_sorted = ranks[order]
    n_tiles = ((width + tile - 1) // tile) * ((height + tile - 1) // tile)
    starts = np.searchsorted(tiles_sorted, np.arange(n_tiles), side="left")
    ends = np.searchsorted(tiles_sorted, np.arange(n_tiles), side="right")
    return tiles_sorted, ranks_sorted, np.stack([starts, ends], axis=1)


def resample_bilinear(img, width, height):
    """metrics.upscale_to restated (Pillow BILINEAR, fixed point)."""
    img = _c(img, np.uint8)
    if img.shape[1] == width and img.shape[0] == height:
        return img
    out = np.empty((height, width, 3), dtype=np.uint8)
    lib().orc_resample_bilinear(_p(img), img.shape[1], img.shape[0], _p(out), width, height)
    return out


def ssim(a, b):
    a = _c(a, np.uint8)
    b = _c(b, np.uint8)
    if a.shape != b.shape:
        raise ValueError("shape mismatch")
    if min(a.shape[0], a.shape[1]) < 11:
        raise ValueError("too small")
    return float(lib().orc_ssim(_p(a), _p(b), a.shape[0], a.shape[1]))


def jpeg(img, quality):
    """render.encode_jpeg restated (Pillow/libjpeg-turbo baseline JPEG,
    4:2:0 below quality 90, 4:4:4 at 90+)."""
    img = _c(img, np.uint8)
    h, w = img.shape[:2]
    cap = 4096 + h * w * 8
    out = np.empty(cap, dtype=np.uint8)
    n = lib().orc_jpeg(_p(img), w, h, int(quality), 1 if quality < 90 else 0, _p(out), cap)
    return out[:n].tobytes()


def psnr(a, b):
    """metrics.py:57-66."""
    mse = np.mean((np.asarray(a).astype(np.float64) - np.asarray(b).astype(np.float64)) ** 2)
    if mse == 0:
        return 100.0
    return min(100.0, 10.0 * math.log10(255.0 ** 2 / mse))


if __name__ == "__main__":  # pragma: no cover
    print(build(force=True))


# --------------------------------------------------------------------------
# PLY load, model.py:105-252 (numpy restatement; transcendental calls through
# the C restatements of numpy's SVML exp/log and glibc's exp)
# --------------------------------------------------------------------------

class PlyError(Exception):
    """Carries the reference's exception class name (model.py:40-57)."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind


PLY_REQUIRED = ("x", "y", "z", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2",
                "rot_3", "opacity", "f_dc_0", "f_dc_1", "f_dc_2")
PLY_REST = tuple(f"f_rest_{i}" for i in range(45))
SH_DC_COEFF = 0.28209479177


def np_exp(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib().orc_np_exp(x.size, _p(x), _p(y))
    return y


def glibc_exp(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib().orc_glibc_exp(x.size, _p(x), _p(y))
    return y


def np_log(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib().orc_np_log(x.size, _p(x), _p(y))
    return y


def ply_header(data: bytes):
    """_parse_header (model.py:105-166): (properties, count, body_offset)."""
    end = data.find(b"end_header")
    if end < 0:
        raise PlyError("MalformedHeader", "no end_header line found")
    newline = data.find(b"\n", end)
    if newline < 0:
        raise PlyError("MalformedHeader", "end_header line is not terminated")
    try:
        text = data[:end].decode("ascii")
    except UnicodeDecodeError as exc:
        raise PlyError("MalformedHeader", f"header is not ASCII: {exc}") from None
    lines = [ln.strip() for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != "ply":
        raise PlyError("MalformedHeader", "missing 'ply' magic line")
    fmt, count, props, in_vertex = False, None, [], False
    for line in lines[1:]:
        parts = line.split()
        bad = lambda m: PlyError("MalformedHeader", m)  # noqa: E731
        if parts[0] == "comment":
            continue
        if parts[0] == "format":
            if parts[1:] != ["binary_little_endian", "1.0"]:
                raise bad(f"unsupported format: {line!r}")
            fmt = True
        elif parts[0] == "element":
            if len(parts) != 3:
                raise bad(f"bad element line: {line!r}")
            if parts[1] != "vertex":
                raise bad(f"unsupported element {parts[1]!r}")
            if count is not None:
                raise bad("multiple vertex elements")
            try:
                count = int(parts[2])
            except ValueError:
                raise bad(f"bad vertex count: {parts[2]!r}") from None
            if count < 0:
                raise bad("negative vertex count")
            in_vertex = True
        elif parts[0] == "property":
            if not in_vertex:
                raise bad("property outside the vertex element")
            if len(parts) != 3:
                raise bad(f"bad property line: {line!r}")
            if parts[1] != "float":
                raise bad(f"only float32 properties supported, got {parts[1]!r}")
            props.append(parts[2])
        else:
            raise bad(f"unexpected header line: {line!r}")
    if not fmt:
        raise PlyError("MalformedHeader", "missing format line")
    if count is None:
        raise PlyError("MalformedHeader", "missing vertex element")
    return props, count, newline + 1


def ply_load(data: bytes) -> dict:
    """activate(parse_ply(data)) (model.py:169-252) + rsq (render.py:476-481).

    Returns the ActivatedPrimitives arrays as a dict, or raises PlyError.
    """
    props, count, off = ply_header(data)
    for name in PLY_REQUIRED:
        if name not in props:
            raise PlyError("MissingProperty", f"required property {name!r} absent")
    n_props = len(props)
    expected = count * n_props * 4
    body = data[off:off + expected]
    if len(body) < expected:
        raise PlyError("TruncatedBody",
                       f"body holds {len(body)} bytes, need {expected} for {count} vertices")
    table = np.frombuffer(body, dtype="<f4").reshape(count, n_props).astype(np.float64)
    col = {name: i for i, name in enumerate(props)}
    grab = lambda names: table[:, [col[n] for n in names]]  # noqa: E731
    means = grab(PLY_REQUIRED[0:3])
    log_scales = grab(PLY_REQUIRED[3:6])
    quats = grab(PLY_REQUIRED[6:10])
    logits = table[:, col["opacity"]]
    sh = np.zeros((count, 16, 3))
    sh[:, 0, :] = grab(PLY_REQUIRED[11:14])
    if all(n in col for n in PLY_REST):
        sh[:, 1:, :] = grab(PLY_REST).reshape(count, 3, 15).transpose(0, 2, 1)
    for name, arr in (("means", means), ("scales", log_scales), ("rotations", quats),
                      ("opacities", logits), ("sh", sh)):
        if not np.all(np.isfinite(arr)):
            raise PlyError("NonFiniteAttribute", f"non-finite values in {name}")
    scales = np_exp(log_scales)
    opac = 1.0 / (1.0 + glibc_exp(-logits))
    s = quats * quats
    norms = np.sqrt(((s[:, 0] + s[:, 1]) + s[:, 2]) + s[:, 3])[:, None]
    with np.errstate(invalid="ignore", divide="ignore"):
        rots = quats / norms
    colors = np.clip(SH_DC_COEFF * sh[:, 0, :] + 0.5, 0.0, 1.0)
    for name, arr in (("scales", scales), ("opacities", opac), ("rotations", rots),
                      ("colors", colors)):
        if not np.all(np.isfinite(arr)):
            raise PlyError("NonFiniteAttribute", f"activation produced non-finite {name}")
    floor = 1.0 / (255.0 * TAIL_SAFETY)
    rsq = np.minimum(2.0 * np_log(np.maximum(opac, floor) / floor), CUTOFF_SIGMA ** 2)
    return {"means": means, "scales": scales, "rotations": rots, "opacities": opac,
            "colors_dc": colors, "sh_coeffs": sh, "rsq": rsq}
