"""Generate golden PLY-load vectors by running the REFERENCE itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ply_golden.py

For each case a PLY byte string is built here (an independent struct/numpy
writer, not the reference's) and passed to the reference's unmodified
``splatstream.model.parse_ply`` + ``activate`` and ``render._cutoff_radius_sq``.
Recorded in tests/golden/ply/:
  cases.json   name -> {"file", "expect": "ok" | exception class, "message",
                        "count", "body_offset"}
  <name>.ply   the input bytes
  arrays.npz   "<name>/<attr>" -> the reference's f64 arrays for "ok" cases
               (means, scales, rotations, opacities, colors_dc, sh_coeffs, rsq)
"""

from __future__ import annotations

import json
import os
import shutil
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_golden")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from splatstream import model as ref_model  # noqa: E402
from splatstream import render as ref_render  # noqa: E402

OUT = Path(__file__).resolve().parent / "ply"

REQ = ["x", "y", "z", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3",
       "opacity", "f_dc_0", "f_dc_1", "f_dc_2"]
REST = [f"f_rest_{i}" for i in range(45)]


def ply(props, table, count=None, fmt="format binary_little_endian 1.0", extra_lines=(),
        newline="\n", element=None):
    table = np.asarray(table, dtype="<f4").reshape(-1, len(props))
    n = table.shape[0] if count is None else count
    lines = ["ply", fmt, *extra_lines, element or f"element vertex {n}"]
    lines += [f"property float {p}" for p in props] + ["end_header"]
    return (newline.join(lines) + newline).encode("ascii") + table.tobytes()


def random_table(rng, n, props, ls=(-6.0, 1.0), logit=(-8.0, 8.0)):
    cols = {}
    for k in range(3):
        cols[f"{'xyz'[k]}"] = rng.uniform(-50, 50, n)
        cols[f"scale_{k}"] = rng.uniform(ls[0], ls[1], n)
        cols[f"f_dc_{k}"] = rng.uniform(-2, 2, n)
    for k in range(4):
        cols[f"rot_{k}"] = rng.normal(size=n)
    cols["opacity"] = rng.uniform(logit[0], logit[1], n)
    for name in REST:
        cols[name] = rng.normal(scale=0.3, size=n)
    return np.stack([cols.get(p, rng.normal(size=n)) for p in props], axis=1)


def cases():
    rng = np.random.default_rng(20260517)
    full = REQ + REST
    out = {}
    out["empty"] = ply(REQ, np.zeros((0, 14)))
    out["single_exact"] = ply(REQ, [[0, 0, 0, np.log(0.5), np.log(0.5), np.log(0.5), 1, 0, 0, 0,
                                     4.0, 1.0, 0, 0]])
    out["random_rest_33"] = ply(full, random_table(rng, 33, full))
    out["random_norest_17"] = ply(REQ, random_table(rng, 17, REQ))
    props = REQ[:3] + ["nx", "ny", "nz"] + REQ[3:]
    out["extra_props"] = ply(props, random_table(rng, 9, props))
    props = REQ + ["opacity"]  # duplicate name: the last column wins (dict)
    out["duplicate_prop"] = ply(props, random_table(rng, 7, props))
    out["partial_rest"] = ply(REQ + REST[:44], random_table(rng, 5, REQ + REST[:44]))
    out["crlf_comments"] = ply(full, random_table(rng, 6, full),
                               extra_lines=("comment made by hand", "  comment   spaced  "),
                               newline="\r\n")
    out["count_underscore"] = ply(REQ, random_table(rng, 12, REQ), element="element vertex 1_2")
    out["count_plus_zeros"] = ply(REQ, random_table(rng, 3, REQ), element="element vertex +003")
    out["wide_ranges_600"] = ply(full, random_table(rng, 600, full, ls=(-30.0, 12.0),
                                                    logit=(-40.0, 40.0)))
    t = random_table(rng, 8, REQ)
    t[:, 10] = [-1000.0, 1000.0, -100.0, 100.0, -745.5, 709.0, -0.0, 1e-30]
    t[:, 3] = [-700.0, 700.0, -80.0, 80.0, 1e-30, -1e-30, 0.0, -0.0]
    t[:, 6:10] = [[1e-30, 0, 0, 0], [0, 0, 0, 3e38], [1, 1, 1, 1], [-1, 0, 0, 0],
                  [1e-20, 1e-20, 0, 0], [2, -3, 5, -7], [0, 0, 1e-40, 0], [0.5, 0.5, 0.5, 0.5]]
    t[:, 11] = [-1e30, 1e30, -1.7724538509, 1.7724538509, 0, -0.0, 3.0, -3.0]
    out["edge_values"] = ply(REQ, t)
    # reference errors
    base = ply(REQ, random_table(rng, 4, REQ))
    out["err_ascii_format"] = ply(REQ, np.zeros((0, 14)), fmt="format ascii 1.0")
    out["err_big_endian"] = ply(REQ, np.zeros((0, 14)), fmt="format binary_big_endian 1.0")
    out["err_no_magic"] = base[4:]
    out["err_missing_opacity"] = ply([p for p in REQ if p != "opacity"], np.zeros((0, 13)))
    out["err_truncated"] = ply(REQ, random_table(rng, 10, REQ))[:-5]
    out["err_uchar_prop"] = ply(REQ, np.zeros((0, 14))).replace(b"property float opacity",
                                                               b"property uchar opacity")
    out["err_no_end_header"] = b"ply\nformat binary_little_endian 1.0\nelement vertex 0\n"
    out["err_end_header_unterminated"] = b"ply\nformat binary_little_endian 1.0\nend_header"
    out["err_non_ascii"] = base.replace(b"ply\n", b"ply\ncomment caf\xc3\xa9\n", 1)
    out["err_element_face"] = ply(REQ, np.zeros((0, 14)), element="element face 3")
    out["err_element_short"] = ply(REQ, np.zeros((0, 14)), element="element vertex")
    out["err_two_vertex_elements"] = ply(REQ, np.zeros((0, 14)),
                                         extra_lines=("element vertex 0",))
    out["err_bad_count"] = ply(REQ, np.zeros((0, 14)), element="element vertex 1__0")
    out["err_negative_count"] = ply(REQ, np.zeros((0, 14)), element="element vertex -1")
    out["err_property_first"] = b"ply\nformat binary_little_endian 1.0\nproperty float x\n" \
                                b"element vertex 0\nend_header\n"
    out["err_property_list"] = ply(REQ, np.zeros((0, 14))).replace(
        b"property float x\n", b"property list uchar int x\n")
    out["err_unexpected_line"] = ply(REQ, np.zeros((0, 14)), extra_lines=("obj_info it's mine",))
    out["err_unexpected_tab"] = ply(REQ, np.zeros((0, 14)), extra_lines=("obj\tinfo \\x",))
    out["err_missing_format"] = b"ply\nelement vertex 0\nproperty float x\nend_header\n"
    out["err_missing_vertex"] = b"ply\nformat binary_little_endian 1.0\nend_header\n"
    out["err_format_extra"] = ply(REQ, np.zeros((0, 14)),
                                  fmt="format binary_little_endian 1.0 extra")
    out["err_comment_end_header"] = b"ply\ncomment end_header\nformat binary_little_endian 1.0\n" \
                                    b"element vertex 0\nend_header\n"
    t = random_table(rng, 3, REQ)
    t[1, 0] = np.nan
    out["err_nan_mean"] = ply(REQ, t)
    t = random_table(rng, 3, REQ)
    t[2, 4] = np.inf
    out["err_inf_log_scale"] = ply(REQ, t)
    t = random_table(rng, 3, REQ)
    t[0, 8] = -np.inf
    out["err_inf_quat"] = ply(REQ, t)
    t = random_table(rng, 3, REQ)
    t[0, 10] = np.nan
    out["err_nan_logit"] = ply(REQ, t)
    t = random_table(rng, 3, full)
    t[1, 14 + 20] = np.nan
    out["err_nan_rest"] = ply(full, t)
    t = random_table(rng, 3, REQ + REST[:10])
    t[1, 14 + 5] = np.nan  # not all f_rest present: ignored
    out["ok_nan_in_ignored_rest"] = ply(REQ + REST[:10], t)
    t = random_table(rng, 3, REQ)
    t[1, 5] = 800.0
    out["err_scale_overflow"] = ply(REQ, t)
    t = random_table(rng, 3, REQ)
    t[2, 6:10] = 0.0
    out["err_zero_quat"] = ply(REQ, t)
    t = random_table(rng, 3, REQ)
    t[1, 0] = np.nan
    t[2, 5] = 800.0
    out["err_raw_before_activation"] = ply(REQ, t)
    return out


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    manifest, arrays = {}, {}
    for name, data in cases().items():
        (OUT / f"{name}.ply").write_bytes(data)
        ent = {"file": f"{name}.ply"}
        try:
            raw = ref_model.parse_ply(data)
            prims = ref_model.activate(raw)
        except ref_model.ModelError as exc:
            ent.update(expect=type(exc).__name__, message=str(exc))
        else:
            ent.update(expect="ok", count=int(raw.count))
            for attr in ("means", "scales", "rotations", "opacities", "colors_dc", "sh_coeffs"):
                arrays[f"{name}/{attr}"] = np.asarray(getattr(prims, attr), dtype=np.float64)
            arrays[f"{name}/rsq"] = np.asarray(ref_render._cutoff_radius_sq(prims.opacities),
                                               dtype=np.float64)
        manifest[name] = ent
    np.savez_compressed(OUT / "arrays.npz", **arrays)
    (OUT / "cases.json").write_text(json.dumps(manifest, indent=1, sort_keys=True) + "\n")
    print(f"{len(manifest)} cases -> {OUT}")


if __name__ == "__main__":
    main()
