"""PLY load: oracle + C-ABI header parse on the CPU,
the device loader (gsr_scene_create_ply) on the GPU.

Golden vectors: tests/golden/ply (made by the reference itself,
tests/golden/make_ply_golden.py).  Bar: bit-exact arrays (f64 bit patterns),
identical exception classes and messages.
"""

from __future__ import annotations

import ctypes
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle
from paper_2605_08699_b200 import _lib

GOLD = Path(__file__).resolve().parent / "golden" / "ply"
CASES = json.loads((GOLD / "cases.json").read_text())
ATTRS = ("means", "scales", "rotations", "opacities", "colors_dc", "sh_coeffs", "rsq")


def _arrays():
    with np.load(GOLD / "arrays.npz") as z:
        return {k: z[k] for k in z.files}


def _data(name):
    return (GOLD / CASES[name]["file"]).read_bytes()


def _same_bits(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


# ----------------------------------------------------------------- CPU -----

def test_oracle_matches_reference_golden():
    arrays = _arrays()
    for name, ent in CASES.items():
        data = _data(name)
        if ent["expect"] == "ok":
            got = oracle.ply_load(data)
            for a in ATTRS:
                assert _same_bits(got[a], arrays[f"{name}/{a}"]), (name, a)
        else:
            with pytest.raises(oracle.PlyError) as ei:
                oracle.ply_load(data)
            assert (ei.value.kind, str(ei.value)) == (ent["expect"], ent["message"]), name


def _svml_dispatch() -> bool:
    feats = np._core._multiarray_umath.__cpu_features__
    return bool(feats.get("AVX512_SKX"))


@pytest.mark.skipif(not _svml_dispatch(), reason="numpy does not dispatch to SVML on this CPU")
def test_oracle_libm_restatements_vs_numpy():
    """The restated SVML exp/log and glibc exp equal numpy / scipy / libm."""
    from scipy.special import expit
    rng = np.random.default_rng(11)
    x = np.concatenate([rng.uniform(-60, 60, 300_000).astype(np.float32).astype(np.float64),
                        rng.uniform(-700, 700, 50_000)])
    assert _same_bits(oracle.np_exp(x), np.exp(x))
    lg = rng.uniform(-60, 60, 300_000).astype(np.float32).astype(np.float64)
    assert _same_bits(1.0 / (1.0 + oracle.glibc_exp(-lg)), expit(lg))
    e = np.concatenate([rng.uniform(-745, 709.7, 20_000), [-745.2, -744.0, -709.5, 600.0, 709.7]])
    assert _same_bits(oracle.glibc_exp(e), np.array([math.exp(v) for v in e]))
    v = np.concatenate([rng.uniform(1.0, 8160.0, 300_000),
                        np.exp(rng.uniform(-700, 700, 50_000))])
    assert _same_bits(oracle.np_log(v), np.log(v))


def test_c_abi_header_parse_matches_reference():
    """gsr_ply_parse_header (host only) vs the reference's header errors."""
    lib = _lib.load()
    header_errors = {"MalformedHeader", "MissingProperty", "TruncatedBody"}
    codes = {"MalformedHeader": _lib.GSR_E_PLY_HEADER, "MissingProperty": _lib.GSR_E_PLY_PROPERTY,
             "TruncatedBody": _lib.GSR_E_PLY_TRUNCATED}
    for name, ent in CASES.items():
        data = _data(name)
        info = _lib.GsrPlyInfo()
        rc = lib.gsr_ply_parse_header(data, len(data), ctypes.byref(info))
        if ent["expect"] in header_errors:
            assert rc == codes[ent["expect"]], name
            assert _lib.last_error() == ent["message"], name
            continue
        assert rc == 0, (name, _lib.last_error())
        props, count, off = oracle.ply_header(data)
        assert (info.count, info.body_offset, info.n_props) == (count, off, len(props)), name
        col = {p: i for i, p in enumerate(props)}
        names = oracle.PLY_REQUIRED + oracle.PLY_REST
        assert [info.col[i] for i in range(59)] == [col.get(n, -1) for n in names], name
        assert bool(info.has_rest) == all(n in col for n in oracle.PLY_REST), name


def test_python_header_api_raises_reference_classes():
    from paper_2605_08699_b200 import model
    hdr = model.parse_ply_header(_data("random_rest_33"))
    assert hdr.count == 33 and hdr.has_rest and hdr.n_props == 59
    for name, cls in (("err_ascii_format", model.MalformedHeader),
                      ("err_missing_opacity", model.MissingProperty),
                      ("err_truncated", model.TruncatedBody)):
        with pytest.raises(cls, match="^" + _re(CASES[name]["message"]) + "$"):
            model.parse_ply_header(_data(name))
    assert issubclass(model.NonFiniteAttribute, model.ModelError)


def _re(s):
    import re
    return re.escape(s)


# ----------------------------------------------------------------- GPU -----

def _read(prims, which):
    lib = _lib.load()
    arr = np.empty(prims.count, dtype=np.float64)
    _lib.check(lib.gsr_scene_read(prims.scene.handle, which, _lib.ptr(arr)))
    return arr


@pytest.mark.gpu
def test_gpu_load_ply_golden_bit_exact():
    from paper_2605_08699_b200 import model
    arrays = _arrays()
    errs = {"MalformedHeader": model.MalformedHeader, "MissingProperty": model.MissingProperty,
            "TruncatedBody": model.TruncatedBody, "NonFiniteAttribute": model.NonFiniteAttribute}
    for name, ent in CASES.items():
        data = _data(name)
        if ent["expect"] != "ok":
            with pytest.raises(errs[ent["expect"]]) as ei:
                model.load_ply(data)
            assert str(ei.value) == ent["message"], name
            continue
        prims = model.load_ply(data)
        assert prims.count == ent["count"]
        for a in ATTRS[:-1]:
            assert _same_bits(getattr(prims, a), arrays[f"{name}/{a}"]), (name, a)
        assert _same_bits(_read(prims, 6), arrays[f"{name}/rsq"]), (name, "rsq")


@pytest.mark.gpu
def test_gpu_load_ply_large_vs_oracle_and_render():
    """200k Gaussians, wide attribute ranges: every array bit-exact vs the
    oracle; frames from the PLY scene equal frames from the host-built scene."""
    from paper_2605_08699_b200 import model, render
    from paper_2605_08699_b200.camera import Intrinsics, pose_from_degrees
    from paper_2605_08699_b200.synth import make_synthetic_set, scale_range_for, serialize_ply
    n = 200_000
    raw = make_synthetic_set(count=n, seed=3, scale_range=scale_range_for(n), include_rest=True)
    rng = np.random.default_rng(5)
    raw.opacity_logits[: n // 10] = rng.uniform(-60, 60, n // 10)   # expit tails
    raw.log_scales[: n // 50] = rng.uniform(-40, 8, (n // 50, 3))   # exp range
    data = serialize_ply(raw, include_rest=True)
    stats = {}
    prims = model.load_ply(data, stats=stats)
    want = oracle.ply_load(data)
    for a in ATTRS[:-1]:
        assert _same_bits(getattr(prims, a), want[a]), a
    assert _same_bits(_read(prims, 6), want["rsq"])
    assert stats["kernel_ms"] > 0 and stats["body_bytes"] == len(data) - data.find(b"end_header\n") - 11
    host = prims.materialize()
    intr = Intrinsics(fx=500.0, fy=500.0, cx=320.0, cy=240.0, width=640, height=480)
    for az in (0.0, 40.0):
        pose = pose_from_degrees(az, 10.0)
        a = render.render_u8(prims, pose, intr, sh_degree=3)
        b = render.render_u8(host, pose, intr, sh_degree=3)
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_gpu_load_ply_evict_keeps_arrays():
    from paper_2605_08699_b200 import model, render
    prims = model.load_ply(_data("random_rest_33"))
    sc = prims.scene
    assert render.device_scene(prims, prims.device) is sc  # no upload
    render.evict(prims)
    assert sc.closed
    arrays = _arrays()
    assert _same_bits(prims.scales, arrays["random_rest_33/scales"])
    assert render.device_scene(prims, prims.device) is not sc  # re-uploaded from host arrays


@pytest.mark.gpu
def test_gpu_load_ply_wide_rows_and_column_order():
    """Rows too wide for shared-memory staging (> 384 properties: the direct
    kernel variant), properties in a shuffled order with extras: bit-exact
    vs the oracle."""
    from paper_2605_08699_b200 import model
    rng = np.random.default_rng(9)
    names = list(oracle.PLY_REQUIRED + oracle.PLY_REST) + [f"extra_{i}" for i in range(360)]
    rng.shuffle(names)
    n = 3000
    table = rng.normal(size=(n, len(names))).astype("<f4")
    col = {p: i for i, p in enumerate(names)}
    table[:, col["opacity"]] *= 6.0
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    header += [f"property float {p}" for p in names] + ["end_header"]
    data = ("\n".join(header) + "\n").encode("ascii") + table.tobytes()
    prims = model.load_ply(data)
    want = oracle.ply_load(data)
    for a in ATTRS[:-1]:
        assert _same_bits(getattr(prims, a), want[a]), a
    assert _same_bits(_read(prims, 6), want["rsq"])
