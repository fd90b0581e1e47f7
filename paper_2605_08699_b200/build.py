"""Build the CUDA library (libgsr.so) in-tree for sm_100a.

    python -m paper_2605_08699_b200.build [--verbose]

nvcc compiles every csrc/*.cu for ``-gencode arch=compute_100a,code=sm_100a``
with ``-fmad=false`` (the reference never contracts a*b+c into an FMA; see
DESIGN.md), ``-lineinfo`` for ncu source views, and links the CUDA runtime
statically so the .so only needs the driver on the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_build"
LIB = OUT_DIR / "libgsr.so"
INCLUDE = PKG.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
              "-cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(sources()) + list(CSRC.glob("*.cuh")) + [INCLUDE / "gsr.h"]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: Path = LIB,
          defines: tuple = ()) -> Path:
    """Compile every csrc/*.cu (in parallel) and link ``out``.  ``defines``
    (e.g. ``("GSR_TILE_H=32",)``) build a tuning variant into another file,
    loaded with GSR_LIB_PATH=<file> (A/B runs on the GPU box)."""
    out = Path(out)
    if out == LIB and not defines and not force and not _stale():
        return LIB
    obj_dir = OUT_DIR if out == LIB else out.parent / (out.stem + "_obj")
    obj_dir.mkdir(parents=True, exist_ok=True)
    host_cc = "/usr/bin/g++" if Path("/usr/bin/g++").exists() else None

    def compile_one(src):
        obj = obj_dir / (src.stem + ".o")
        cmd = [nvcc(), *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", str(INCLUDE),
               "-c", str(src), "-o", str(obj)]
        if host_cc:
            cmd[1:1] = ["-ccbin", host_cc]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return str(obj)

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    LIB_ = out
    tmp = LIB_.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    if host_cc:
        cmd[1:1] = ["-ccbin", host_cc]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_)
    for o in objs:
        Path(o).unlink(missing_ok=True)
    return LIB_


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=str(LIB))
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=True, verbose=a.verbose, out=Path(a.out), defines=tuple(a.defines)))
