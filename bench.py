#!/usr/bin/env python
"""Benchmark of the per-pose render path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gsr|reference]
                    [--workload config3|config2|config4|config1|config5|config5w]
                    [--dry-run]

metric: 1080p frames/s at 3M Gaussians (config 3's 1080p rung: synthetic
3M-Gaussian scene, SH degree 3, 1920x1080), plus p50/p99 render latency.
A step = one frame of one client session at the next pose of its seeded
EyeNavGS-style trace.  Sessions are independent (server.py:1-7), so with N
GPUs (one process per GPU; `--gpus N` re-launches itself under
torch.distributed.run when WORLD_SIZE is not set) rank r serves its own
session on its own GPU: weak scaling, no data-path collective (the only NCCL
calls are the barrier and the max-over-ranks timing reduction).
--workload config5 / config5w: BASELINE config 5 (64 sessions over 14 scene
sizes, strong scaling / 8 sessions per GPU, weak scaling), all-1080p and
ABR-mixed (tests/golden/abr_sequence.json) with per-frame p50/p99.
--dry-run: no CUDA (gloo): the launcher, sharding and max-over-ranks path only.

value      device throughput with --streams S (default 4) frames in flight:
           K frames enqueued round-robin on S contexts (CUDA streams), the
           scene resident in HBM; CUDA events (start on stream 0, which the
           others wait on; end on every stream), max over ranks; frames of
           all ranks / that time.  value_single_stream: the same with S = 1.
e2e        the public serving API (RenderPipeline(depth=S).submit), wall
           clock over K frames; every step uploads its camera (160 B of kernel
           parameters) and copies its u8 frame (6.2 MB) to pinned host memory
           inside the timed region.  e2e_single: render_u8 one call at a time.
latency_ms one render_u8 call at a time (wall) and its device time (events).
roofline   the dominant kernel's algorithmic bytes (or FP32 ops) per launch /
           its mean event-timed duration, against MEASURED_PEAKS.json.
cpu_baseline  the reference's own render_framebuffer + framebuffer_to_u8
           (numba, all host cores; the unmodified package installed into
           baseline/_ref) on the same scene and poses, bounded to ~20 s after
           its JIT warm-up, rank 0 at N=1; the C oracle port (OpenMP) is timed
           beside it as cpu_port.  Without baseline/_ref the port is the
           baseline (kind "port").
--impl reference  the reference arm: the same reference render on the host
           cores (or the port, see above), bounded to a few minutes.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

METRIC = "1080p frames/sec/GPU and p50/p99 render ms at 3M Gaussians"
METRIC5 = "box fps at 1/2/4/8 GPUs: config 5, 64 sessions x 14 scene sizes, 1080p"

WORKLOADS = {
    "config1": dict(n=10_000, sh=0, w=256, h=256, scale=(0.02, 0.12),
                    desc="config1: synthetic 10k-Gaussian scene, SH0, 256x256"),
    "config2": dict(n=500_000, sh=3, w=1280, h=720, scale=None,
                    desc="config2: synthetic 500k-Gaussian scene, SH3, 1280x720, pose trace"),
    "config3": dict(n=3_000_000, sh=3, w=1920, h=1080, scale=None,
                    desc="config3: synthetic 3M-Gaussian scene, SH3, 1920x1080 rung, pose trace"),
    "config4": dict(n=6_000_000, sh=3, w=1920, h=1080, scale=None,
                    desc="config4: synthetic 6M-Gaussian scene, SH3, 1920x1080, pose trace"),
    "config5": dict(config5=True, weak=False, n=None, sh=3, w=1920, h=1080,
                    desc="config5: 64 pose-trace sessions over 14 scene sizes (250k..6M "
                         "Gaussians, SH3, 1920x1080), session i -> GPU i mod N"),
    "config5w": dict(config5=True, weak=True, n=None, sh=3, w=1920, h=1080,
                     desc="config5w: 8 pose-trace sessions per GPU over the 14 scene sizes "
                          "(SH3, 1920x1080), session i -> GPU i mod N (weak scaling)"),
}

NVML_REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
                0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
                0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
                0x100: "display_clock_setting"}


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    def __init__(self, device: int, period_s: float = 0.01):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in NVML_REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


class Dist:
    """One process per GPU (torchrun env).  NCCL only for the start barrier
    and the max-over-ranks timing reduction (no data-path collective);
    gloo on CPU for --dry-run."""

    def __init__(self, dry: bool = False):
        self.rank, self.local_rank, self.world = dist_env()
        self.dry = dry
        if not dry:
            import torch
            torch.cuda.set_device(self.local_rank)
        if self.world > 1:
            import torch
            import torch.distributed as dist
            if dry:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local_rank))

    def barrier(self):
        import torch
        if self.world > 1:
            torch.distributed.barrier()
        if not self.dry:
            torch.cuda.synchronize()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.dry else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.dry else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
        return float(t.item())

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        import torch
        out = [None] * self.world
        torch.distributed.all_gather_object(out, obj)
        return out

    def close(self):
        if self.world > 1:
            import torch
            torch.distributed.barrier()
            torch.distributed.destroy_process_group()


def relaunch(nproc: int, argv) -> int:
    """`--gpus N` without a torchrun environment: run this script under
    torch.distributed.run with N processes on this node (127.0.0.1)."""
    import socket
    import subprocess
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def build_scene(wl, seed=7):
    from paper_2605_08699_b200.synth import synthetic_scene
    return synthetic_scene(wl["n"], seed=seed, sh_degree=wl["sh"], scale_range=wl["scale"])


def intrinsics(wl):
    from paper_2605_08699_b200.camera import Intrinsics, scale_intrinsics
    from paper_2605_08699_b200.synth import base_intrinsics_1080p
    if wl["w"] == wl["h"]:
        f = (wl["w"] / 2) / np.tan(np.radians(30.0))
        return Intrinsics(fx=f, fy=f, cx=wl["w"] / 2, cy=wl["h"] / 2, width=wl["w"],
                          height=wl["h"])
    return scale_intrinsics(base_intrinsics_1080p(), wl["w"], wl["h"])


def poses_for(rank, count):
    from paper_2605_08699_b200.camera import pose_from_degrees
    from paper_2605_08699_b200.synth import pose_trace
    return [pose_from_degrees(p.azimuth_deg, p.elevation_deg, p.translation)
            for p in pose_trace(count, seed=rank)]


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def _parity(u8, gpu_u8, psnr):
    d = np.abs(u8.astype(np.int16) - gpu_u8.astype(np.int16))
    return {"frame0_u8_max_abs_diff": int(d.max()), "frame0_psnr_db": psnr(u8, gpu_u8),
            "frame0_bit_exact": bool(np.array_equal(u8, gpu_u8))}


def host_cpu() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_port(prims, poses, intr, sh, budget_s, gpu_u8=None):
    """The oracle port (oracle/oracle.c, OpenMP) on the host cores, bounded."""
    from oracle import oracle as orc
    orc.build()
    cores = orc.num_threads()
    times, parity = [], None
    t_all = time.perf_counter()
    for i, pose in enumerate(poses):
        rot, w2c = orc.world_to_camera(pose.azimuth, pose.elevation, pose.translation)
        t0 = time.perf_counter()
        fr = orc.render(prims.means, prims.scales, prims.rotations, prims.opacities,
                        prims.colors_dc, prims.sh_coeffs, w2c, rot, intr.fx, intr.fy, intr.cx,
                        intr.cy, intr.width, intr.height, (0.0, 0.0, 0.0), sh)
        times.append(time.perf_counter() - t0)
        if i == 0 and gpu_u8 is not None:
            parity = _parity(fr.u8, gpu_u8, orc.psnr)
        if time.perf_counter() - t_all > budget_s:
            break
    fps = len(times) / sum(times)
    return {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port",
            "sample": f"{len(times)} frame(s) of the same workload, oracle/oracle.c "
                      f"(OpenMP, {cores} threads), {sum(times):.1f} s",
            "ms_per_frame": 1000.0 * sum(times) / len(times), "host_cpu": host_cpu()}, parity


REF_DIR = ROOT / "baseline" / "_ref"


def reference_modules():
    """The unmodified reference package (pip-installed from /root/reference/pkg
    into baseline/_ref): (render, camera, model, numba)
    with numba on every host core, or None when it is not shipped."""
    if not (REF_DIR / "splatstream" / "render.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gsr_bench_numba_cache")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import numba
        import splatstream.camera as C
        import splatstream.model as M
        import splatstream.render as R
    except Exception as exc:  # noqa: BLE001
        print(f"bench: reference package not importable ({exc}); using the port",
              file=sys.stderr)
        return None
    numba.set_num_threads(numba.config.NUMBA_NUM_THREADS)
    return R, C, M, numba


def cpu_reference(prims, poses, intr, sh, budget_s, gpu_u8=None):
    """The reference's own render_framebuffer + framebuffer_to_u8 (render.py:
    484-485, 516-524) on all host cores, after one JIT warm-up
    frame (test_acceptance.py:155), bounded to ~budget_s.  None without
    baseline/_ref."""
    mods = reference_modules()
    if mods is None:
        return None, None
    R, C, M, numba = mods
    ap = M.ActivatedPrimitives(means=prims.means, scales=prims.scales,
                               rotations=prims.rotations, opacities=prims.opacities,
                               colors_dc=prims.colors_dc, sh_coeffs=prims.sh_coeffs)
    ri = C.Intrinsics(fx=intr.fx, fy=intr.fy, cx=intr.cx, cy=intr.cy, width=intr.width,
                      height=intr.height)

    def frame(p):
        pose = C.CameraPose(p.azimuth, p.elevation, tuple(p.translation))
        return R.framebuffer_to_u8(R.render_framebuffer(ap, pose, ri, (0.0, 0.0, 0.0), sh))

    t0 = time.perf_counter()
    frame(poses[0])
    jit_s = time.perf_counter() - t0
    times, parity = [], None
    for i, p in enumerate(poses):
        t0 = time.perf_counter()
        u8 = frame(p)
        times.append(time.perf_counter() - t0)
        if i == 0 and gpu_u8 is not None:
            from oracle import oracle as orc
            parity = _parity(u8, gpu_u8, orc.psnr)
        if sum(times) > budget_s:
            break
    cores = int(numba.get_num_threads())
    return {"value": len(times) / sum(times), "unit": "frames/s", "cores": cores,
            "kind": "reference",
            "sample": f"{len(times)} frame(s) of the same workload through the unmodified "
                      f"reference's render_framebuffer + framebuffer_to_u8 (numba "
                      f"{numba.__version__}, {cores} threads, os.cpu_count() {os.cpu_count()}), "
                      f"{sum(times):.1f} s after a {jit_s:.1f} s JIT warm-up frame",
            "ms_per_frame": 1000.0 * sum(times) / len(times), "host_cpu": host_cpu()}, parity


def run_reference(args, wl):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    if wl.get("config5"):
        return run_reference_config5(args, wl)
    prims = build_scene(wl)
    intr = intrinsics(wl)
    poses = poses_for(0, args.warmup + args.steps)
    budget = float(os.environ.get("BENCH_REF_BUDGET_S", "150"))
    base, _ = cpu_reference(prims, poses[args.warmup:], intr, wl["sh"], budget)
    if base is None:
        from oracle import oracle as orc
        orc.build()
        pose = poses[0]  # warm-up (page-in, OpenMP pool)
        rot, w2c = orc.world_to_camera(pose.azimuth, pose.elevation, pose.translation)
        orc.render(prims.means, prims.scales, prims.rotations, prims.opacities, prims.colors_dc,
                   prims.sh_coeffs, w2c, rot, intr.fx, intr.fy, intr.cx, intr.cy, intr.width,
                   intr.height, (0.0, 0.0, 0.0), wl["sh"])
        base, _ = cpu_port(prims, poses[args.warmup:], intr, wl["sh"], budget)
    line = {
        "metric": METRIC,
        "value": base["value"], "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": base["ms_per_frame"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": wl["desc"], "gaussians": wl["n"], "sh_degree": wl["sh"],
                   "width": wl["w"], "height": wl["h"],
                   "parallelism": f"session-sharded x{world} (no collective)"},
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# dram__bytes_read.sum + dram__bytes_write.sum per launch of each kernel, from
# the committed `ncu --set full` capture (tools/ncu_traffic.py writes it)
TRAFFIC = {}
_tp = ROOT / "profiles" / "ncu_traffic_config3.json"
if _tp.exists():
    TRAFFIC = json.loads(_tp.read_text())


def load_simt_peaks():
    """FP32/FP64/smem peaks measured by tools/peaks.cu on a B200 of this
    pool (profiles/measured_simt_peaks.json), else the nominal figures."""
    p = ROOT / "profiles" / "measured_simt_peaks.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured (tools/peaks.cu)"
        return d
    # nominal: 148 SMs x 128 FP32 lanes x 1.965 GHz (no FMA), FP64 at half rate
    return {"fp32_tops": 37.2, "fp64_tops": 18.6, "source": "nominal"}


def kernel_work(name, wl, c):
    """Algorithmic units of a kernel over ONE frame, all its launches
    (DESIGN.md section 4): (bytes, fp32 ops).  KA / KB: splats sorted by the
    first / second depth slice (K, 0 for a one-pass frame)."""
    n, k, d, p = wl["n"], c["K"], c["D"], c["P"]
    ks = c["KA"] + c["KB"]  # splats ranked, coloured and binned over the slices
    sh_bytes = 12 * (wl["sh"] + 1) ** 2 if wl["sh"] else 12
    px = wl["w"] * wl["h"]
    sliced = c["KB"] > 0 or c["KA"] < k
    table = {
        # mean/scale/rotation/rsq f64 + opacity f32 in; key for all N; record of kept
        # (+ the 8 B item box of each kept splat when the frame is sliced)
        "preprocess_geo": (n * 92 + n * 8 + k * 32 + (k * 8 if sliced else 0), 0),
        # order + mean f64 + SH row (or DC) of each ranked splat in; colour out
        "color_ranked": (ks * (4 + 24 + sh_bytes + 16), 0),
        # one pass: f64 depth key of all N in, span key out; slice A: f64 key
        # of all N in, the slice's (span key, index) pairs out; slice B: its
        # appended span keys in
        "radix32_hist": ((n * 8 + c["KA"] * 8 + c["KB"] * 4) if sliced else n * 12, 0),
        "radix32_pass": (3 * ks * 16, 0),  # per pass: key + index read and written
        "depth_fixup": (ks * 4, 0),
        # depth key of all N; item box of each kept splat behind the front slice
        "slice_b_filter": (n * 8 + max(k - c["KA"], 0) * 8, 0),
        # order + geometry gathered, 32 B record written
        "bin_gather": (ks * (4 + 32 + 32), 0),
        # records in, pairs out; 20 FP32 ops per exact row interval (render.py:383-397)
        # evaluated (pairs whose span the f64 band bound settles need none)
        "bin_pairs": (ks * 32 + p * 8, 20 * c["Rp"]),
        "seg_count": (p * 8, 0),
        "seg_place": (p * 8 + d * 4, 0),
        # lists + each record and colour once + u8 frame; 20 FP32 ops per
        # composited evaluation (render.py:405-421) and per row interval (383-397)
        "blend": (d * 4 + ks * 48 + 3 * px, 20 * (c["E"] + c["Rb"])),
    }
    return table.get(name, (0, 0))


BOUND = {"bin_pairs": "fp32", "blend": "fp32"}


def kernel_profile(lib, ctx, sc, cams, sh, frames, wl, peaks, simt):
    """Per-kernel device times of the serving kernels: a CUDA event is recorded
    on the render stream after every launch (gsr_ctx_set_kernel_timing,
    GSR_TIMING_EVENTS); mean over `frames` frames.  The blend's work counters
    (E, Rb) need its counting variant, which is slower, so they come from
    separate frames of the same poses (GSR_TIMING_COUNTERS)."""
    from paper_2605_08699_b200 import _lib
    from paper_2605_08699_b200.render import _bg
    names = ctypes.create_string_buffer(64 * 48)
    ms = (ctypes.c_float * 64)()
    cnt = ctypes.c_int(0)
    agg, launches, counters = {}, {}, []
    st = _lib.GsrStats()
    try:
        _lib.check(lib.gsr_ctx_set_kernel_timing(ctx.handle, 1))  # events only
        for cam in cams[:frames]:
            _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(cam), _bg((0, 0, 0)), sh,
                                      1, None, None, None, ctypes.byref(st)))
            _lib.check(lib.gsr_ctx_kernel_times(ctx.handle, 64, names, ms, ctypes.byref(cnt)))
            for i in range(cnt.value):
                nm = names.raw[48 * i:48 * i + 48].split(b"\0", 1)[0].decode()
                agg[nm] = agg.get(nm, 0.0) + ms[i]
                launches[nm] = launches.get(nm, 0) + 1
        _lib.check(lib.gsr_ctx_set_kernel_timing(ctx.handle, 2))  # counters only
        for cam in cams[:frames]:
            _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(cam), _bg((0, 0, 0)), sh,
                                      1, None, None, None, ctypes.byref(st)))
            raw = (ctypes.c_uint64 * 15)()
            _lib.check(lib.gsr_debug_frame_counters(ctx.handle, raw, 15))
            counters.append({"K": raw[0], "D": raw[1], "P": raw[2], "E": raw[3], "Rb": raw[4],
                             "Rp": raw[5], "KA": raw[13], "KB": raw[14]})
    finally:
        lib.gsr_ctx_set_kernel_timing(ctx.handle, 0)
    nf = max(1, len(counters))  # same frames for both passes
    mean_c = {key: float(np.mean([c[key] for c in counters])) for key in counters[0]}
    hbm = float(peaks["hbm_gbs"])
    fp32 = float(simt["fp32_tops"])
    out = {}
    if "blend_a" in agg:  # the two slices' blends, as one kernel for the roofline
        agg["blend"] = agg.get("blend_a", 0.0) + agg.get("blend_b", 0.0)
        launches["blend"] = launches.get("blend_a", 0) + launches.get("blend_b", 0)
    for nm, tot in agg.items():
        per_frame = tot / nf
        nl = launches[nm] / nf
        b, f = kernel_work(nm, wl, mean_c)  # per frame
        e = {"ms_per_frame": round(per_frame, 4), "launches_per_frame": nl,
             "bound": BOUND.get(nm, "hbm") if f or nm not in BOUND else "hbm"}
        if b and per_frame > 0:
            gbs = b / (per_frame * 1e-3) / 1e9
            e.update(alg_bytes=int(b), achieved_gbs=round(gbs, 1), frac_hbm=round(gbs / hbm, 4))
        if f and per_frame > 0:
            tf = f / (per_frame * 1e-3) / 1e12
            e.update(alg_fp32_ops=int(f), achieved_tflops=round(tf, 2),
                     frac_fp32=round(tf / fp32, 4))
        out[nm] = e
    return out, mean_c


def bench_scene_load(wl, peaks, peak_kind, with_cpu=True, reps=3):
    """load_ply of the workload's scene as a binary PLY (model.py:169-252, 354)."""
    from paper_2605_08699_b200 import model
    from paper_2605_08699_b200.synth import make_synthetic_set, scale_range_for, serialize_ply
    n = wl["n"]
    raw = make_synthetic_set(count=n, seed=7, scale_range=scale_range_for(n),
                             include_rest=wl["sh"] > 0)
    data = serialize_ply(raw, include_rest=wl["sh"] > 0)
    runs = []
    for _ in range(reps + 1):
        st = {}
        t0 = time.perf_counter()
        p = model.load_ply(data, stats=st)
        st["wall_ms"] = (time.perf_counter() - t0) * 1000.0
        p.scene.close()
        runs.append(st)
    best = min(runs[1:], key=lambda r: r["wall_ms"])
    row = best["body_bytes"] // max(n, 1)
    alg = n * (row + 304)  # vertex table read + activated planes written (K10)
    out = {"gaussians": n, "ply_bytes": len(data), "ms_wall": best["wall_ms"],
           "ms_native": best["total_ms"], "ms_h2d": best["h2d_ms"], "ms_kernel": best["kernel_ms"],
           "h2d_gbs": best["body_bytes"] / best["h2d_ms"] / 1e6,
           "kernel_roofline": {"bound": "hbm", "achieved": alg / best["kernel_ms"] / 1e6,
                               "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                               "frac": alg / best["kernel_ms"] / 1e6 / float(peaks["hbm_gbs"]),
                               "alg_bytes": alg, "peak_source": peak_kind},
           "api": "model.load_ply(bytes) -> DeviceActivatedPrimitives (bit-exact arrays)"}
    if with_cpu:
        from oracle import oracle
        m = min(n, 300_000)
        sub = make_synthetic_set(count=m, seed=7, scale_range=scale_range_for(n),
                                 include_rest=wl["sh"] > 0)
        sdata = serialize_ply(sub, include_rest=wl["sh"] > 0)
        t0 = time.perf_counter()
        oracle.ply_load(sdata)
        cpu_s = time.perf_counter() - t0
        out["cpu_baseline"] = {"ms_for_full_scene": cpu_s * 1000.0 * n / m, "cores": 1,
                               "kind": "port",
                               "sample": f"parse_ply + activate + rsq of {m} Gaussians "
                                         "(oracle.ply_load, numpy), scaled to the scene"}
    return out


def run_gsr(args, wl):
    import torch
    d = Dist()
    rank, local_rank, world = d.rank, d.local_rank, d.world
    import paper_2605_08699_b200 as g
    from paper_2605_08699_b200 import _lib
    from paper_2605_08699_b200.render import _bg, device_scene, make_camera
    g.set_device(local_rank)

    prims = build_scene(wl)
    intr = intrinsics(wl)
    K, W = args.steps, args.warmup
    n_lat = max(K, args.latency_calls)
    poses = poses_for(rank, W + max(K, n_lat))
    sc = device_scene(prims, local_rank)
    ctx = _lib.context(local_rank)
    lib = ctx.lib
    cams = [make_camera(p, intr) for p in poses]
    bg = _bg((0.0, 0.0, 0.0))

    # warm-up: capacities, page-in, JIT of nothing (all AOT)
    st = _lib.GsrStats()
    for i in range(W):
        _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(cams[i]), bg, wl["sh"], 1,
                                  None, None, None, ctypes.byref(st)))

    # ---- device throughput: K frames back to back on the render stream ----
    stream = torch.cuda.ExternalStream(lib.gsr_ctx_stream(ctx.handle))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    d.barrier()
    with ClockSampler(local_rank) as clocks:
        ev0.record(stream)
        for i in range(W, W + K):
            _lib.check(lib.gsr_render_async(ctx.handle, sc.handle, ctypes.byref(cams[i]), bg,
                                            wl["sh"], 1))
        ev1.record(stream)
        _lib.check(lib.gsr_ctx_finish(ctx.handle, None, ctypes.byref(st)))
        torch.cuda.synchronize()
    launches_single = int(st.kernel_launches)
    # frames that would need a re-render (buffer growth / 64-bit depth sort);
    # the throughput loops do not complete every frame, so they are counted
    # on the device and reported (0 expected: capacities come from warm-up)
    retry = {"overflow_frames": int(st.overflow_frames),
             "long_run_frames": int(st.long_run_frames)}
    dev_ms = d.max(ev0.elapsed_time(ev1))
    value_single = world * K / (dev_ms / 1000.0)

    # ---- pipelined device throughput: frames alternate over S contexts
    # (streams), as a server with S requests in flight runs them ----
    S = max(1, args.streams)
    ctxs = [ctx] + [_lib.Context(local_rank) for _ in range(S - 1)]
    for c in ctxs[1:]:
        for i in range(W):
            _lib.check(lib.gsr_render(c.handle, sc.handle, ctypes.byref(cams[i]), bg, wl["sh"], 1,
                                      None, None, None, ctypes.byref(st)))
    streams = [torch.cuda.ExternalStream(lib.gsr_ctx_stream(c.handle)) for c in ctxs]
    ends = [torch.cuda.Event(enable_timing=True) for _ in ctxs]
    launches = 0
    d.barrier()
    with ClockSampler(local_rank) as clocks:
        ev0.record(streams[0])
        for sm in streams[1:]:
            sm.wait_event(ev0)
        for i in range(W, W + K):
            c = ctxs[(i - W) % S]
            _lib.check(lib.gsr_render_async(c.handle, sc.handle, ctypes.byref(cams[i]), bg,
                                            wl["sh"], 1))
        for e, sm in zip(ends, streams):
            e.record(sm)
        for c in ctxs:
            _lib.check(lib.gsr_ctx_finish(c.handle, None, ctypes.byref(st)))
            launches += int(st.kernel_launches)
            retry["overflow_frames"] += int(st.overflow_frames)
            retry["long_run_frames"] += int(st.long_run_frames)
        torch.cuda.synchronize()
    pipe_ms = d.max(max(ev0.elapsed_time(e) for e in ends))
    value = world * K / (pipe_ms / 1000.0)
    launches = int(d.sum(launches))  # kernels all ranks ran in the timed region

    # ---- per-call latency (>= --latency-calls calls, independent of --steps)
    # and e2e through the public API (pinned host frame) ----
    out = ctx.pinned("bench_frame", (intr.height, intr.width, 3), np.uint8)
    lat, dev_lat = [], []
    rs = g.RenderStats()
    d.barrier()
    t_e2e = time.perf_counter()
    for i in range(W, W + K):
        g.render_u8(prims, poses[i], intr, sh_degree=wl["sh"], stats=rs, out=out)
    e2e_single_s = d.max(time.perf_counter() - t_e2e)
    for i in range(W, W + n_lat):
        t0 = time.perf_counter()
        g.render_u8(prims, poses[i], intr, sh_degree=wl["sh"], stats=rs, out=out)
        lat.append((time.perf_counter() - t0) * 1000.0)
        dev_lat.append(rs.device_ms)
    # pipelined e2e: RenderPipeline keeps S frames in flight; every step still
    # uploads its camera and copies its u8 frame to pinned host memory
    pipe = g.RenderPipeline(intr, sh_degree=wl["sh"], depth=S, device=local_rank)
    for i in range(max(W, len(pipe.ctxs))):  # every context captures its graph here
        pipe.submit(prims, poses[i % len(poses)])
    pipe.drain()
    checksum = 0
    d.barrier()
    t_e2e = time.perf_counter()
    for i in range(W, W + K):
        r = pipe.submit(prims, poses[i])
        if r is not None:
            checksum += int(r[1][0, 0, 0])
    for _, f in pipe.drain():
        checksum += int(f[0, 0, 0])
    e2e_s = d.max(time.perf_counter() - t_e2e)
    pipe.close()
    # per-stage device timings (event pairs inside the ABI, GSR_TIMING_STAGES:
    # four event nodes in the frame graph, off while serving), separate pass
    _lib.check(lib.gsr_ctx_set_kernel_timing(ctx.handle, 4))
    stage_stats = []
    for i in range(W, W + min(K, 50)):
        _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(cams[i]), bg, wl["sh"], 1,
                                  None, None, None, ctypes.byref(st)))
        stage_stats.append(st.as_dict())
    stages = {k[3:]: round(float(np.mean([x[k] for x in stage_stats])), 4)
              for k in ["ms_preprocess", "ms_depth_sort", "ms_binning", "ms_blend", "ms_slice_b"]}
    peaks, peak_kind = load_peaks()
    simt = load_simt_peaks()
    kernels, counters = kernel_profile(lib, ctx, sc, cams[W:], wl["sh"], min(K, 30), wl, peaks,
                                       simt)
    dom = max((x for x in kernels if x not in ("blend_a", "blend_b")),
              key=lambda x: kernels[x]["ms_per_frame"])
    dk = kernels[dom]
    if dk["bound"] == "fp32":
        roof = {"bound": "fp32", "kernel": dom, "achieved": dk["achieved_tflops"],
                "peak": float(simt["fp32_tops"]), "unit": "TFLOP/s", "frac": dk["frac_fp32"],
                "peak_source": simt["source"]}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": dk["achieved_gbs"],
                "peak": float(peaks["hbm_gbs"]), "unit": "GB/s", "frac": dk["frac_hbm"],
                "peak_source": peak_kind}
    roof["traffic"] = TRAFFIC.get(dom)
    roof["alg_per_frame"] = dk.get("alg_fp32_ops") or dk.get("alg_bytes")
    roof["ms_per_frame"] = dk["ms_per_frame"]
    roof["launches_per_frame"] = dk["launches_per_frame"]
    roof["timed_variant"] = "serving (no work counters); counters from separate frames"
    if roof["bound"] == "fp32":
        # the contract's two bounds are hbm / tensor; this kernel is bound by
        # neither (FP32/FP64 issue of the exact compositing) -- the HBM view
        # of the same kernel is reported beside it
        roof["note"] = ("issue-bound exact compositing (glibc expf in f64, reference op order): "
                        "neither HBM nor tensor cores; see roofline_hbm and DESIGN.md section 8")
    roofline_hbm = {"bound": "hbm", "kernel": dom, "achieved": dk.get("achieved_gbs"),
                    "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                    "frac": dk.get("frac_hbm"), "traffic": TRAFFIC.get(dom),
                    "alg_per_frame": dk.get("alg_bytes"), "peak_source": peak_kind}

    # the north-star binning design on 16x16 tiles ((tile|rank) keys, radix
    # sort, ranges: contract.cu), timed on the same frames beside the render
    # path's sort-free 32x16 binning
    contract = contract_profile(ctx, lib, sc, cams[W:], wl, bg, min(K, 10))

    # config 3's full ABR ladder: base + 3 rungs rendered, upsampled, SSIM-scored
    ladder = None
    if wl["w"] == 1920 and wl["h"] == 1080 and not args.no_ladder:
        from paper_2605_08699_b200.metrics import ladder_ssim
        from paper_2605_08699_b200.synth import ladder_1080p
        rungs = [(r["width"], r["height"]) for r in ladder_1080p()[1:]]
        ladder_ssim(prims, poses[W], intr, rungs, sh_degree=wl["sh"])  # warm
        lt, ss = [], []
        for i in range(W, W + min(K, 10)):
            t0 = time.perf_counter()
            ss, _ = ladder_ssim(prims, poses[i], intr, rungs, sh_degree=wl["sh"])
            lt.append((time.perf_counter() - t0) * 1000.0)
        ladder = {"rungs": ["1920x1080"] + [f"{w}x{h}" for w, h in rungs],
                  "ssim_vs_1080p_last_pose": [round(x, 6) for x in ss],
                  "ms_per_ladder_p50": float(np.percentile(lt, 50)),
                  "what": "per pose: render 1080p + 3 rungs, upscale_to 1080p, ssim, on device"}

    # JPEG of the rendered frame on the device (render_view's
    # encode), byte-identical to Pillow; Pillow on the host timed beside it
    jpeg = None
    if not args.no_ladder:
        import io
        from PIL import Image
        from paper_2605_08699_b200.render import _jpeg
        frame = g.render_u8(prims, poses[W], intr, sh_degree=wl["sh"]).copy()
        jpeg = {}
        for q in (90, 65, 35):
            for _ in range(3):
                _jpeg(ctx, None, intr.width, intr.height, q)  # warm (device frame)
            jt = []
            for _ in range(20):
                g.render_u8(prims, poses[W], intr, sh_degree=wl["sh"], out=out)
                t0 = time.perf_counter()
                payload = _jpeg(ctx, None, intr.width, intr.height, q)
                jt.append((time.perf_counter() - t0) * 1000.0)
            buf = io.BytesIO()
            t0 = time.perf_counter()
            Image.fromarray(frame, "RGB").save(buf, format="JPEG", quality=q,
                                               subsampling=2 if q < 90 else 0)
            pil_ms = (time.perf_counter() - t0) * 1000.0
            jpeg[f"q{q}"] = {"gpu_ms_p50": float(np.percentile(jt, 50)), "bytes": len(payload),
                             "pillow_ms": pil_ms,
                             "identical_to_pillow": payload == buf.getvalue()}

    # PLY bytes in host memory -> resident scene (load_ply),
    # the reference's parse_ply + activate (oracle port) timed beside it
    scene_load = None
    if not args.no_load and rank == 0:
        scene_load = bench_scene_load(wl, peaks, peak_kind, with_cpu=not args.no_cpu_baseline)

    result = None
    if rank == 0:
        frame0 = g.render_u8(prims, poses[W], intr, sh_degree=wl["sh"])
        base, parity, port = None, None, None
        if world == 1 and not args.no_cpu_baseline:
            base, parity = cpu_reference(prims, poses[W:], intr, wl["sh"], args.cpu_budget,
                                         gpu_u8=frame0)
            port, port_parity = cpu_port(prims, poses[W:], intr, wl["sh"],
                                         args.cpu_budget / 2, gpu_u8=frame0)
            if base is None:
                base, parity, port = port, port_parity, None
            else:
                parity = {"reference": parity, "port": port_parity}
        result = {
            "metric": METRIC,
            "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": pipe_ms / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic",
            "config": {"workload": wl["desc"], "gaussians": wl["n"], "sh_degree": wl["sh"],
                       "width": wl["w"], "height": wl["h"],
                       "parallelism": f"session-sharded x{world} (no collective)",
                       "l2": "inputs larger than L2 (scene "
                             f"{sc.device_bytes / 1e6:.0f} MB > 126 MB)"},
            "latency_ms": {"p50": float(np.percentile(lat, 50)),
                           "p99": float(np.percentile(lat, 99)),
                           "device_p50": float(np.percentile(dev_lat, 50)),
                           "device_p99": float(np.percentile(dev_lat, 99)),
                           "calls": len(lat), "api": "render_u8 into a pinned frame, one call "
                                                     "at a time (wall) / its CUDA events"},
            "value_single_stream": value_single,
            "streams": S,
            "e2e": {"value": world * K / e2e_s, "unit": "frames/s",
                    "h2d_bytes_per_step": ctypes.sizeof(_lib.GsrCamera),
                    "d2h_bytes_per_step": int(out.nbytes),
                    "api": f"RenderPipeline(depth={S}).submit: {S} frames in flight"},
            "e2e_single": {"value": world * K / e2e_single_s, "unit": "frames/s",
                           "api": "render_u8, one call at a time"},
            "gpu_launches": launches,
            "gpu_launches_per_frame": launches_single / max(K, 1),
            "retry_frames": retry,
            "stages_ms": stages,
            "kernels": kernels,
            "counters": {k: int(v) for k, v in counters.items()},
            "roofline": roof,
            "roofline_hbm": roofline_hbm,
            "contract_binning": contract,
            "ladder": ladder,
            "jpeg": jpeg,
            "scene_load": scene_load,
            "clocks": clocks.summary(),
        }
        if base is not None:
            result["cpu_baseline"] = base
            result["parity"] = parity
            if port is not None:
                result["cpu_port"] = port
    d.close()
    if result is not None:
        print(json.dumps(result), flush=True)
    return 0


def contract_profile(ctx, lib, sc, cams, wl, bg, frames):
    """Device time of the exact 16x16 contract lists built the north-star way
    (gsr_debug_contract_tiles: (tile|rank) keys + 64-bit radix sort + ranges)
    on the render path's own frames, beside that frame's binning stage."""
    from paper_2605_08699_b200 import _lib
    st = _lib.GsrStats()
    ms, d_keys, binning = [], [], []
    lib.gsr_ctx_set_kernel_timing(ctx.handle, 4)  # stage times (the binning stage)
    for cam in cams[:frames]:
        _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(cam), bg, wl["sh"], 1,
                                  None, None, None, ctypes.byref(st)))
        binning.append(st.ms_binning)
        n = ctypes.c_int64(0)
        t = ctypes.c_float(0.0)
        _lib.check(lib.gsr_debug_contract_tiles(ctx.handle, 16, ctypes.byref(n), None, None,
                                                 None, ctypes.byref(t)))
        ms.append(t.value)
        d_keys.append(n.value)
    lib.gsr_ctx_set_kernel_timing(ctx.handle, 0)
    if not ms:
        return None
    dk = float(np.mean(d_keys))
    k = float(wl["n"])
    return {"ms_keys_sort_ranges": float(np.mean(ms)), "D16": dk,
            "alg_bytes": int(24 * k + 28 * dk),
            "achieved_gbs": (24 * k + 28 * dk) / (float(np.mean(ms)) * 1e-3) / 1e9,
            "render_path_binning_ms": float(np.mean(binning)),
            "what": "exact 16x16 contract, north-star item (2): (tile|rank) u64 keys, "
                    "Onesweep radix sort, range identification (SURVEY 8d B_sort = 24K + 28D), "
                    "from the depth-ranked records; the render path's sort-free 32x16 binning "
                    "stage (gather + pairs + lists) of the same frames beside it"}


ABR_FIXTURE = ROOT / "tests" / "golden" / "abr_sequence.json"


def config5_plan(wl, rank, world):
    """Sessions of this rank: config 5 (64 sessions, strong scaling) or
    config 5w (8 sessions per GPU, weak scaling); session i -> GPU i mod N."""
    from paper_2605_08699_b200.sessions import config5_sessions, shard
    n = 8 * world if wl.get("weak") else 64
    return n, shard(config5_sessions(n), rank, world)


def run_config5(args, wl):
    """BASELINE config 5: pose-trace sessions over the 14 synthetic scene sizes
    N_k = round(250k * 24^(k/13)) (250k ... 6M), session i -> GPU i mod N, no
    collective (sessions.py).  Each rank holds replicas of the scenes its
    sessions use and serves its sessions round-robin.
      all-1080p  RenderPipeline (--streams frames in flight): u8 frames to
                 pinned host memory; value = frames of all ranks / max-over-
                 ranks wall time; per-frame latency = submit -> frame returned
                 (wall) and the frame's device time (CUDA events).
      abr_mixed  every frame at the rung the reference's LatencyAbr chose for
                 that session and step (tests/golden/abr_sequence.json), served
                 as the server does (render_view: render + JPEG on the
                 device, JPEG bytes to the host) by --streams worker threads,
                 one context each (server.py:99-114)."""
    import concurrent.futures as cf
    import torch  # noqa: F401
    d = Dist()
    rank, local_rank, world = d.rank, d.local_rank, d.world
    import paper_2605_08699_b200 as g
    from paper_2605_08699_b200.sessions import scenes_for
    from paper_2605_08699_b200.synth import base_intrinsics_1080p, ladder_1080p, synthetic_scene
    g.set_device(local_rank)
    n_sessions, mine = config5_plan(wl, rank, world)
    scenes = {k: synthetic_scene(next(s.gaussians for s in mine if s.scene == k), seed=k,
                                 sh_degree=3) for k in scenes_for(mine)}
    intr = base_intrinsics_1080p()
    K, W, S = args.steps, args.warmup, max(1, args.streams)
    # a session's k-th timed frame is step W + k * stride of its 300-step
    # trace, so the ABR-mixed run samples the whole controller trajectory
    # (it starts at the worst rung) rather than its first frames
    per = (K + len(mine) - 1) // len(mine)
    stride = max(1, (300 - W) // max(per, 1))
    traces = {s.index: poses_for(s.index, 300) for s in mine}
    order = [(mine[i % len(mine)], min(299, W + (i // len(mine)) * stride)) for i in range(K)]

    # ---- all-1080p through RenderPipeline ----
    pipe = g.RenderPipeline(intr, sh_degree=3, depth=S, device=local_rank, record_stats=True)
    # upload every scene and warm every (context, scene) pair: a context
    # captures one CUDA graph per scene configuration on its first frame of
    # it, which must not land in the timed region (the pipeline's contexts
    # rotate per submit, so each scene is submitted once per context)
    nctx = len(pipe.ctxs)
    # twice: a graph is keyed by the context's buffer capacities, which the
    # larger scenes grow during the first pass
    for _ in range(2):
        for s in mine:
            for t in range(max(W, nctx)):
                pipe.submit(scenes[s.scene], traces[s.index][t % 300])
    pipe.drain()
    pipe.frame_ms.clear()
    pipe.kernel_launches = 0
    t_sub = {}
    lat = []
    d.barrier()
    with ClockSampler(local_rank) as clocks:
        t0 = time.perf_counter()
        for i, (s, t) in enumerate(order):
            t_sub[i] = time.perf_counter()
            r = pipe.submit(scenes[s.scene], traces[s.index][t], tag=i)
            if r is not None:
                lat.append((time.perf_counter() - t_sub[r[0]]) * 1000.0)
        for tag, _ in pipe.drain():
            lat.append((time.perf_counter() - t_sub[tag]) * 1000.0)
        wall = time.perf_counter() - t0
    wall = d.max(wall)
    dev_ms = list(pipe.frame_ms)
    launches5 = int(d.sum(pipe.kernel_launches))  # kernels of the timed frames, all ranks
    pipe.close()

    # ---- ABR-mixed: the server's per-request work at the ABR's rung ----
    fx = json.loads(ABR_FIXTURE.read_text())
    levels = {e["index"]: e["levels"] for e in fx["sessions"]}
    rungs = fx["rungs"]

    class Profile:
        def __init__(self, r):
            self.width, self.height, self.jpeg_quality = r["width"], r["height"], \
                r["jpeg_quality"]

    profiles = [Profile(r) for r in rungs]
    abr_order = [(s, t, int(levels[s.index][t % len(levels[s.index])])) for s, t in order]

    def serve(item):
        s, t, lv = item
        t0 = time.perf_counter()
        payload, st = g.render_view(scenes[s.scene], traces[s.index][t], intr, profiles[lv],
                                    sh_degree=3, device=local_rank)
        return (time.perf_counter() - t0) * 1000.0, st.device_ms, len(payload), lv

    with cf.ThreadPoolExecutor(max_workers=S) as ex:
        for _ in range(2):  # warm (twice: graphs are keyed by the grown capacities too)
            list(ex.map(serve, [(s, 0, lv) for s in mine for lv in range(len(rungs))]))
        d.barrier()
        t0 = time.perf_counter()
        res = list(ex.map(serve, abr_order))
        abr_wall = d.max(time.perf_counter() - t0)
    abr_hist = [0] * len(rungs)
    for r in res:
        abr_hist[r[3]] += 1

    # gather per-frame latencies of every rank for the box percentiles
    lat_all = [x for part in d.gather(lat) for x in part]
    dev_all = [x for part in d.gather(dev_ms) for x in part]
    abr_lat = [x for part in d.gather([r[0] for r in res]) for x in part]
    abr_dev = [x for part in d.gather([r[1] for r in res]) for x in part]
    abr_bytes = sum(r[2] for r in res)

    parity, base = None, None
    if rank == 0 and not args.no_cpu_baseline:
        parity = config5_spot_check(g, scenes, traces, mine, intr, profiles, levels, W)
        if world == 1:
            base = config5_cpu(scenes, traces, mine, intr, W, args.cpu_budget)
    if rank == 0:
        pct = lambda xs, q: float(np.percentile(xs, q)) if xs else None  # noqa: E731
        line = {
            "metric": METRIC5,
            "value": world * K / wall, "unit": "frames/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": 1000.0 * wall / K, "higher_is_better": True,
            "scaling": "weak" if wl.get("weak") else "strong", "vs_baseline": None,
            "dtype": "f64+f32", "data": "synthetic",
            "config": {"workload": wl["desc"], "sessions": n_sessions,
                       "sessions_per_gpu": len(mine), "scenes_per_gpu": len(scenes),
                       "gaussians_resident": int(sum(p.count for p in scenes.values())),
                       "parallelism": f"session-sharded x{world} (no collective)",
                       "frames_in_flight": S, "levels": "all 1920x1080",
                       "l2": "inputs larger than L2 (scenes >= 76 MB each, 6.2 MB frames)"},
            "latency_ms": {"p50": pct(lat_all, 50), "p99": pct(lat_all, 99),
                           "device_p50": pct(dev_all, 50), "device_p99": pct(dev_all, 99),
                           "frames": len(lat_all),
                           "what": f"per frame under the {n_sessions}-session load: submit -> "
                                   "frame returned (wall, includes queueing behind the frames "
                                   "in flight) and the frame's device time (CUDA events)"},
            "e2e": {"value": world * K / wall, "unit": "frames/s", "h2d_bytes_per_step": 160,
                    "d2h_bytes_per_step": 3 * intr.width * intr.height,
                    "api": f"RenderPipeline(depth={S}).submit"},
            "abr_mixed": {"value": world * K / abr_wall, "unit": "frames/s",
                          "latency_ms": {"p50": pct(abr_lat, 50), "p99": pct(abr_lat, 99),
                                         "device_p50": pct(abr_dev, 50),
                                         "device_p99": pct(abr_dev, 99)},
                          "level_histogram": abr_hist,
                          "rungs": [f"{r['width']}x{r['height']}q{r['jpeg_quality']}"
                                    for r in rungs],
                          "jpeg_bytes_per_frame": abr_bytes / max(len(res), 1),
                          "api": f"render_view (render + JPEG on the device) from {S} server "
                                 "threads, one context each",
                          "levels_from": "tests/golden/abr_sequence.json (reference LatencyAbr "
                                         "+ TokenBucketShaper, virtual time)"},
            "gpu_launches": launches5,
            "clocks": clocks.summary(),
        }
        if parity is not None:
            line["parity"] = parity
        if base is not None:
            line["cpu_baseline"] = base
        print(json.dumps(line), flush=True)
    d.close()
    return 0


def config5_spot_check(g, scenes, traces, mine, intr, profiles, levels, W):
    """Frames of 3 sessions vs the C oracle: the 1080p u8 frame through
    RenderPipeline, and the ABR rung's JPEG through render_view vs Pillow's
    encode of the oracle frame at that rung (byte-equal)."""
    import io
    from PIL import Image
    from oracle import oracle as orc
    orc.build()
    out = []
    pipe = g.RenderPipeline(intr, sh_degree=3, depth=2)
    for s in mine[:3]:
        prims, pose = scenes[s.scene], traces[s.index][W]
        pipe.submit(prims, pose)
        (_, u8), = pipe.drain()
        rot, w2c = orc.world_to_camera(pose.azimuth, pose.elevation, pose.translation)

        def oracle_u8(ii):
            return orc.render(prims.means, prims.scales, prims.rotations, prims.opacities,
                              prims.colors_dc, prims.sh_coeffs, w2c, rot, ii.fx, ii.fy, ii.cx,
                              ii.cy, ii.width, ii.height, (0.0, 0.0, 0.0), 3).u8

        ref = oracle_u8(intr)
        lv = int(levels[s.index][W])
        prof = profiles[lv]
        payload, _ = g.render_view(prims, pose, intr, prof, sh_degree=3)
        ri = g.scale_intrinsics(intr, prof.width, prof.height)
        buf = io.BytesIO()
        Image.fromarray(oracle_u8(ri), "RGB").save(buf, format="JPEG", quality=prof.jpeg_quality,
                                                   subsampling=2 if prof.jpeg_quality < 90 else 0)
        out.append({"session": s.index, "gaussians": s.gaussians,
                    "u8_1080p_bit_exact": bool(np.array_equal(u8, ref)),
                    "abr_level": lv, "jpeg_identical": payload == buf.getvalue()})
    pipe.close()
    return out


def config5_cpu(scenes, traces, mine, intr, W, budget):
    """config 5 on the host: sequential frames over the size mix,
    the reference's render (numba, all cores) when shipped, else the port;
    sessions in serving order, bounded to ~budget seconds."""
    mods = reference_modules()
    times, kind = [], "reference" if mods else "port"
    t_all = time.perf_counter()
    cores = None
    for i, s in enumerate(mine):
        prims, pose = scenes[s.scene], traces[s.index][W]
        if mods:
            b, _ = cpu_reference(prims, [pose], intr, 3, 0.0)
            cores = b["cores"]
        else:
            b, _ = cpu_port(prims, [pose], intr, 3, 0.0)
            cores = b["cores"]
        times.append(b["ms_per_frame"] / 1000.0)
        if time.perf_counter() - t_all > budget:
            break
    return {"value": len(times) / sum(times), "unit": "frames/s", "cores": cores, "kind": kind,
            "sample": f"{len(times)} sequential 1080p frame(s), one per session in serving order "
                      f"(sessions {[s.index for s in mine[:len(times)]]}), "
                      f"{sum(times):.1f} s (JIT warm-up excluded)",
            "host_cpu": host_cpu()}


def run_reference_config5(args, wl):
    from paper_2605_08699_b200.sessions import scenes_for
    from paper_2605_08699_b200.synth import base_intrinsics_1080p, synthetic_scene
    n_sessions, mine = config5_plan(wl, 0, 1)
    budget = float(os.environ.get("BENCH_REF_BUDGET_S", "150"))
    intr = base_intrinsics_1080p()
    scenes, base = {}, None
    traces = {s.index: poses_for(s.index, args.warmup + 1) for s in mine}
    # scenes are built lazily in serving order so the budget bounds the work
    built = []
    for k in scenes_for(mine):
        scenes[k] = synthetic_scene(next(s.gaussians for s in mine if s.scene == k), seed=k,
                                    sh_degree=3)
        built.append(k)
        if len(built) >= 4:
            break
    sub = [s for s in mine if s.scene in scenes]
    base = config5_cpu(scenes, traces, sub, intr, args.warmup, budget)
    line = {"metric": METRIC5, "value": base["value"], "unit": "frames/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / base["value"],
            "higher_is_better": True, "scaling": "weak" if wl.get("weak") else "strong",
            "vs_baseline": None, "dtype": "f64+f32", "data": "synthetic", "impl": "reference",
            "config": {"workload": wl["desc"], "sessions": n_sessions,
                       "parallelism": "host cores"},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_dry(args, wl):
    """--dry-run: the multi-process path without CUDA (gloo): rank r takes its
    sessions (config 3: trace seed r; config 5: i mod N), prepares each
    step's camera on the host, and the max-over-ranks timing reduction runs
    as in the real bench.  Used by the CPU tests of the launcher."""
    d = Dist(dry=True)
    from paper_2605_08699_b200.render import make_camera
    if wl.get("config5"):
        n_sessions, mine = config5_plan(wl, d.rank, d.world)
        ids = [s.index for s in mine]
    else:
        n_sessions, ids = d.world, [d.rank]
    intr = intrinsics(wl) if not wl.get("config5") else None
    if intr is None:
        from paper_2605_08699_b200.synth import base_intrinsics_1080p
        intr = base_intrinsics_1080p()
    poses = {i: poses_for(i, args.warmup + args.steps) for i in ids}
    d.barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        make_camera(poses[ids[k % len(ids)]][args.warmup + k // len(ids)], intr)
    el = d.max(time.perf_counter() - t0)
    all_ids = d.gather(ids)
    if d.rank == 0:
        print(json.dumps({"metric": METRIC5 if wl.get("config5") else METRIC,
                          "value": d.world * args.steps / max(el, 1e-9), "unit": "steps/s",
                          "n_gpus": d.world, "steps": args.steps, "warmup": args.warmup,
                          "dry_run": True, "sessions": n_sessions, "sessions_by_rank": all_ids,
                          "config": {"workload": wl["desc"],
                                     "parallelism": f"session-sharded x{d.world} "
                                                    "(no collective)"}}), flush=True)
    d.close()
    return 0


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["gsr", "reference"], default="gsr")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="config3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-ladder", action="store_true")
    ap.add_argument("--no-load", action="store_true", help="skip the PLY scene-load section")
    ap.add_argument("--streams", type=int, default=4,
                    help="frames in flight (contexts/streams) for value and e2e")
    ap.add_argument("--latency-calls", type=int, default=200,
                    help="one-call latency samples (p50/p99), independent of --steps")
    ap.add_argument("--dry-run", action="store_true",
                    help="no CUDA: launcher, sharding and max-over-ranks only (gloo)")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args.gpus, argv)
    wl = WORKLOADS[args.workload]
    if args.dry_run:
        return run_dry(args, wl)
    if args.impl == "reference":
        return run_reference(args, wl)
    if wl.get("config5"):
        return run_config5(args, wl)
    return run_gsr(args, wl)


if __name__ == "__main__":
    sys.exit(main())
