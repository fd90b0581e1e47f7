"""Blend instrumentation at a workload (VERDICT r1 "next" 4): list entries
walked per work item, the share whose row range meets the item's rows,
composite-loop iterations and lane efficiency, from the counting blend
variant (GSR_TIMING_COUNTERS), beside the serving blend's event time.

    python tools/blend_profile.py [config3] [frames]
"""

from __future__ import annotations

import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

NAMES = ["K", "D", "P", "E", "Rb", "Rp", "walked", "hit", "batches", "iters_x32", "lanes",
         "items", "used", "KA", "KB"]


def main():
    wl_name = sys.argv[1] if len(sys.argv) > 1 else "config3"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    wl = bench.WORKLOADS[wl_name]
    from paper_2605_08699_b200 import _lib
    from paper_2605_08699_b200.render import _bg, device_scene, make_camera, tile_size
    prims = bench.build_scene(wl)
    intr = bench.intrinsics(wl)
    poses = bench.poses_for(0, frames + 3)
    sc = device_scene(prims, 0)
    ctx = _lib.context(0)
    lib = ctx.lib
    st = _lib.GsrStats()
    bg = _bg((0.0, 0.0, 0.0))
    cams = [make_camera(p, intr) for p in poses]
    for c in cams[:3]:
        _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(c), bg, wl["sh"], 1, None,
                                  None, None, ctypes.byref(st)))
    rows, blend_ms, items = [], [], []
    out = (ctypes.c_uint64 * 15)()
    for c in cams[3:]:
        _lib.check(lib.gsr_ctx_set_kernel_timing(ctx.handle, 4))  # stage times
        _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(c), bg, wl["sh"], 1, None,
                                  None, None, ctypes.byref(st)))
        blend_ms.append(st.ms_blend)
        _lib.check(lib.gsr_ctx_set_kernel_timing(ctx.handle, 2))
        _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(c), bg, wl["sh"], 1, None,
                                  None, None, ctypes.byref(st)))
        _lib.check(lib.gsr_debug_frame_counters(ctx.handle, out, 15))
        rows.append([int(x) for x in out])
        tw, th = tile_size()
        n_items = ((intr.width + tw - 1) // tw) * ((intr.height + th - 1) // th) * (th // 2)
        info = np.empty(n_items, dtype=np.uint32)
        _lib.check(lib.gsr_debug_blend_items(ctx.handle, info.ctypes.data, n_items))
        items.append(info)
    lib.gsr_ctx_set_kernel_timing(ctx.handle, 0)
    m = {k: float(np.mean([r[i] for r in rows])) for i, k in enumerate(NAMES)}
    iters = m["iters_x32"] / 32.0
    res = {
        "workload": wl["desc"], "frames": len(rows),
        "blend_ms_serving": float(np.mean(blend_ms)),
        "counters": m,
        "items": m["items"],
        "entries_walked_per_item": m["walked"] / m["items"],
        "list_entries_D": m["D"],
        "walk_fraction_of_full_lists": m["walked"] / (m["D"] * 32.0),
        "hit_fraction": m["hit"] / m["walked"],
        "batches_per_item": m["batches"] / m["items"],
        "composites_E": m["E"],
        "composite_iterations_warp": iters,
        "lane_efficiency": m["lanes"] / (2.0 * m["iters_x32"]),
        "composites_per_iteration": m["E"] / iters,
        "composites_per_batch": m["E"] / m["batches"],
        "splats_colour_read_fraction_of_K": m["used"] / m["K"],
        "tile": list(tile_size()),
        "slices": {"KA": m["KA"], "KB": m["KB"],
                   "note": "counters sum both slices of a depth-sliced frame"},
    }
    sat = np.concatenate([(x >> 31) == 1 for x in items])
    last = np.concatenate([(x & 0x7fffffff) for x in items]).astype(np.float64)
    kk = np.concatenate([np.full(len(x), r[0], dtype=np.float64) for x, r in zip(items, rows)])
    frac = last / kk
    res["items_unsaturated_fraction"] = float(1.0 - sat.mean())
    res["saturated_items_last_rank_fraction_of_K"] = {
        q: float(np.percentile(frac[sat], q)) for q in (50, 90, 99, 99.9, 100)} if sat.any() else None
    res["unsaturated_items_last_rank_fraction_of_K"] = {
        q: float(np.percentile(frac[~sat], q)) for q in (50, 90, 100)} if (~sat).any() else None
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
