"""Debug: one-pass vs depth-sliced frames at a workload, with slice counters."""
import ctypes, json, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench
import paper_2605_08699_b200 as g
from paper_2605_08699_b200 import _lib
from paper_2605_08699_b200.render import set_slicing

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "config3"]
prims = bench.build_scene(wl)
intr = bench.intrinsics(wl)
poses = bench.poses_for(0, 6)
ctx = _lib.context(0)
for i, pose in enumerate(poses):
    set_slicing(1 << 40)
    one = g.render_framebuffer(prims, pose, intr, sh_degree=wl["sh"])
    set_slicing()
    sl = g.render_framebuffer(prims, pose, intr, sh_degree=wl["sh"])
    raw = (ctypes.c_uint64 * 15)()
    _lib.check(ctx.lib.gsr_debug_frame_counters(ctx.handle, raw, 15))
    d = np.abs(sl._rgb32 - one._rgb32).max(axis=2)
    bad = np.argwhere(d > 0)
    t = np.abs(sl._t32 - one._t32)
    print(json.dumps({"pose": i, "KA": raw[13], "KB": raw[14], "K": raw[0],
                      "mismatch_px": int(len(bad)), "T_mismatch": int((t > 0).sum()),
                      "first_bad": bad[:5].tolist(),
                      "bad_rows": sorted(set(int(y) for y, x in bad))[:20]}), flush=True)
