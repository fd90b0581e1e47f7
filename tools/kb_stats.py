"""Slice sizes along the bench trace (config 3): KA, KB, unsaturated items."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2605_08699_b200 import _lib  # noqa: E402
from paper_2605_08699_b200.render import _bg, device_scene, make_camera  # noqa: E402

wl = bench.WORKLOADS["config3"]
prims = bench.build_scene(wl)
intr = bench.intrinsics(wl)
poses = bench.poses_for(0, 110)
ctx = _lib.context(0)
lib = ctx.lib
sc = device_scene(prims, 0)
st = _lib.GsrStats()
out = (ctypes.c_uint64 * 16)()
ka, kb, nu = [], [], []
for p in poses:
    cam = make_camera(p, intr)
    _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(cam), _bg((0.0, 0.0, 0.0)), 3, 1,
                              None, None, None, ctypes.byref(st)))
    _lib.check(lib.gsr_debug_frame_counters(ctx.handle, out, 16))
    v = [int(x) for x in out]
    ka.append(v[13]); kb.append(v[14]); nu.append(v[15])
kb = np.array(kb)
print("KA median", int(np.median(ka)), "KB pct 10/50/90/max", [int(np.percentile(kb, q)) for q in (10, 50, 90, 100)],
      "KB==0", int((kb == 0).sum()), "of", len(kb), "n_unsat median", int(np.median(nu)))
