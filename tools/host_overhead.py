"""Where the one-call latency goes beyond the device time (config 3):
python-side render_u8 vs the raw ABI call vs enqueue / wait split.

    python tools/host_overhead.py [calls]
"""
import ctypes
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2605_08699_b200 as g  # noqa: E402
from paper_2605_08699_b200 import _lib  # noqa: E402
from paper_2605_08699_b200.render import _bg, device_scene, make_camera  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
wl = bench.WORKLOADS["config3"]
prims = bench.build_scene(wl)
intr = bench.intrinsics(wl)
poses = bench.poses_for(0, n + 10)
ctx = _lib.context(0)
lib = ctx.lib
sc = device_scene(prims, 0)
out = ctx.pinned("ho_frame", (intr.height, intr.width, 3), np.uint8)
st = _lib.GsrStats()
bg = _bg((0.0, 0.0, 0.0))
cams = [make_camera(p, intr) for p in poses]
for c in cams[:10]:
    _lib.check(lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(c), bg, 3, 1, _lib.ptr(out),
                              None, None, ctypes.byref(st)))


def med(xs):
    return round(statistics.median(xs) * 1e3, 4)


res = {}
t = []
for p in poses[10:]:
    t0 = time.perf_counter()
    g.render_u8(prims, p, intr, sh_degree=3, out=out)
    t.append(time.perf_counter() - t0)
res["render_u8_wall_ms"] = med(t)
t, dev = [], []
for c in cams[10:]:
    t0 = time.perf_counter()
    lib.gsr_render(ctx.handle, sc.handle, ctypes.byref(c), bg, 3, 1, _lib.ptr(out), None, None,
                   ctypes.byref(st))
    t.append(time.perf_counter() - t0)
    dev.append(st.ms_device / 1e3)
res["gsr_render_wall_ms"] = med(t)
res["device_ms"] = med(dev)
t = []
for p in poses[10:]:
    t0 = time.perf_counter()
    make_camera(p, intr)
    t.append(time.perf_counter() - t0)
res["make_camera_ms"] = med(t)
te, tw = [], []
for c in cams[10:]:
    t0 = time.perf_counter()
    lib.gsr_render_async(ctx.handle, sc.handle, ctypes.byref(c), bg, 3, 1)
    t1 = time.perf_counter()
    lib.gsr_ctx_finish(ctx.handle, None, ctypes.byref(st))
    t2 = time.perf_counter()
    te.append(t1 - t0)
    tw.append(t2 - t1)
res["enqueue_ms"] = med(te)
res["enqueue_plus_wait_ms"] = round(med(te) + med(tw), 4)
print(res)
