"""Render config-3 frames for ncu captures; the LAST frame runs inside an NVTX
range "frame" so captures can select exactly one whole frame:

    ncu --nvtx --nvtx-include "frame/" ... python tools/profile_frame.py [n_frames] [workload]
"""
import os
import sys
from pathlib import Path

# ncu cannot profile the kernel nodes of graphs with conditional nodes:
# direct launches (same kernels, slice B sized on the host)
os.environ.setdefault("GSR_GRAPHS", "0")

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402  (NVTX markers only)

import bench  # noqa: E402
import paper_2605_08699_b200 as g  # noqa: E402

wl = bench.WORKLOADS[sys.argv[2] if len(sys.argv) > 2 else "config3"]
prims = bench.build_scene(wl)
intr = bench.intrinsics(wl)
nf = int(sys.argv[1]) if len(sys.argv) > 1 else 3
first = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # first pose of the bench trace
poses = bench.poses_for(0, first + nf)[first:]
st = g.RenderStats()
mark_all = len(sys.argv) > 3 and sys.argv[3] == "all"  # every frame in the NVTX range
for i, p in enumerate(poses):
    last = mark_all or i == len(poses) - 1
    if last:
        torch.cuda.nvtx.range_push("frame")
    g.render_u8(prims, p, intr, sh_degree=wl["sh"], stats=st)
    if last:
        torch.cuda.nvtx.range_pop()
print("frames", len(poses), "drawn", st.splats_drawn, "D", st.tile_keys)
