import os, sys
sys.path.insert(0, ".")
os.environ["GSR_SLICE_MIN"] = "1"
import paper_2605_08699_b200 as g
from paper_2605_08699_b200.synth import synthetic_scene
prims = synthetic_scene(20000, seed=3, sh_degree=3)
intr = g.Intrinsics(fx=300.0, fy=300.0, cx=160.0, cy=120.0, width=320, height=240)
print("scene", flush=True)
import numpy as np
out = np.empty((240, 320, 3), np.uint8)
g.render_u8(prims, g.CameraPose(0.0, 0.0), intr, sh_degree=3, out=out)
print("render_u8 pageable", flush=True)
g.render_framebuffer(prims, g.CameraPose(0.01, 0.0), intr, sh_degree=3)
print("render_framebuffer", flush=True)
g.render_u8(prims, g.CameraPose(0.02, 0.0), intr, sh_degree=3)
print("render_u8", flush=True)
