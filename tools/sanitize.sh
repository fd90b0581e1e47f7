# compute-sanitizer over a small render (config-1-like), the ladder, JPEG and
# the depth-tie / overflow paths, depth-sliced frames (forced on the small
# scene) through render_u8 / render_framebuffer / fresh pipeline contexts:
# memcheck (device memory errors) and
# racecheck / synccheck (shared-memory hazards, barrier misuse).
mkdir -p gpurun_out
rm -f gpurun_out/sanitizer_summary.txt
python -c "import __graft_entry__ as g; g.build()" || exit 1
cat > /tmp/san_case.py <<'PY'
import os
import sys
sys.path.insert(0, ".")
os.environ["GSR_SLICE_MIN"] = "1"  # every context slices (the pipeline's too)
import numpy as np
import paper_2605_08699_b200 as g
from paper_2605_08699_b200.render import set_slicing
from paper_2605_08699_b200.synth import synthetic_scene
prims = synthetic_scene(20000, seed=3, sh_degree=3)
intr = g.Intrinsics(fx=300.0, fy=300.0, cx=160.0, cy=120.0, width=320, height=240)
for i in range(2):
    fb = g.render_framebuffer(prims, g.CameraPose(0.02 * i, -0.01, (0.0, 0.0, 0.1)), intr,
                              sh_degree=3)
jp = g.encode_jpeg(fb, 75)
up = g.upscale_to(fb.u8[::2, ::2].copy(), 320, 240)
s = g.ssim(up, fb.u8)
pipe = g.RenderPipeline(intr, sh_degree=3, depth=2)
for i in range(3):
    pipe.submit(prims, g.CameraPose(0.01 * i, 0.0))
pipe.drain()
pipe.close()
# PLY load on the device (K10) + a render from the loaded scene
from paper_2605_08699_b200.synth import make_synthetic_set, serialize_ply
dp = g.load_ply(serialize_ply(make_synthetic_set(count=5000, seed=4, include_rest=True)))
g.render_u8(dp, g.CameraPose(0.0, 0.0), intr, sh_degree=3)
_ = dp.scales, dp.colors_dc, dp.sh_coeffs
# depth-sliced frames on this small scene (forced): front slices of 15 % and
# 2 % (a larger second slice), render_u8 + render_framebuffer + a pipeline of
# fresh contexts (first frames overflow their buffers and re-render)
for frac in (0.15, 0.02):
    set_slicing(1, frac)
    for i in range(2):
        g.render_u8(prims, g.CameraPose(0.03 * i, 0.01, (0.0, 0.0, 0.05)), intr, sh_degree=3)
    g.render_framebuffer(prims, g.CameraPose(-0.02, 0.0), intr, sh_degree=3)
    pipe = g.RenderPipeline(intr, sh_degree=3, depth=2)
    for i in range(3):
        pipe.submit(prims, g.CameraPose(0.01 * i, 0.0))
    pipe.drain()
    pipe.close()
set_slicing(-1, 0.0)
# a scene large enough that every persistent preprocess CTA takes several
# 256-Gaussian tiles (its two bulk-copy stages are refilled), one-pass and
# sliced, on a small image
big = synthetic_scene(400000, seed=5, sh_degree=3)
small = g.Intrinsics(fx=60.0, fy=60.0, cx=32.0, cy=32.0, width=64, height=64)
for mn, frac in ((10 ** 12, 0.0), (1, 0.15)):  # one-pass, then sliced
    set_slicing(mn, frac)
    g.render_u8(big, g.CameraPose(0.0, 0.0), small, sh_degree=3)
set_slicing(-1, 0.0)
print("case ok", len(jp), round(s, 6))
PY
for tool in memcheck racecheck synccheck; do
  # racecheck cannot follow the graphs' device-side conditional nodes (the
  # process dies under it even with an empty case): frames run as direct
  # launches there -- the same kernels
  extra=""; envs=""
  [ "$tool" != memcheck ] && extra="--num-cuda-barriers 8"
  [ "$tool" = racecheck ] && envs="GSR_GRAPHS=0"
  env $envs timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 python /tmp/san_case.py \
    > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool exit=$?" | tee -a gpurun_out/sanitizer_summary.txt
  tail -3 gpurun_out/sanitizer_$tool.txt
done
