"""Replay one randomised soak case (tests/test_parity_soak.py) and report how
the GPU frame differs from the oracle: python tools/debug_soak_case.py SEED K"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_2605_08699_b200 as g  # noqa: E402
from paper_2605_08699_b200 import synth  # noqa: E402
from test_parity_soak import _case  # noqa: E402


def main(seed, k, start=None):
    """Cases start..k-1 are rendered first in this process (the soak's history)."""
    from oracle import oracle
    oracle.build()
    rng = np.random.default_rng(seed)
    for i in range(k + 1):
        prims, intr, pose, sh, bg = _case(g, synth, rng)
        if start is not None and start <= i < k:
            g.render_framebuffer(prims, pose, intr, bg, sh)
            g.evict(prims)
    print("case", k, prims.count, "sh", sh, intr, pose, bg)
    print("scales min/max", prims.scales.min(), prims.scales.max())
    st = g.RenderStats()
    fb = g.render_framebuffer(prims, pose, intr, bg, sh, st)
    rot, w2c = oracle.world_to_camera(pose.azimuth, pose.elevation, pose.translation)
    ref = oracle.render(prims.means, prims.scales, prims.rotations, prims.opacities,
                        prims.colors_dc, prims.sh_coeffs, w2c, rot, intr.fx, intr.fy,
                        intr.cx, intr.cy, intr.width, intr.height, bg, sh)
    print("drawn", st.splats_drawn, ref.splats_drawn, "stats", {k: getattr(st, k) for k in dir(st) if not k.startswith("_")})
    du = fb.u8.astype(int) - ref.u8.astype(int)
    bad = np.argwhere(np.any(du != 0, axis=2))
    print("u8 pixels differing:", len(bad), "max |d|", np.abs(du).max())
    dr = fb._rgb32.view(np.uint32) != ref.rgb32.view(np.uint32)
    dt = fb._t32.view(np.uint32) != ref.trans32.view(np.uint32)
    print("rgb32 differing:", int(np.any(dr, axis=2).sum()) if dr.ndim == 3 else int(dr.sum()),
          "t32 differing:", int(dt.sum()))
    if len(bad):
        ys, xs = bad[:, 0], bad[:, 1]
        print("rows", ys.min(), ys.max(), "cols", xs.min(), xs.max())
        print("tiles (32x16):", sorted(set(zip((ys // 16).tolist(), (xs // 32).tolist())))[:40])
        y, x = bad[0]
        print("first", (y, x), "gpu", fb._rgb32[y, x], fb._t32[y, x], "ref", ref.rgb32[y, x], ref.trans32[y, x])
    return 0 if (not len(bad) and not dr.any() and not dt.any()) else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else None))
