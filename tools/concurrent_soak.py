"""Several server-like threads, each with its own context, rendering random
soak cases concurrently; every frame bit-compared (u8) with the oracle.
python tools/concurrent_soak.py THREADS CASES_PER_THREAD SEED"""
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import paper_2605_08699_b200 as g  # noqa: E402
from paper_2605_08699_b200 import synth  # noqa: E402
from test_parity_soak import _case  # noqa: E402


def main(nt, per, seed):
    from oracle import oracle
    oracle.build()
    rng = np.random.default_rng(seed)
    cases = [[_case(g, synth, rng) for _ in range(per)] for _ in range(nt)]
    frames = [[None] * per for _ in range(nt)]
    errs = []

    def run(t):
        try:
            for k, (prims, intr, pose, sh, bg) in enumerate(cases[t]):
                frames[t][k] = g.render_framebuffer(prims, pose, intr, bg, sh).u8.copy()
        except BaseException as e:  # noqa: BLE001
            errs.append((t, repr(e)))
    ths = [threading.Thread(target=run, args=(t,)) for t in range(nt)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    assert not errs, errs
    bad = 0
    for t in range(nt):
        for k, (prims, intr, pose, sh, bg) in enumerate(cases[t]):
            rot, w2c = oracle.world_to_camera(pose.azimuth, pose.elevation, pose.translation)
            ref = oracle.render(prims.means, prims.scales, prims.rotations, prims.opacities,
                                prims.colors_dc, prims.sh_coeffs, w2c, rot, intr.fx, intr.fy,
                                intr.cx, intr.cy, intr.width, intr.height, bg, sh)
            if not np.array_equal(frames[t][k], ref.u8):
                bad += 1
                print("MISMATCH thread", t, "case", k, prims.count, intr.width, intr.height)
    print(f"concurrent soak: {nt} threads x {per} frames, {bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])))
