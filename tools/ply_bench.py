"""Time the GPU PLY load (gsr_scene_create_ply) on a config-3-sized scene.

    python tools/ply_bench.py [count] [repeats]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_2605_08699_b200 import model  # noqa: E402
from paper_2605_08699_b200.synth import make_synthetic_set, scale_range_for, serialize_ply  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
raw = make_synthetic_set(count=n, seed=7, scale_range=scale_range_for(n), include_rest=True)
data = serialize_ply(raw, include_rest=True)
rows = []
for i in range(reps):
    st = {}
    t0 = time.perf_counter()
    p = model.load_ply(data, stats=st)
    st["wall_ms"] = (time.perf_counter() - t0) * 1e3
    rows.append(st)
    p.scene.close()
best = min(rows, key=lambda r: r["wall_ms"])
out = {"count": n, "ply_bytes": len(data), "best": best,
       "body_gbs_h2d": best["body_bytes"] / best["h2d_ms"] / 1e6,
       "kernel_gbs": (best["body_bytes"] + best["scene_bytes"]) / best["kernel_ms"] / 1e6}
print(json.dumps(out))
