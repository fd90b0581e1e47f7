# Round-2 evidence on one B200: parity tests, smoke, the default bench line
# (config 3 with the numba CPU baseline), the reference arm, configs 1/2/4/5/5w,
# a launch list and one `ncu --set full` capture of a whole config-3 frame.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
timeout 1200 python bench.py --steps 200 --warmup 10 2>gpurun_out/bench_config3.err | tail -1 > gpurun_out/bench_config3.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 2>/dev/null | tail -1 > gpurun_out/bench_reference.json
for wl in config1 config2 config4; do
  timeout 900 python bench.py --workload $wl --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_$wl.json
done
timeout 1500 python bench.py --workload config5 --steps 256 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_config5.json
timeout 900 python bench.py --workload config5w --steps 64 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench_config5w.json
for f in gpurun_out/bench_*.json; do python - "$f" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read())
except Exception as e:
    print(sys.argv[1], "unparsable", e); sys.exit()
print(sys.argv[1], d.get("value"), d.get("unit"), "e2e", (d.get("e2e") or {}).get("value"),
      "lat", d.get("latency_ms"), "launches", d.get("gpu_launches"), "clocks", d.get("clocks"))
PY
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "frame/" \
  --csv --log-file gpurun_out/launches.csv python tools/profile_frame.py 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 1 > gpurun_out/launches.txt
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "frame/" \
  -o gpurun_out/frame_full -f python tools/profile_frame.py 3 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/frame_full.ncu-rep gpurun_out/ncu_traffic_config3.json gpurun_out/ncu_frame_summary.txt
head -40 gpurun_out/ncu_frame_summary.txt
