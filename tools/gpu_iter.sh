# One GPU iteration: parity tests, a short bench, a launch list of 4 frames.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 ${BENCH_ARGS:---no-cpu-baseline} 2>&1 | tail -1 > gpurun_out/bench.json
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['latency_ms'], d['gpu_launches'], d['e2e']); print(json.dumps(d['stages_ms'])); print(json.dumps(d['roofline'])); [print(k, v) for k, v in d['kernels'].items()]; print(d.get('ladder'))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "frame/" --csv --log-file gpurun_out/launches.csv python tools/profile_frame.py 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 1 | tee gpurun_out/launches.txt
