# Quick GPU iteration: build, pytest -m gpu, two bench runs with the per-kernel table.
# Usage (from the repo root): gpurun --timeout 1500 -- bash tools/gpu_quick.sh
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for m in 0 1; do
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-ladder 2>&1 | tail -1 > gpurun_out/bench$m.json
python -c "import json; d=json.load(open('gpurun_out/bench$m.json')); print(d['value'], d['value_single_stream'], d['e2e']['value'], d['latency_ms']); [print(k, v['ms_per_frame']) for k, v in d['kernels'].items()]"
done
