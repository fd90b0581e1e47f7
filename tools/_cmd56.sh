python -c "import __graft_entry__ as g; g.build()" || exit 1
GSR_BLEND_SETS=4 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for m in 2 4 2 4; do
GSR_BLEND_SETS=$m timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-ladder --no-load 2>&1 | tail -1 > gpurun_out/bench_s$m.json
echo "sets $m"; python -c "import json; d=json.load(open('gpurun_out/bench_s$m.json')); print(d['value'], d['value_single_stream'], d['e2e']['value'], d['latency_ms']['p50'], d['kernels']['blend']['ms_per_frame'])"
done
