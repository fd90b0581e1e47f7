python -c "import __graft_entry__ as g; g.build()" || exit 1
for r in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pipeline or pinned or concurrent" 2>&1 | tail -2; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for z in 1 0; do
GSR_ZERO_COPY=$z timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-ladder --no-load 2>&1 | tail -1 > gpurun_out/zc$z.json
python -c "import json; d=json.load(open('gpurun_out/zc$z.json')); print('zc=$z', round(d['value'],1), round(d['value_single_stream'],1), round(d['e2e']['value'],1), round(d['e2e_single']['value'],1), d['latency_ms'], d['kernels']['blend']['ms_per_frame'])"
done
