python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-ladder 2>&1 | tail -1 > gpurun_out/bench.json
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['value_single_stream'], d['e2e']['value'], d['latency_ms']); [print(k, v['ms_per_frame']) for k, v in d['kernels'].items()]"
bash tools/sanitize.sh 2>&1 | grep -E "exit=|SUMMARY"
