python -c "import __graft_entry__ as g; g.build()" || exit 1
for s in 1 2 3 4; do
timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-ladder --streams $s 2>&1 | tail -1 > gpurun_out/bench_s$s.json
python -c "import json; d=json.load(open('gpurun_out/bench_s$s.json')); print($s, d['value'], d['value_single_stream'], d['e2e']['value'])"
done
