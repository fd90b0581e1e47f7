python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench.json
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['latency_ms'], json.dumps(d['stages']))"
NCU_K="bin_pairs|seg_place|bin_gather|blend_kernel|preprocess" NCU_S=6 NCU_C=6 NCU_NAME=bp bash tools/ncu_full.sh
