mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench.json
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['latency_ms'], d['gpu_launches'], json.dumps(d['stages']))"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 25 --csv --log-file gpurun_out/launches.csv python tools/profile_frame.py 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 1
