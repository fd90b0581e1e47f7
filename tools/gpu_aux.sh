# Secondary evidence: compute-sanitizer on the current code, the other
# BASELINE workloads as bench lines, and the reference arm.
# Usage (from the repo root): gpurun --timeout 2400 -- bash tools/gpu_aux.sh
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for w in config5 config2 config4 config1; do
  timeout 900 python bench.py --workload $w --steps 50 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$w.json
  head -c 400 gpurun_out/bench_$w.json; echo
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -1 > gpurun_out/bench_reference.json
head -c 600 gpurun_out/bench_reference.json; echo
bash tools/sanitize.sh
