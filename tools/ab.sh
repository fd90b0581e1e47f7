# A/B of tuning builds on one box.  Usage: VARIANTS="base:;t32:GSR_TILE_H=32" bash tools/ab.sh
# Each variant "name:DEF1,DEF2" is built into _build/ab_<name>.so and benched twice.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "${VS[@]}"; do
  name="${v%%:*}"; defs="${v#*:}"
  args=""; IFS=',' read -ra DS <<< "$defs"; for d in "${DS[@]}"; do [ -n "$d" ] && args="$args -D $d"; done
  python -m paper_2605_08699_b200.build --out paper_2605_08699_b200/_build/ab_$name.so $args > /dev/null || { echo "build $name failed"; continue; }
done
for rep in 1 2; do
for v in "${VS[@]}"; do
  name="${v%%:*}"
  GSR_LIB_PATH=paper_2605_08699_b200/_build/ab_$name.so timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-ladder --no-load ${BENCH_ARGS} 2>/dev/null | tail -1 > gpurun_out/ab_${name}_$rep.json
  python - "$name" gpurun_out/ab_${name}_$rep.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
k = d["kernels"]
bl = {n: round(v["ms_per_frame"], 4) for n, v in k.items() if n.startswith("blend") or n in ("seg_place", "bin_pairs", "radix32_pass", "slice_b_filter")}
print(f"{sys.argv[1]:10s} value={d['value']:.1f} single={d.get('value_single_stream', 0):.1f} e2e={d['e2e']['value']:.1f} "
      f"p50={d['latency_ms']['p50']:.3f} dev_p50={d['latency_ms']['device_p50']:.3f} {bl}")
PY
done
done
