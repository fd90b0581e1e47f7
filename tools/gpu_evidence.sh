# Round evidence on one B200: parity tests, SIMT peaks, the bench line (with
# the CPU baseline), a launch list and one `ncu --set full` capture of a whole
# config-3 frame -> per-kernel DRAM traffic (profiles/ncu_traffic_config3.json).
mkdir -p gpurun_out tools/_build
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
nvcc -O3 -fmad=false -gencode arch=compute_100a,code=sm_100a tools/peaks.cu -o tools/_build/peaks && \
  tools/_build/peaks > gpurun_out/measured_simt_peaks.json
cat gpurun_out/measured_simt_peaks.json
cp gpurun_out/measured_simt_peaks.json profiles/measured_simt_peaks.json
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "frame/" \
  -o gpurun_out/frame_full -f python tools/profile_frame.py 3 > gpurun_out/ncu_full.log 2>&1
python tools/ncu_traffic.py gpurun_out/frame_full.ncu-rep profiles/ncu_traffic_config3.json gpurun_out/ncu_frame_summary.txt
cat gpurun_out/ncu_frame_summary.txt
cp profiles/ncu_traffic_config3.json gpurun_out/
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "frame/" \
  --csv --log-file gpurun_out/launches.csv python tools/profile_frame.py 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 1 | tee gpurun_out/launches.txt
timeout 900 python bench.py --steps 200 --warmup 10 2>&1 | tail -1 > gpurun_out/bench.json
cat gpurun_out/bench.json
# K10 (PLY load): one ncu --set full capture of the activation kernel of a 3M load
timeout 600 ncu --set full --clock-control none -k regex:ply_activate -s 3 -c 1 \
  -o gpurun_out/ply_full -f python tools/ply_bench.py 3000000 1 > gpurun_out/ncu_ply.log 2>&1
python tools/ncu_summary.py gpurun_out/ply_full.ncu-rep > gpurun_out/ncu_ply_summary.txt 2>&1
head -40 gpurun_out/ncu_ply_summary.txt
