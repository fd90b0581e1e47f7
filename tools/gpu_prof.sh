# Launch list of one config-3 frame + one ncu --set full capture of its kernels.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "frame/" \
  --csv --log-file gpurun_out/launches.csv python tools/profile_frame.py 4 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 1 | tee gpurun_out/launches.txt
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "frame/" \
  -o gpurun_out/${NCU_NAME:-frame_full} -f python tools/profile_frame.py 3 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
