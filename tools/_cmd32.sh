python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "frame/" -k regex:"blend|seg_place|bin_pairs" -o gpurun_out/k3 -f python tools/profile_frame.py 3 > gpurun_out/k3.log 2>&1
tail -2 gpurun_out/k3.log
