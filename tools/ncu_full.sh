# One ncu --set full capture of the hot kernels of one config-3 frame (frame 2).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"${NCU_K:-bin_pairs|blend_kernel|seg_place|onesweep|preprocess_kernel|bin_gather}" \
  -s ${NCU_S:-13} -c ${NCU_C:-13} -o gpurun_out/${NCU_NAME:-full} -f \
  python tools/profile_frame.py 3 ${NCU_WL:-config3} > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out
