python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
NCU_K="preprocess|bin_pairs|onesweep|depth_|radix_hist" NCU_S=14 NCU_C=14 NCU_NAME=pp bash tools/ncu_full.sh
