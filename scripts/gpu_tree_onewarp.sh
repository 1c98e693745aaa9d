#!/bin/bash
# attention_tree.cu one-warp instantiation (7 CTAs per SM): bitwise tests and A/B at the c5 / c3 verify shapes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_group_attention.py tests/test_gpu_stress.py -x -q > gpurun_out/ow_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ow_tests.log
tail -2 gpurun_out/ow_tests.log
for ow in 0 1 0 1; do
  for shp in "32 4 2048 32" "48 4 2048 32" "48 4 4096 32" "32 6 2048 32" "48 8 2048 32" "16 13 1100 28" "64 3 1024 28"; do
    echo "ow=$ow $(SGB_TREE_ONE_WARP=$ow python scripts/probes/one_tree_attn.py $shp)"
  done
done | tee gpurun_out/tree_onewarp_ab.txt
