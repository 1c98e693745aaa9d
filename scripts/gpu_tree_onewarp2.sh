#!/bin/bash
# attention_tree.cu one-warp instantiation chosen by waves: GPU tests, microbenchmark A/B, c3 line
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/ow2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ow2_tests.log
tail -2 gpurun_out/ow2_tests.log
for ow in 0 -1; do
  for shp in "32 4 2048 32" "48 4 2048 32" "24 4 2048 32" "32 8 2048 32" "64 3 1024 28" "16 13 1100 28" "1 211 640 28" "4 52 640 28"; do
    echo "ow=$ow $(SGB_TREE_ONE_WARP=$ow python scripts/probes/one_tree_attn.py $shp)"
  done
done | tee gpurun_out/tree_onewarp_ab2.txt
for ow in 0 -1; do
  SGB_TREE_ONE_WARP=$ow timeout 900 python bench.py --config c3 --no-cpu-baseline --no-profile --steps 1 --warmup 1 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 ow=$ow', d['value'], d['tau'], d['speedup_vs_ar'], d['ar']['value'])"
done
