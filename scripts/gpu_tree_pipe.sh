#!/bin/bash
# attention_tree.cu: software-pipelined prefix chunks (S of chunk c+1 before softmax / P.V of chunk c)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_group_attention.py tests/test_gpu_stress.py tests/test_gpu_rollout.py tests/test_gpu_reject.py -x -q > gpurun_out/pipe_tests.log 2>&1
echo "rc=$?" >> gpurun_out/pipe_tests.log; tail -2 gpurun_out/pipe_tests.log
for shp in "1 211 640 28" "4 52 640 28" "16 13 1100 28" "32 4 2048 32" "48 4 2048 32" "48 8 2048 32" "64 3 1024 28" "1 211 2200 28"; do
  echo "$(python scripts/probes/one_tree_attn.py $shp)"
done | tee gpurun_out/tree_pipe.txt
