#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_group_attention.py tests/test_gpu_rollout.py tests/test_gpu_stress.py -q -m gpu > gpurun_out/merge_tests.log 2>&1
tail -2 gpurun_out/merge_tests.log
: > gpurun_out/attn_merge.jsonl
for env in "SGB_ATTN_MERGE=0" "SGB_ATTN_MERGE=1" "SGB_ATTN_MERGE=1 SGB_ATTN_QW=1"; do
  env $env python scripts/attn_knobs.py >> gpurun_out/attn_merge.jsonl 2>&1
done
cat gpurun_out/attn_merge.jsonl
