#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_group_attention.py tests/test_gpu_rollout.py tests/test_gpu_stress.py tests/test_gpu_waves.py tests/test_gpu_reject.py -q -m gpu > gpurun_out/attn_tests.log 2>&1
tail -2 gpurun_out/attn_tests.log
python scripts/attn_knobs.py > gpurun_out/attn_knobs2.jsonl 2>&1
SGB_ATTN_MERGE=0 python scripts/attn_knobs.py >> gpurun_out/attn_knobs2.jsonl 2>&1
cat gpurun_out/attn_knobs2.jsonl
