#!/bin/bash
# decode attention merge A/B in one process pool: SGB_DECODE_MERGE=0 (one block per DSMEM trip) vs 1 (batched)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_group_attention.py -x -q > gpurun_out/dm2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dm2_tests.log
tail -2 gpurun_out/dm2_tests.log
for m in 0 1 0 1; do
  echo "== SGB_DECODE_MERGE=$m" >> gpurun_out/decode_merge_ab.jsonl
  SGB_DECODE_MERGE=$m timeout 600 python scripts/bench_decode_attn.py 2>&1 | grep '"B": [14],' >> gpurun_out/decode_merge_ab.jsonl
done
cat gpurun_out/decode_merge_ab.jsonl
