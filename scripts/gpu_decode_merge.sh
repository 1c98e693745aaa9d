#!/bin/bash
# decode attention: batched DSMEM merge over 32 lanes -- bitwise tests, microbenchmark, B=1..16 step costs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/dm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dm_tests.log
tail -2 gpurun_out/dm_tests.log
timeout 600 python scripts/bench_decode_attn.py > gpurun_out/decode_attn_merge.jsonl 2>&1
head -8 gpurun_out/decode_attn_merge.jsonl
timeout 900 python scripts/bench_lowb.py 1 4 16 --config=c3 --vanilla > gpurun_out/lowb_c3_vanilla.jsonl 2>&1
cat gpurun_out/lowb_c3_vanilla.jsonl
