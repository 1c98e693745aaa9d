#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_group_attention.py -x -q > gpurun_out/dec_tests.log 2>&1
echo "rc=$?" >> gpurun_out/dec_tests.log
tail -3 gpurun_out/dec_tests.log
grep -q "rc=0" gpurun_out/dec_tests.log || exit 1
timeout 300 python scripts/bench_decode_attn.py > gpurun_out/decode_attn.jsonl 2>&1
cat gpurun_out/decode_attn.jsonl
timeout 600 python scripts/bench_lowb.py 1 4 16 --config=c3 --vanilla > gpurun_out/ar_tail_decode.jsonl 2>&1
cat gpurun_out/ar_tail_decode.jsonl
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/dec_all.log 2>&1
echo "all rc=$?" >> gpurun_out/dec_all.log
tail -3 gpurun_out/dec_all.log
