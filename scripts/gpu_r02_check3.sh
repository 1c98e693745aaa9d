#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c3_all.log 2>&1
echo "all rc=$?" >> gpurun_out/c3_all.log
tail -3 gpurun_out/c3_all.log
timeout 600 python scripts/bench_lowb.py 1 4 16 --config=c3 --vanilla > gpurun_out/ar_tail_final.jsonl 2>&1
timeout 600 python scripts/bench_lowb.py 4 16 --config=c3r > gpurun_out/c3r_steps_final.jsonl 2>&1
cat gpurun_out/ar_tail_final.jsonl gpurun_out/c3r_steps_final.jsonl
