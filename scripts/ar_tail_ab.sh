#!/bin/bash
# AR tail (7B shape, B = 1 / 4 / 16): attention.cu vs attention_tree.cu for AR steps of few rows
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in 0 64; do
  SGB_TREE_AR_MAX=$v timeout 600 python scripts/bench_lowb.py 1 4 16 --config=c3 --vanilla | sed "s/^/{\"tree_ar_max\": $v, \"r\": /; s/$/}/"
done > gpurun_out/ar_tail_ab.jsonl 2>&1
cat gpurun_out/ar_tail_ab.jsonl
