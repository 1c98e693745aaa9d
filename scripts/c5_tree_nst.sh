#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/c5_tree_nst.jsonl
: > $out
for n in 6 4 3 2; do
  echo "{\"env\": \"SGB_TREE_NST=$n\"}" >> $out
  SGB_TREE_NST=$n timeout 300 python scripts/bench_c5_attn.py >> $out 2>&1
  SGB_TREE_NST=$n timeout 300 python scripts/bench_tree_attn2.py >> $out 2>&1
done
cat $out
