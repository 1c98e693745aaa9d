#!/bin/bash
# c5 verify attention (B=48 x 4 rows, 32 heads): attention.cu launch knobs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/c5_attn_knobs.jsonl
: > $out
for env in "" "SGB_ATTN_MERGE=0" "SGB_ATTN_MERGE=0 SGB_ATTN_G=8" "SGB_ATTN_MERGE=0 SGB_ATTN_G=16" "SGB_ATTN_G=8" "SGB_ATTN_BOUNDARY=0" "SGB_ATTN_MERGE=0 SGB_ATTN_BALANCE=1" "SGB_ATTN_MERGE=0 SGB_ATTN_BALANCE=0" "SGB_ATTN_MERGE=0 SGB_ATTN_MAXSM=6"; do
  echo "{\"env\": \"$env\"}" >> $out
  env $env timeout 300 python scripts/bench_c5_attn.py >> $out 2>&1
done
cat $out
