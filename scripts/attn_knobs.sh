#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/attn_knobs.jsonl
for env in "" "SGB_ATTN_QW=1" "SGB_ATTN_QW=4" "SGB_ATTN_BOUNDARY=0" "SGB_ATTN_G=32" "SGB_ATTN_G=8" "SGB_ATTN_G=4" "SGB_ATTN_BALANCE=0" "SGB_ATTN_PERSM=2"; do
  env $env python scripts/attn_knobs.py >> gpurun_out/attn_knobs.jsonl 2>&1
done
