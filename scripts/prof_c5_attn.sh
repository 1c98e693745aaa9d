#!/bin/bash
# ncu --set full: c5-shaped verify attention (B=48 x 4 rows, ctx 2048, prefix-shared tiles) vs the AR launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 14 -c 1 \
    -o gpurun_out/c5_verify_group python scripts/probes/one_c5_attn.py verify > gpurun_out/ncu_c5v.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 \
    -o gpurun_out/c5_ar_row python scripts/probes/one_c5_attn.py ar > gpurun_out/ncu_c5a.log 2>&1
ls gpurun_out/*.ncu-rep
