#!/bin/bash
# ncu evidence for the attention kernel at a decode shape (B rows x ctx keys, c2 width).
# usage: scripts/prof_attn.sh B:ctx tag
set -x
python scripts/bench_attn.py $1 > gpurun_out/attn_plain_$2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 -o gpurun_out/attn_$2 \
    python scripts/bench_attn.py $1 > gpurun_out/ncu_attn_$2.log 2>&1
tail -3 gpurun_out/ncu_attn_$2.log
