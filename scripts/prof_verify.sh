#!/bin/bash
# ncu evidence for the compute-bound head of a speculative step at the 7B shape (c3, B=1):
# the four layer GEMMs at M=211 verify rows (isolated, cold weights) and the tree-verify
# attention launch (1 sequence x 211 tree rows x 640 committed keys). Each ncu command runs
# only after the same command exited 0 without ncu.
set -x
G="211x10752x3584 211x3584x3584 211x18944x3584 211x3584x18944"
python scripts/bench_gemm.py $G > gpurun_out/verify_gemm_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/verify_gemm_qkv python scripts/bench_gemm.py 211x10752x3584 > gpurun_out/ncu_vg1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/verify_gemm_w1 python scripts/bench_gemm.py 211x18944x3584 > gpurun_out/ncu_vg3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/verify_gemm_w2 python scripts/bench_gemm.py 211x3584x18944 > gpurun_out/ncu_vg4.log 2>&1
python scripts/bench_tree_attn.py 1 211 640 28 > gpurun_out/verify_attn_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 3 -c 1 -o gpurun_out/verify_attn python scripts/bench_tree_attn.py 1 211 640 28 > gpurun_out/ncu_va.log 2>&1
ls gpurun_out
