#!/bin/bash
# Boundary-block rule check: group-attention parity, GPU suite, tree-verify A/B, c3 + c2 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/bnd2_gpu.log 2>&1; tail -3 gpurun_out/bnd2_gpu.log
for b in 0 1; do echo "== SGB_ATTN_BOUNDARY=$b"; for sh in "1 211 680 28" "1 211 640 28" "4 52 700 28" "16 13 680 28" "16 13 1100 28" "16 13 1100 12" "16 13 680 12"; do SGB_ATTN_BOUNDARY=$b timeout 300 python scripts/bench_tree_attn.py $sh; done; done > gpurun_out/bnd2_tree.log 2>&1; cut -c1-160 gpurun_out/bnd2_tree.log
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bnd2_bench_c3.log 2>&1; grep '^{' gpurun_out/bnd2_bench_c3.log | tail -1 | cut -c1-120
timeout 600 python bench.py > gpurun_out/bnd2_bench_c2.log 2>&1; grep '^{' gpurun_out/bnd2_bench_c2.log | tail -1 | cut -c1-120
