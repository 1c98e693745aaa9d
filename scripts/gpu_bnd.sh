#!/bin/bash
# Round trip after the boundary-block attention change: group-attention parity first (bit-exact
# vs the per-row kernel), full GPU suite, tree-verify microbench A/B, low-B step costs, c3 bench.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_group_attention.py -x -q > gpurun_out/bnd_grp.log 2>&1; tail -15 gpurun_out/bnd_grp.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/bnd_gpu.log 2>&1; tail -15 gpurun_out/bnd_gpu.log
for b in 0 1; do echo "== SGB_ATTN_BOUNDARY=$b"; for sh in "1 211 680 28" "1 211 640 28" "4 52 700 28" "16 13 680 28" "16 13 1100 12"; do SGB_ATTN_BOUNDARY=$b timeout 300 python scripts/bench_tree_attn.py $sh; done; done > gpurun_out/bnd_tree.log 2>&1; cat gpurun_out/bnd_tree.log | cut -c1-250
for b in 0 1; do echo "== SGB_ATTN_BOUNDARY=$b"; SGB_ATTN_BOUNDARY=$b timeout 600 python scripts/bench_lowb.py 1 4 16 --config=c3; done > gpurun_out/bnd_lowb.log 2>&1; cut -c1-130 gpurun_out/bnd_lowb.log
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bnd_bench_c3.log 2>&1; grep '^{' gpurun_out/bnd_bench_c3.log | tail -1 | cut -c1-200
