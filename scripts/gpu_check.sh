#!/bin/bash
# One GPU round trip: probes, parity tests, attention microbenchmarks, per-step costs.
#   gpurun -- bash scripts/gpu_check.sh [quick]
mkdir -p gpurun_out
(cd scripts/probes && [ -x probe_mma ] && timeout 60 ./probe_mma) > gpurun_out/probe_mma.log 2>&1; cat gpurun_out/probe_mma.log
timeout 300 python -m pytest tests/test_gpu_group_attention.py tests/test_gpu_kernels.py -x -q > gpurun_out/t_kernels.log 2>&1; tail -3 gpurun_out/t_kernels.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; tail -3 gpurun_out/t_gpu.log
timeout 300 python scripts/bench_attn.py > gpurun_out/attn_ar.log 2>&1; cat gpurun_out/attn_ar.log
timeout 300 python scripts/bench_tree_attn.py > gpurun_out/tree_attn.log 2>&1; cat gpurun_out/tree_attn.log
[ "$1" = quick ] && exit 0
timeout 600 python scripts/step_costs.py c3 1 4 16 64 > gpurun_out/step_costs.log 2>&1; cat gpurun_out/step_costs.log
