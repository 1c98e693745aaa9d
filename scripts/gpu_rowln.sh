#!/bin/bash
# Round trip after the row-kernel change: GPU tests, low-B step costs (7B shape), c2 + c3 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/rl_gpu.log 2>&1; tail -3 gpurun_out/rl_gpu.log
timeout 600 python scripts/bench_lowb.py 1 4 16 --config=c3 > gpurun_out/rl_lowb.log 2>&1; cut -c1-130 gpurun_out/rl_lowb.log
timeout 600 python bench.py > gpurun_out/rl_bench_c2.log 2>&1; grep '^{' gpurun_out/rl_bench_c2.log | tail -1 | cut -c1-200
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/rl_bench_c3.log 2>&1; grep '^{' gpurun_out/rl_bench_c3.log | tail -1 | cut -c1-200
