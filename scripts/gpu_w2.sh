#!/bin/bash
# Round trip after a GEMM change: GPU tests, one-token 7B GEMMs, low-B step costs, c3 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/w2_gpu.log 2>&1; tail -3 gpurun_out/w2_gpu.log
timeout 300 python scripts/bench_gemm.py 1x3584x18944 1x3584x7168 16x3584x18944 211x3584x18944 1x4096x14336 > gpurun_out/w2_gemm.log 2>&1; cat gpurun_out/w2_gemm.log
timeout 600 python scripts/bench_lowb.py 1 4 16 64 --config=c3 > gpurun_out/w2_lowb.log 2>&1; cut -c1-200 gpurun_out/w2_lowb.log
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/w2_bench_c3.log 2>&1; tail -c 400 gpurun_out/w2_bench_c3.log
