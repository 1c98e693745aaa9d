#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stress.py -x -q > gpurun_out/w_stress.log 2>&1; tail -15 gpurun_out/w_stress.log
SPLITS=-1,0 timeout 300 python scripts/bench_gemm.py 211x3584x18944 211x3584x3584 211x10752x3584 211x18944x3584 > gpurun_out/w_gemm211.log 2>&1; cat gpurun_out/w_gemm211.log
timeout 1500 python bench.py --config c5 --no-cpu-baseline > gpurun_out/w_bench_c5.log 2>&1; grep '^{' gpurun_out/w_bench_c5.log | tail -1 | cut -c1-160
