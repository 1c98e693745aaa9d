#!/bin/bash
# GEMM longest-processing-time placement (129..256 rows, 75..147 single-chunk tiles): bitwise tests, A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_kernels.py -x -q > gpurun_out/lpt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lpt_tests.log
tail -2 gpurun_out/lpt_tests.log
SH="192x12288x4096 160x12288x4096 256x12288x4096 211x10752x3584 160x10752x3584 192x14336x4096 211x18944x3584 192x4608x1536 211x8960x1536"
for l in 0 1 0 1; do
  echo "== SGB_GEMM_LPT=$l"
  SGB_GEMM_LPT=$l SPLITS=0 python scripts/bench_gemm.py $SH
done | tee gpurun_out/gemm_lpt_ab.txt
