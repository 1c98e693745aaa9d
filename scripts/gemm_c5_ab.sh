#!/bin/bash
# verify / AR GEMM shapes at c5 (M = 192 verify rows, 48 AR rows): default tiling vs 128-token tiles
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SH="192x12288x4096 192x4096x4096 192x14336x4096 192x4096x14336 48x12288x4096 48x14336x4096 384x12288x4096"
for env in "" "SGB_GEMM_MAXBN=128"; do
  echo "== $env" >> gpurun_out/gemm_c5_ab.jsonl
  env $env SPLITS=0 python scripts/bench_gemm.py $SH >> gpurun_out/gemm_c5_ab.jsonl 2>&1
  env $env SPLITS=-1 python scripts/bench_gemm.py 192x4096x4096 192x4096x14336 >> gpurun_out/gemm_c5_ab.jsonl 2>&1
done
cat gpurun_out/gemm_c5_ab.jsonl
