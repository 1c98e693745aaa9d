#!/bin/bash
# ncu --set full of one CTA-pair GEMM launch vs the 1-CTA kernel (M=512 N=18944 K=3584, M=211)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for shape in 512x18944x3584 211x18944x3584; do
for pair in 1 0; do
  SGB_GEMM_PAIR=$pair timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 3 -c 1 \
     -o gpurun_out/pair_${pair}_$shape python scripts/bench_gemm.py $shape > gpurun_out/ncu_pair_$pair.log 2>&1
  echo "pair=$pair rc=$?"
done
done
ls gpurun_out/*.ncu-rep
