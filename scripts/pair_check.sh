#!/bin/bash
# CTA-pair GEMM: numerics + batch invariance first (short timeouts: a barrier bug hangs), then
# the full GPU suite and the c3 shape sweep against the 1-CTA kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_kernels.py -x -q -k gemm > gpurun_out/pair_gemm.log 2>&1
echo "gemm tests rc=$?" >> gpurun_out/pair_gemm.log
tail -5 gpurun_out/pair_gemm.log
grep -q "rc=0" gpurun_out/pair_gemm.log || exit 1
out=gpurun_out/gemm_pair_sweep.jsonl
: > $out
for pair in 1 0; do
  for M in 128 211 512; do
    SGB_GEMM_PAIR=$pair SPLITS=0 timeout 120 python scripts/bench_gemm.py ${M}x10752x3584 ${M}x18944x3584 ${M}x4608x1536 ${M}x8960x1536 | sed "s/^/{\"pair\": $pair, \"r\": /; s/$/}/" >> $out 2>&1
    SGB_GEMM_PAIR=$pair SPLITS=-1 timeout 120 python scripts/bench_gemm.py ${M}x3584x3584 ${M}x3584x18944 ${M}x1536x1536 ${M}x1536x8960 | sed "s/^/{\"pair\": $pair, \"r\": /; s/$/}/" >> $out 2>&1
  done
done
cat $out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pair_all.log 2>&1
echo "all rc=$?" >> gpurun_out/pair_all.log
tail -5 gpurun_out/pair_all.log
