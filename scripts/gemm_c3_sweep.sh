#!/bin/bash
# c3 (7B-shape) GEMMs at decode / verify row counts: pipelined (PDL) device time per launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/gemm_c3_sweep.jsonl
: > $out
for M in 1 4 16 64 211; do
  SPLITS=0 python scripts/bench_gemm.py ${M}x10752x3584 ${M}x18944x3584 ${M}x152064x3584 >> $out 2>&1
  SPLITS=-1,0 python scripts/bench_gemm.py ${M}x3584x3584 ${M}x3584x18944 >> $out 2>&1
done
cat $out
