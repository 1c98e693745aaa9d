#!/bin/bash
# the engine's GEMM modes at the BASELINE shapes (default 1-CTA kernel): QKV / w1 / LM head unsplit
# (SPLITS=0), wo / w2 raw chunk partials (SPLITS=-1), M = 1 / 192-211 / 512, cold weights
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
echo "== unsplit (QKV, w1, LM head)"
SPLITS=0 python scripts/bench_gemm.py 512x4608x1536 512x8960x1536 512x151936x1536 512x10752x3584 512x18944x3584 \
  211x10752x3584 211x18944x3584 192x12288x4096 192x14336x4096 1x10752x3584 1x18944x3584 1x152064x3584
echo "== partials (wo, w2)"
SPLITS=-1 python scripts/bench_gemm.py 512x1536x1536 512x1536x8960 512x3584x3584 512x3584x18944 211x3584x3584 \
  211x3584x18944 192x4096x4096 192x4096x14336
echo "== one-token split-K finisher (wo, w2)"
SPLITS=0 python scripts/bench_gemm.py 1x3584x3584 1x3584x18944
} | tee gpurun_out/gemm_table.txt
