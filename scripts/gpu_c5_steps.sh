#!/bin/bash
# per-launch device times of c5-shaped AR and speculative steps (B = 32 sequences at ~2k keys),
# C_peak 128 -> (N,K,L) = (4,3,1) and 256 -> (8,7,2); split per step by steps_from_launches.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cp in 128 256; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/c5_steps_cp$cp.csv python scripts/bench_lowb.py 32 --config=c5 --ncu --ctx=2048 --cpeak=$cp \
      > gpurun_out/c5_steps_cp$cp.log 2>&1
  echo "cp=$cp rc=$?"
  python scripts/steps_from_launches.py gpurun_out/c5_steps_cp$cp.csv > gpurun_out/c5_steps_cp$cp.txt 2>&1
  tail -12 gpurun_out/c5_steps_cp$cp.txt
done
