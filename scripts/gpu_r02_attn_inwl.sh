#!/bin/bash
# c2 attention inside the benchmarked workload: launch count of an 8-token rollout, then
# ncu --set full of the attention launch at step ~500 (every sequence at ~629 keys), and the
# SGB_PROMPT_TILES A/B of the attention class time.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/attn_traffic_c2.sh count > gpurun_out/attn_count.txt
N8=$(tail -1 gpurun_out/attn_count.txt)
SKIP=$((N8 + 492 * 28))
echo "N8=$N8 SKIP=$SKIP" | tee -a gpurun_out/attn_count.txt
bash scripts/attn_traffic_c2.sh $SKIP
ncu -i gpurun_out/c2_attn_inworkload.ncu-rep --page details > gpurun_out/c2_attn_inworkload.txt 2>&1
ncu -i gpurun_out/c2_attn_inworkload.ncu-rep --page raw --csv > gpurun_out/c2_attn_inworkload_raw.csv 2>&1
for pt in 0 1; do
  SGB_PROMPT_TILES=$pt python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-ar > gpurun_out/c2_pt$pt.json 2>/dev/null
done
