#!/bin/bash
# ncu --set full of one attention launch INSIDE the c2 bench workload (step 500 of the rollout,
# every sequence at 629 context keys): `roofline.traffic` from the benchmarked workload itself.
#   pass 1 (count): scripts/attn_traffic_c2.sh count   -> launch list of an 8-token rollout
#   pass 2:         scripts/attn_traffic_c2.sh SKIP    -> capture launch SKIP (0-based) of attn_kernel
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ "$1" = "count" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_kernel --csv \
      --log-file gpurun_out/c2_attn_count.csv python bench.py --steps 1 --warmup 0 --max-new 8 \
      --no-cpu-baseline --no-ar --no-profile > gpurun_out/c2_attn_count.log 2>&1
  grep -c attn_kernel gpurun_out/c2_attn_count.csv
else
  timeout 2400 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s $1 -c 1 \
      -o gpurun_out/c2_attn_inworkload python bench.py --steps 1 --warmup 0 --max-new 512 \
      --no-cpu-baseline --no-ar --no-profile > gpurun_out/c2_attn_inworkload.log 2>&1
  echo rc=$?
  ls -la gpurun_out/c2_attn_inworkload.ncu-rep
fi
