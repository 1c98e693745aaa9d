#!/bin/bash
# per-launch device times (ncu launch list) of short rollouts, AR then spec: the sum of kernel
# times per step against the unprofiled ms_per_step separates kernel time from launch gaps.
#   scripts/prof_steps.sh [config] [B] [extra bench_lowb args]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfg=${1:-c3r}
B=${2:-4}
shift 2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_steps_$cfg.csv python scripts/bench_lowb.py $B --config=$cfg --ncu "$@" \
    > gpurun_out/launches_steps_$cfg.log 2>&1
echo rc=$? >> gpurun_out/launches_steps_$cfg.log
wc -l gpurun_out/launches_steps_$cfg.csv
