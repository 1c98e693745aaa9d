#!/bin/bash
# per-launch device times (ncu launch list) of short c3r rollouts at B=4, AR then spec: the sum of
# kernel times per step against the unprofiled ms_per_step separates kernel time from launch gaps
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfg=${1:-c3r}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_steps_$cfg.csv python scripts/bench_lowb.py 4 --config=$cfg --ncu \
    > gpurun_out/launches_steps_$cfg.log 2>&1
echo rc=$? >> gpurun_out/launches_steps_$cfg.log
wc -l gpurun_out/launches_steps_$cfg.csv
