#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_reject.py tests/test_gpu_waves.py tests/test_gpu_rollout.py -x -q -s > gpurun_out/rc_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/rc_tests.log
timeout 600 python scripts/bench_lowb.py 4 16 --config=c3r > gpurun_out/r02_step_costs_c3r_cluster.jsonl 2>&1
scripts/prof_steps.sh c3r
head -8 gpurun_out/rc_tests.log; tail -3 gpurun_out/rc_tests.log; cat gpurun_out/r02_step_costs_c3r_cluster.jsonl
