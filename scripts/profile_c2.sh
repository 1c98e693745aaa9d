#!/bin/bash
# ncu evidence for the c2 bench (a short rollout of the same workload shape): the launch list
# (serialised, cold-cache per launch) and full captures of the attention kernel and one
# decoder layer's four GEMMs. Each ncu command runs only after the same command exited 0.
set -x
CMD="python bench.py --steps 1 --warmup 3 --max-new 32 --no-cpu-baseline --no-ar"
$CMD > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 600 --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 300 -c 1 -o gpurun_out/attn_c2 $CMD > gpurun_out/ncu_attn.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 1200 -c 4 -o gpurun_out/gemm_c2 $CMD > gpurun_out/ncu_gemm.log 2>&1
ls -la gpurun_out
