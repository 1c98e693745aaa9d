#!/bin/bash
# c5 at its stated size (BASELINE configs[4]): one timed rollout after one warm-up, AR beside it
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 3000 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-profile \
    > gpurun_out/r02_bench_c5_final.json 2> gpurun_out/r02_bench_c5_final.err
echo "rc=$?"
tail -c 600 gpurun_out/r02_bench_c5_final.json
