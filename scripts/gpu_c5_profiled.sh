#!/bin/bash
# c5 line with the kernel-class split (one extra, profiled rollout after the timed one)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 3300 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/final5_bench_c5.json 2> gpurun_out/final5_bench_c5.err
echo "rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/final5_bench_c5.json'))
print(d['value'], d['tau'], d['speedup_vs_ar'], d['ar']['value'])
for k,v in d['roofline']['classes'].items(): print(k, v)"
