#!/bin/bash
# c3r and c5 lines after the attention exponential change
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python bench.py --config c3r --no-cpu-baseline > gpurun_out/final6_bench_c3r.json 2> gpurun_out/final6_bench_c3r.err
echo "c3r rc=$?"; python -c "import json; d=json.load(open('gpurun_out/final6_bench_c3r.json')); print(d['value'], d['tau'], d['speedup_vs_ar'], d['ar']['value'])"
timeout 2400 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-profile > gpurun_out/final6_bench_c5.json 2> gpurun_out/final6_bench_c5.err
echo "c5 rc=$?"; python -c "import json; d=json.load(open('gpurun_out/final6_bench_c5.json')); print(d['value'], d['tau'], d['speedup_vs_ar'], d['ar']['value'], d['ar']['per_concurrency'])"
