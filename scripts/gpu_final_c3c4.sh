#!/bin/bash
# c3 and c4 lines on the final code
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c3 c4; do
  timeout 1500 python bench.py --config $c --no-cpu-baseline > gpurun_out/final7_bench_$c.json 2> gpurun_out/final7_bench_$c.err
  echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/final7_bench_$c.json')); print(d['value'], d['e2e']['value'], d['tau'], d['speedup_vs_ar'], (d.get('ar') or {}).get('value'))"
done
