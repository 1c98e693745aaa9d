#!/bin/bash
# end-of-round c3 / c3r / c4 lines with the final code (per-B tables label each bucket's most frequent plan)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c3 c3r c4; do
  timeout 1500 python bench.py --config $c --no-cpu-baseline > gpurun_out/final4_bench_$c.json 2> gpurun_out/final4_bench_$c.err
  echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/final4_bench_$c.json')); print(d['value'], d['tau'], d['speedup_vs_ar'], (d.get('ar') or {}).get('value'))"
done
