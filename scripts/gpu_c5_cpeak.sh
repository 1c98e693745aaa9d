#!/bin/bash
# c5 controller sensitivity: C_peak above the analytic 211 (deeper trees at the KV-bound long contexts)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cp in 384 768; do
  timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-profile --no-ar --c-peak $cp \
      > gpurun_out/c5_cpeak$cp.json 2> gpurun_out/c5_cpeak$cp.err
  echo "cp=$cp rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/c5_cpeak$cp.json')); print(d['value'], d['tau'], d.get('ar',{}).get('per_concurrency'))"
done
