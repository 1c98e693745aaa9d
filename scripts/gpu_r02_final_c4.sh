#!/bin/bash
# end-of-round lines for c4 (c3 + online draft step with NCCL, per GPU shard) and c3r (T = 1, rejection sampling)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in c4 c3r; do
  timeout 1500 python bench.py --config $c --no-cpu-baseline > gpurun_out/final_bench_$c.json 2> gpurun_out/final_bench_$c.err
  echo "$c rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/final_bench_$c.json')); print(d['value'], d['tau'], d['speedup_vs_ar'], (d.get('ar') or {}).get('value'), d.get('online_draft_step', {}).get('device_ms_per_step'))"
done
