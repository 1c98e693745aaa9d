#!/bin/bash
# Two-lane AR steps: bitwise tests, the overlap microbenchmark and c2 A/B (short rollouts).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_lanes.py -x -q > gpurun_out/lanes_test.log 2>&1; echo "rc=$?" >> gpurun_out/lanes_test.log
tail -2 gpurun_out/lanes_test.log
timeout 600 python scripts/bench_overlap.py > gpurun_out/overlap.jsonl 2>&1
cat gpurun_out/overlap.jsonl
for L in "0" "256" "256,100,48" "256,110,38" "256,90,58" "256,100,48,0" "256,0,0,0"; do
  echo "== lanes $L" >> gpurun_out/lanes_c2.txt
  timeout 300 python bench.py --steps 1 --warmup 1 --max-new 512 --no-cpu-baseline --no-ar --no-profile --lanes $L \
     2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" >> gpurun_out/lanes_c2.txt
done
cat gpurun_out/lanes_c2.txt
