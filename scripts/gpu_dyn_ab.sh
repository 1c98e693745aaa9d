#!/bin/bash
# attention.cu dynamic chunk schedule: GPU tests, microbenchmark and c2 A/B
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/dyn_tests.log 2>&1; echo "rc=$?" >> gpurun_out/dyn_tests.log
tail -3 gpurun_out/dyn_tests.log
for cfg in "0 850" "8 850" "8 700" "16 900" "4 800"; do
  set -- $cfg
  echo "== SGB_ATTN_DYN_M=$1 SGB_ATTN_DYN_F=$2" >> gpurun_out/dyn_ab.txt
  SGB_ATTN_DYN_M=$1 SGB_ATTN_DYN_F=$2 timeout 300 python scripts/bench_attn.py 512:640 512:1151 128:640:28 128:1151:28 >> gpurun_out/dyn_ab.txt 2>&1
  SGB_ATTN_DYN_M=$1 SGB_ATTN_DYN_F=$2 timeout 300 python bench.py --steps 1 --warmup 1 --max-new 512 --no-cpu-baseline --no-ar \
     2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['roofline']['classes']['attention']; print('c2-512', d['value'], d['ms_per_step'], c['ms_per_step'], c['GBps'])" >> gpurun_out/dyn_ab.txt
done
cat gpurun_out/dyn_ab.txt
