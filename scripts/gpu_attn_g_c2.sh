#!/bin/bash
# c2 attention head grouping A/B (SGB_ATTN_G: heads split into G groups per item; default = most resident warps)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for g in 0 2 3 4; do
  if [ $g = 0 ]; then unset SGB_ATTN_G; else export SGB_ATTN_G=$g; fi
  echo "G=$g $(python scripts/bench_attn.py 512:640 512:1151 | tr '\n' ' ')"
  timeout 300 python bench.py --steps 1 --warmup 1 --max-new 512 --no-cpu-baseline --no-ar 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['roofline']['classes']['attention']; print('  c2-512 G=$g', d['value'], c['ms_per_step'], c['GBps'])"
done | tee gpurun_out/attn_g_c2.txt
