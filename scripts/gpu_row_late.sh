#!/bin/bash
# reduce_residual_ln LATE variant (2 CTAs / SM above 148 rows at d >= 3584): tests + per-step ncu at the c5 shape
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_widths.py tests/test_gpu_rollout.py tests/test_gpu_kernels.py -x -q > gpurun_out/late_tests.log 2>&1
echo "rc=$?" >> gpurun_out/late_tests.log; tail -2 gpurun_out/late_tests.log
for late in 0 1; do
  SGB_ROW_LATE=$late timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:reduce_residual \
      --log-file gpurun_out/row_late$late.csv python scripts/bench_lowb.py 32 --config=c5 --ncu --ctx=2048 --cpeak=256 \
      > gpurun_out/row_late$late.log 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('gpurun_out/row_late$late.csv')) if len(r) > 10]
h=rows[0]; rows=rows[1:]
gi=h.index('Grid Size'); vi=h.index('Metric Value')
big=[float(r[vi]) for r in rows if r[gi].strip('()').split(',')[0].strip() not in ('32','1','2','3')]
import statistics
g=[r[gi] for r in rows]
print('late=$late', len(rows), 'launches; grid sizes', sorted(set(g))[:8])
by={}
for r in rows: by.setdefault(r[gi],[]).append(float(r[vi]))
for k,v in sorted(by.items(), key=lambda x:-len(x[1]))[:6]: print('  grid', k, 'n', len(v), 'median ns', statistics.median(v))
PY
done
