#!/bin/bash
# A/B of the row kernel's first-round width at d = 3584 (7B): SGB_ROW_FR14=4/5.
mkdir -p gpurun_out
SGB_ROW_FR14=5 timeout 600 python -m pytest tests/test_gpu_stress.py -x -q 2>&1 | tail -1
for fr in 4 5; do echo "== SGB_ROW_FR14=$fr"; SGB_ROW_FR14=$fr timeout 300 python scripts/bench_lowb.py 1 16 --config=c3 --vanilla | cut -c1-80; SGB_ROW_FR14=$fr timeout 900 python bench.py --config c3 --no-cpu-baseline | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ar']['value'], d['roofline']['classes']['rowops'])"; done > gpurun_out/fr14.log 2>&1; cat gpurun_out/fr14.log
