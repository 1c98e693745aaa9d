#!/bin/bash
# A/B of the residual/LN row kernel's first-round width at the c2 shape (d = 1536): SGB_ROW_FR=4/6/12.
mkdir -p gpurun_out
for fr in 6 12; do SGB_ROW_FR=$fr timeout 600 python -m pytest tests/test_gpu_rollout.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -1; done > gpurun_out/fr_tests.log; cat gpurun_out/fr_tests.log
for fr in 4 6 12 4; do echo "== SGB_ROW_FR=$fr"; SGB_ROW_FR=$fr timeout 600 python bench.py --no-cpu-baseline | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['classes']['rowops'])"; done > gpurun_out/fr_bench.log 2>&1; cat gpurun_out/fr_bench.log
