#!/bin/bash
# GPU tests after the dev-library split; c2 A/B of single-chunk QKV at d = 1536 (SGB_CHUNK_TILES_MAX=32)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/devlib_tests.log 2>&1; echo "rc=$?" >> gpurun_out/devlib_tests.log
tail -2 gpurun_out/devlib_tests.log
timeout 300 python scripts/bench_attn.py 512:640 > gpurun_out/devlib_bench_attn.txt 2>&1; cat gpurun_out/devlib_bench_attn.txt
for ct in 64 32 64 32; do
  SGB_CHUNK_TILES_MAX=$ct timeout 300 python bench.py --steps 1 --warmup 1 --max-new 512 --no-cpu-baseline --no-ar \
     2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['roofline']['classes']; print('CT=$ct', d['value'], d['ms_per_step'], c['gemm_tcgen05']['ms_per_step'], c['rowops']['ms_per_step'])"
done
