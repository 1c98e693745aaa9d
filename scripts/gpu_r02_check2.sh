#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r02_gputest2.log 2>&1
tail -3 gpurun_out/r02_gputest2.log
bash scripts/sanitize.sh
python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
tail -c 400 gpurun_out/r02_bench_c2.json
