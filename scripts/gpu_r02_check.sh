#!/bin/bash
# Round-2 GPU check: the full -m gpu suite, the tree-attention microbenchmark, a c3 bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r02_gputest.log 2>&1
tail -3 gpurun_out/r02_gputest.log
python scripts/bench_tree_attn2.py > gpurun_out/r02_tree_attn.jsonl 2>&1
python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_c3.json 2> gpurun_out/r02_bench_c3.err
tail -c 600 gpurun_out/r02_bench_c3.json
