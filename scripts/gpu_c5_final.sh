#!/bin/bash
# c5 at its stated per-GPU shard with AR beside it (the end-of-round c5 line)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests/test_gpu_group_attention.py -x -q 2>&1 | tail -1
timeout 3000 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-profile \
    > gpurun_out/final_bench_c5.json 2> gpurun_out/final_bench_c5.err
echo "rc=$?"
python -c "import json; d=json.load(open('gpurun_out/final_bench_c5.json')); print(d['value'], d['tau'], d['speedup_vs_ar'], d['ar']['value'], d.get('host_loop'))"
