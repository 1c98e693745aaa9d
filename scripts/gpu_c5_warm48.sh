#!/bin/bash
# c5 with a longer online warm-up of the draft (48 iterations x 4 AdamW steps), C_peak 211 and 384, AR beside the first
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 2400 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-profile --warm-iters 48 \
    > gpurun_out/c5_warm48.json 2> gpurun_out/c5_warm48.err
echo "cp211 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c5_warm48.json')); print(d['value'], d['tau'], d['speedup_vs_ar'], d['ar']['value'], d['draft_warm'])"
timeout 2400 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-profile --warm-iters 48 --c-peak 384 --no-ar \
    > gpurun_out/c5_warm48_cp384.json 2> gpurun_out/c5_warm48_cp384.err
echo "cp384 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/c5_warm48_cp384.json')); print(d['value'], d['tau'], d['draft_warm'])"
