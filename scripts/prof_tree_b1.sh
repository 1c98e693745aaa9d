#!/bin/bash
# ncu --set full (+ source) of attention_tree.cu at B = 1 x 211 rows x 640 keys x 28 heads (latency-bound)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/probes/one_tree_attn.py 1 211 640 28 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 2 -c 1 \
    -o gpurun_out/tree_b1 python scripts/probes/one_tree_attn.py 1 211 640 28 > gpurun_out/ncu_tree_b1.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/tree_b1.ncu-rep --page details > gpurun_out/tree_b1_details.txt 2>&1
ncu -i gpurun_out/tree_b1.ncu-rep --page source --csv > gpurun_out/tree_b1_source.csv 2>&1
ncu -i gpurun_out/tree_b1.ncu-rep --page raw --csv > gpurun_out/tree_b1_raw.csv 2>&1
ls -la gpurun_out/tree_b1*
