#!/bin/bash
# ncu --set full (+ source) of attention_tree.cu at the c5 verify shapes where it trails the AR launch
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python scripts/probes/one_tree_attn.py 32 4 2048 32 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_attn -s 2 -c 1 \
    -o gpurun_out/tree_c5_32_4 python scripts/probes/one_tree_attn.py 32 4 2048 32 > gpurun_out/ncu_tree_c5.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/tree_c5_32_4.ncu-rep --page details > gpurun_out/tree_c5_32_4_details.txt 2>&1
ncu -i gpurun_out/tree_c5_32_4.ncu-rep --page source --csv > gpurun_out/tree_c5_32_4_source.csv 2>&1
ncu -i gpurun_out/tree_c5_32_4.ncu-rep --page raw --csv > gpurun_out/tree_c5_32_4_raw.csv 2>&1
ls -la gpurun_out/tree_c5_32_4*
