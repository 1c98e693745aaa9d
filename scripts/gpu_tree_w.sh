#!/bin/bash
# tree-verify attention tile width A/B at low B (SGB_TREE_W = consumer warps per tile)
cd "$(dirname "$0")/.."
for w in 0 1 2 4 8; do
  for shp in "1 211 640 28" "4 52 640 28" "16 13 1100 28" "1 211 2200 28"; do
    echo "W=$w $(SGB_TREE_W=$w python scripts/probes/one_tree_attn.py $shp)"
  done
done | tee gpurun_out/tree_w.txt
