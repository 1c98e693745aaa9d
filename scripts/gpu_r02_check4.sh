#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c4_all.log 2>&1
echo "all rc=$?" >> gpurun_out/c4_all.log
tail -3 gpurun_out/c4_all.log
scripts/lowb_r02.sh
