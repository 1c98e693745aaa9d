#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_driver.py
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --target-processes all python scripts/sanitize_driver.py \
      > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.txt
  tail -3 gpurun_out/sanitizer_$tool.txt
done
