#!/bin/bash
# attention chunk exponentials on the SFU (__expf): every GPU test, then the attention microbenchmarks
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/fastexp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fastexp_tests.log
tail -3 gpurun_out/fastexp_tests.log
{
for shp in "1 211 640 28" "4 52 640 28" "16 13 1100 28" "32 4 2048 32" "48 4 2048 32" "1 211 2200 28"; do
  echo "tree $(python scripts/probes/one_tree_attn.py $shp)"
done
python scripts/bench_attn.py 512:640 512:1151 128:640:28 128:1151:28
python scripts/bench_decode_attn.py | grep '"B": [14],'
} | tee gpurun_out/fastexp_bench.txt
