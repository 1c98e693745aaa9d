#!/bin/bash
# Build libsgrpo_b200 variants of the GEMM tuning macros into _build/var_<name>.so
# usage: scripts/build_variants.sh name "-DSGB_KSUB128=2 ..." [name flags]...
set -e
cd "$(dirname "$0")/.."
python -m paper_2509_21792_b200.build > /dev/null
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     --expt-relaxed-constexpr -I include $flags -c paper_2509_21792_b200/csrc/gemm.cu -o /tmp/gemm_$name.o
  objs=$(ls paper_2509_21792_b200/_build/*.o | grep -v gemm.cu.o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2509_21792_b200/_build/var_$name.so $objs /tmp/gemm_$name.o -lnccl
  echo built $name
done
