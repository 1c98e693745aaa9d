#!/bin/bash
# attention.cu at the c5 verify shape (B=48 x 4 tree rows, ctx 2200, 32 heads) vs the AR shape:
# ncu --set full of one launch each
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cat > /tmp/one_group.py <<'PY'
import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2509_21792_b200 import capi
mode = sys.argv[1]
a, b = C.c_double(), C.c_double()
if mode == "verify":
    capi.dev_lib().sgb_bench_tree_attention(48, 4, 2200, 32, 128, 2, C.byref(a), C.byref(b))
else:
    capi.dev_lib().sgb_bench_attention(48, 2200, 32, 128, 3, C.byref(a))
PY
timeout 600 ncu --set full --clock-control none -k regex:attn_kernel -s 5 -c 1 -o gpurun_out/grp_verify python /tmp/one_group.py verify > gpurun_out/ncu_grp_verify.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:attn_kernel -s 3 -c 1 -o gpurun_out/grp_ar python /tmp/one_group.py ar > gpurun_out/ncu_grp_ar.log 2>&1
ls gpurun_out/*.ncu-rep
