"""GEMM variant sweep (cold weights): the c2 decode/verify shapes x token counts x splits.
    SGB_LIB=paper_2509_21792_b200/_build/var_X.so python scripts/gemm_sweep.py"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
var = os.path.basename(os.environ.get("SGB_LIB", "default"))
tot = {}
for M in (1, 16, 160, 211, 512):
    best_sum = 0.0
    for N, K in ((4608, 1536), (1536, 1536), (8960, 1536), (1536, 8960)):
        res = {}
        for sp in (0, 1, 2, 3, 6):
            ms = C.c_double()
            if lib.sgb_bench_gemm(M, N, K, sp, 30, C.byref(ms)):
                continue
            res[sp] = round(ms.value * 1e3, 1)
        best = min(res.values())
        best_sum += best
        print(json.dumps(dict(var=var, M=M, N=N, K=K, us=res, best=best)), flush=True)
    tot[M] = round(best_sum, 1)
print(json.dumps(dict(var=var, layer_us_best=tot)), flush=True)
