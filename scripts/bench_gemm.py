"""GEMM microbenchmark (cold weights: copies rotate past L2): achieved TB/s and TFLOP/s.

    python scripts/bench_gemm.py                # c2 shapes x M sweep, auto split vs S=1
    python scripts/bench_gemm.py 211x1536x8960  # explicit MxNxK
    SPLITS=-1,0 python scripts/bench_gemm.py ...  # -1 = kEpiPartials (raw chunk sums, the engine's wo/w2)
"""
import os
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
shapes = [tuple(int(a) for a in s.split('x')) for s in sys.argv[1:]]
if not shapes:
    for M in (1, 16, 64, 128, 211, 256, 512):
        for N, K in ((4608, 1536), (1536, 1536), (8960, 1536), (1536, 8960), (151936, 1536)):
            shapes.append((M, N, K))
for M, N, K in shapes:
    for sp in [int(v) for v in os.environ.get("SPLITS", "0,1").split(",")]:
        ms = C.c_double()
        rc = lib.sgb_bench_gemm(M, N, K, sp, 30, C.byref(ms))
        if rc:
            print("error", lib.sgb_dev_last_error())
            continue
        t = ms.value * 1e-3
        by = 2 * N * K + 2 * M * K + 4 * M * N
        print(json.dumps(dict(M=M, N=N, K=K, splits=sp, us=round(ms.value * 1e3, 1),
                              TBps=round(by / t / 1e12, 2), TFLOPs=round(2 * M * N * K / t / 1e12, 1))), flush=True)
