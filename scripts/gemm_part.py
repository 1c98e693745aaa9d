"""Partial-mode (kEpiPartials) GEMMs at the residual shapes: time vs token tile."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
for M in (65, 128, 160, 211, 256, 384, 512):
    for N, K in ((1536, 1536), (1536, 8960), (3584, 3584), (3584, 18944)):
        r = {}
        for sp in (-1, 0):
            ms = C.c_double()
            if lib.sgb_bench_gemm(M, N, K, sp, 30, C.byref(ms)) == 0:
                r["partials" if sp < 0 else "finisher"] = round(ms.value * 1e3, 1)
        print(json.dumps(dict(M=M, N=N, K=K, **r)), flush=True)
