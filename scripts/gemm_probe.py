"""GEMM latency anatomy: one 128-row weight tile per CTA (S=1), varying CTA count and K.
time(K) - time(K0) isolates the streaming rate of one SM; the intercept is the fixed cost."""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
for K in (512, 1536, 4096, 8960):
    for tiles in (1, 8, 37, 74, 148):
        ms = C.c_double()
        lib.sgb_bench_gemm(16, 128 * tiles, K, 1, 50, C.byref(ms))
        us = ms.value * 1e3
        per_cta = 128 * K * 2
        print(json.dumps(dict(K=K, ctas=tiles, us=round(us, 2), MB_per_cta=round(per_cta / 1e6, 3),
                              GBps_per_sm=round(per_cta / (us * 1e-6) / 1e9, 1))), flush=True)
