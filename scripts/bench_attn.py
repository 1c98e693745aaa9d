"""Decode-attention microbenchmark: achieved HBM GB/s on K/V reads."""
import ctypes as C, sys, json
sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi
lib = capi.lib()
cases = [(512, 128), (512, 640), (512, 1151), (64, 1151), (8, 1151), (1, 1151)]
for B, ctx in cases:
    ms = C.c_double()
    rc = lib.sgb_bench_attention(B, ctx, 12, 128, 20, C.byref(ms))
    if rc:
        print("error", lib.sgb_last_error()); continue
    t = ms.value * 1e-3
    by = B * (ctx + 1) * 1536 * 2 * 2
    print(json.dumps(dict(B=B, ctx=ctx, us=round(ms.value * 1e3, 1), GBps=round(by / t / 1e9, 1))))
