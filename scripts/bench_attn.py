"""Decode-attention microbenchmark: achieved HBM GB/s on K/V reads.

    python scripts/bench_attn.py [B:ctx ...]
"""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
# B:ctx[:H] (H heads of 128; default 12 = the c2 width, 28 = c3/c4)
cases = [tuple(int(x) for x in a.split(':')) for a in sys.argv[1:]] or \
    [(512, 128), (512, 640), (512, 1151), (211, 150), (64, 1151), (16, 150), (8, 1151), (1, 150), (1, 1151),
     (128, 640, 28), (128, 1151, 28), (16, 1151, 28), (1, 1151, 28)]
for case in cases:
    B, ctx = case[0], case[1]
    H = case[2] if len(case) > 2 else 12
    ms = C.c_double()
    rc = lib.sgb_bench_attention(B, ctx, H, 128, 20, C.byref(ms))
    if rc:
        print("error", lib.sgb_dev_last_error())
        continue
    t = ms.value * 1e-3
    by = B * (ctx + 1) * H * 128 * 2 * 2
    print(json.dumps(dict(B=B, ctx=ctx, H=H, us=round(ms.value * 1e3, 1), GBps=round(by / t / 1e9, 1))), flush=True)
