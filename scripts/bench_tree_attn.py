"""Tree-verify attention: per-row kernel vs prefix-shared group kernel (sgb_bench_tree_attention).

    python scripts/bench_tree_attn.py
Prints per shape: ms per launch of each kernel, algorithmic K/V GB/s of the group kernel
(each sequence's committed K/V read once) and its useful TFLOP/s (4*d flops per row-key).
"""
import ctypes as C
import json
import sys

sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
shapes = [(1, 211, 640), (1, 211, 1100), (4, 52, 640), (16, 13, 640), (16, 13, 1100), (64, 3, 640), (105, 2, 640)]
heads = [(28, 128), (12, 128)]
iters = 20
if len(sys.argv) > 1:  # one shape (profiling): B N ctx H
    B, N, ctx, H = (int(x) for x in sys.argv[1:5])
    shapes, heads, iters = [(B, N, ctx)], [(H, 128)], 2
for H, dh in heads:
    d = H * dh
    for B, N, ctx in shapes:
        a, b = C.c_double(), C.c_double()
        rc = lib.sgb_bench_tree_attention(B, N, ctx, H, dh, iters, C.byref(a), C.byref(b))
        if rc:
            print(json.dumps(dict(H=H, B=B, N=N, ctx=ctx, err=capi.dev_lib().sgb_dev_last_error().decode())))
            continue
        kv = B * (ctx + N) * d * 4
        fl = 4.0 * B * N * (ctx + 4) * d
        print(json.dumps(dict(H=H, B=B, N=N, ctx=ctx, row_ms=round(a.value, 4), group_ms=round(b.value, 4),
                              speedup=round(a.value / b.value, 2), group_kv_GBps=round(kv / b.value / 1e6, 1),
                              group_TFLOPs=round(fl / b.value / 1e9, 2))), flush=True)
