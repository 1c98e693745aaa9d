"""c5-shaped attention per layer (32 heads x 128, long generated contexts, no prompt sharing):
verify rows N per sequence through the per-row / prefix-shared group (attention.cu) / tree
kernels, against the AR decode of the same B x ctx. ms per launch."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
for (B, N, ctx) in [(32, 6, 2048), (48, 4, 2048), (48, 4, 4096), (32, 2, 4096), (64, 3, 1024), (48, 8, 2048)]:
    a, b, t = C.c_double(), C.c_double(), C.c_double()
    lib.sgb_bench_tree_attention(B, N, ctx, 32, 128, 10, C.byref(a), C.byref(b))
    lib.sgb_bench_tree_attention_tree(B, N, ctx, 32, 128, 10, C.byref(t))
    r, tt, dd = capi.bench_attention_decode(B, ctx, 32, 128, 10)
    kv = B * ctx * 32 * 128 * 2 * 2
    print(json.dumps({"B": B, "N": N, "ctx": ctx, "verify_row": round(a.value, 3), "verify_group": round(b.value, 3),
                      "verify_tree": round(t.value, 3), "ar_row": round(r, 3), "ar_decode": round(dd, 3),
                      "ar_GBps": round(kv / (r * 1e-3) / 1e9)}), flush=True)
