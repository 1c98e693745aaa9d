"""Tree-verify attention at the speculative-step shapes: per-row kernel vs prefix-shared group
kernel (attention.cu) vs attention_tree.cu. Prints one JSON line per shape (ms per layer launch)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
for (B, N, ctx, H, dh) in [(1, 211, 640, 28, 128), (4, 52, 640, 28, 128), (16, 13, 1100, 28, 128),
                           (48, 4, 2200, 32, 128), (1, 211, 640, 12, 128), (64, 3, 640, 12, 128)]:
    a, b, t = C.c_double(), C.c_double(), C.c_double()
    rc = lib.sgb_bench_tree_attention(B, N, ctx, H, dh, 20, C.byref(a), C.byref(b))
    rc2 = lib.sgb_bench_tree_attention_tree(B, N, ctx, H, dh, 20, C.byref(t))
    kv_bytes = B * (ctx + N) * H * dh * 2 * 2
    print(json.dumps({"B": B, "N": N, "ctx": ctx, "H": H, "ms_row": round(a.value, 4), "ms_group": round(b.value, 4),
                      "ms_tree": round(t.value, 4), "rc": [rc, rc2],
                      "tree_GBps_kv": round(kv_bytes / (t.value * 1e-3) / 1e9, 1) if t.value else None}))
