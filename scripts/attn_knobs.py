"""A/B of attention.cu's tiling knobs at the c5 verify shape (B=48 x 4 tree rows, ctx 2200, 32 heads)
and the AR shape (48 rows) -- run once per environment setting by scripts/attn_knobs.sh."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_21792_b200 import capi  # noqa: E402

lib = capi.dev_lib()
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("SGB_")}}
for (B, N, ctx, H) in [(48, 4, 2200, 32), (1, 211, 640, 28), (16, 13, 1100, 28)]:
    a, b, t = C.c_double(), C.c_double(), C.c_double()
    lib.sgb_bench_tree_attention(B, N, ctx, H, 128, 20, C.byref(a), C.byref(b))
    lib.sgb_bench_tree_attention_tree(B, N, ctx, H, 128, 20, C.byref(t))
    out[f"tree_B{B}_N{N}"] = {"row": round(a.value, 4), "group": round(b.value, 4), "tree": round(t.value, 4)}
m = C.c_double()
lib.sgb_bench_attention(48, 2200, 32, 128, 20, C.byref(m))
out["ar_B48_ctx2200"] = round(m.value, 4)
lib.sgb_bench_attention(1, 640, 28, 128, 20, C.byref(m))
out["ar_B1_ctx640"] = round(m.value, 4)
print(json.dumps(out))
