"""AR attention per layer (device ms per launch): attention.cu row path vs the tree kernel vs
the cluster decode kernel, B rows x ctx keys, 7B (28 x 128) and c5 (32 x 128) head shapes.

    python scripts/bench_decode_attn.py
"""
import json
import sys

sys.path.insert(0, ".")
from paper_2509_21792_b200 import capi  # noqa: E402

for H in (28, 32):
    for B in (1, 4, 16, 48):
        for ctx in (200, 640, 2200, 4200):
            r, t, d = capi.bench_attention_decode(B, ctx, H, 128, 20)
            kv = B * ctx * H * 128 * 2 * 2
            print(json.dumps(dict(H=H, B=B, ctx=ctx, row_us=round(r * 1e3, 1), tree_us=round(t * 1e3, 1),
                                  decode_us=round(d * 1e3, 1), decode_GBps=round(kv / (d * 1e-3) / 1e9))), flush=True)
