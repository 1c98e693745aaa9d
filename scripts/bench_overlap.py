"""Two-lane concurrency microbenchmark (sgb_bench_overlap): one decoder layer's attention on
one stream and its four GEMMs on another, each on a capped persistent grid.

    python scripts/bench_overlap.py [B ctx H dff M]
"""
import json
import sys

sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi  # noqa: E402

B, ctx, H, dff, M = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (256, 640, 12, 8960, 256)
full = capi.bench_overlap(2 * B, ctx, H, dff, 2 * M, 0, 0)
print(json.dumps(dict(case="full batch, serial", B=2 * B, M=2 * M, attn_ms=round(full[0], 4), gemm_ms=round(full[1], 4),
                      serial_ms=round(full[0] + full[1], 4))), flush=True)
for ac, gc in [(0, 0), (148, 148), (128, 20), (120, 28), (110, 38), (100, 48), (90, 58), (80, 68), (64, 84)]:
    a, g, both = capi.bench_overlap(B, ctx, H, dff, M, ac, gc)
    print(json.dumps(dict(B=B, ctx=ctx, H=H, M=M, attn_cap=ac, gemm_cap=gc, attn_ms=round(a, 4), gemm_ms=round(g, 4),
                          both_ms=round(both, 4), two_halves_ms=round(2 * both, 4))), flush=True)
