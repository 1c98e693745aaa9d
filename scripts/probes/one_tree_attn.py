"""One shape of attention_tree.cu's tree-verify kernel (for ncu): B sequences x N rows over ctx keys."""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2509_21792_b200 import capi  # noqa: E402

B, N, ctx, H = (int(x) for x in sys.argv[1:5])
t = C.c_double()
capi.dev_lib().sgb_bench_tree_attention_tree(B, N, ctx, H, 128, 3, C.byref(t))
print(B, N, ctx, H, t.value)
