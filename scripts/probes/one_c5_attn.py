import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2509_21792_b200 import capi
lib = capi.dev_lib()
a, b = C.c_double(), C.c_double()
if sys.argv[1] == "verify":
    lib.sgb_bench_tree_attention(48, 4, 2048, 32, 128, 10, C.byref(a), C.byref(b))
else:
    capi.bench_attention_decode(48, 2048, 32, 128, 10)
