import ctypes as C, json, sys
sys.path.insert(0, '.')
from paper_2509_21792_b200 import capi
lib = capi.dev_lib()
for M, N, K in [(1, 10752, 3584), (1, 3584, 18944), (1, 3584, 3584), (1, 18944, 3584), (1, 4608, 1536), (1, 8960, 1536), (1, 1536, 8960), (8, 10752, 3584), (8, 3584, 18944)]:
    row = []
    for sp in (1, 2, 3, 4, 5, 6, 8, 12):
        ms = C.c_double()
        if lib.sgb_bench_gemm(M, N, K, sp, 30, C.byref(ms)) == 0:
            row.append((sp, round(ms.value * 1e3, 1)))
    a = C.c_double(); lib.sgb_bench_gemm(M, N, K, 0, 30, C.byref(a))
    print(json.dumps(dict(M=M, N=N, K=K, auto=round(a.value * 1e3, 1), forced=row)), flush=True)
