// Host interface of the tcgen05 GEMM (gemm.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace sgb {

// A K-major bf16 weight [N][K] (device) with its TMA map and its fixed K split.
struct GemmWeight {
    const __nv_bfloat16* ptr = nullptr;
    int N = 0, K = 0, splits = 1;
    CUtensorMap map;
    void init(const __nv_bfloat16* p, int n, int k);
};

// A bf16 activation buffer [cap_rows][K] with one TMA map per supported token tile.
struct GemmAct {
    const __nv_bfloat16* ptr = nullptr;
    int cap_rows = 0, K = 0;
    CUtensorMap maps[5];
    void init(const __nv_bfloat16* p, int rows, int k);
    const CUtensorMap& map_for_bn(int bn) const;
};

CUtensorMap make_kmajor_map(const void* ptr, int rows, int K, int box_rows);
int gemm_splits(int N, int K);
int gemm_bn_for(int M);
// partials: [w.splits][M][w.N] fp32
void gemm_launch(const GemmWeight& w, const GemmAct& x, float* partials, int M, cudaStream_t st);

}  // namespace sgb
