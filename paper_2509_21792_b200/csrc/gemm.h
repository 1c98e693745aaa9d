// Host interface of the tcgen05 GEMM (gemm.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace sgb {

// A K-major bf16 weight [N][K] (device) with its TMA map.
struct GemmWeight {
    const __nv_bfloat16* ptr = nullptr;
    int N = 0, K = 0;
    int chunk_kb = 16;  // accumulation chunk in 64-wide k-blocks (gemm_chunk_kb: fixed per weight shape)
    CUtensorMap map;
    // chunk_kb > 0 overrides the per-shape chunk width (training operands: one chunk, no
    // intermediate TMEM readouts; their numerics need determinism, not batch invariance)
    void init(const __nv_bfloat16* p, int n, int k, int chunk_kb_override = 0);
};

// A bf16 activation buffer [cap_rows][K] with one TMA map per supported token tile.
struct GemmAct {
    const __nv_bfloat16* ptr = nullptr;
    int cap_rows = 0, K = 0;
    CUtensorMap maps[5];
    void init(const __nv_bfloat16* p, int rows, int k);
    const CUtensorMap& map_for_bn(int bn) const;
};

// Fused epilogues applied to the final fp32 sum v of (token row t, output feature o).
enum GemmEpiKind : int {
    kEpiF32 = 0,      // f32[t*ld + o] = v
    kEpiBF16 = 1,     // b16[t*ld + o] = bf16(v)
    kEpiGeluBF16 = 2, // b16[t*ld + o] = bf16(gelu_tanh(v))                  (nn.hpp:128-133)
    kEpiResid = 3,    // x[t*ld + o] += v   (residual stream, fp32)           (tinylm.hpp:396-403)
    kEpiQKV = 4,      // o<d: q[t*d+o]=v; K/V[kv_dst[t]*d + o-d|o-2d] = bf16(v) (tinylm.hpp:325-327,405-408)
    kEpiFusePos = 5,  // x[t*ld + o] = v + pos_emb[pos[t]*ld + o]            (tinylm.hpp:528-533)
    kEpiPartials = 6, // f32[(c*M + t)*ld + o] = raw chunk sum c (one unit per chunk); the row
                      // kernel that follows adds the chunks in order (launch_reduce_residual_ln)
};

struct GemmEpi {
    int kind = kEpiF32;
    float* f32 = nullptr;
    __nv_bfloat16* b16 = nullptr;
    const long long* kv_dst = nullptr;
    __nv_bfloat16* K = nullptr;
    __nv_bfloat16* V = nullptr;
    const float* pos_emb = nullptr;
    const int* pos = nullptr;
    int ld = 0;
    int d = 0;
};

// Split-K workspace: per-tile chunk partials + arrival counters (zeroed once).
struct GemmWorkspace {
    float* buf = nullptr;
    size_t cap_floats = 0;
    int* ctr = nullptr;
    int ctr_cap = 0;
};

// persistent-grid caps (0 = all SMs): a launch of a concurrent lane runs on a subset of the SMs
extern int g_gemm_sm_cap;

CUtensorMap make_kmajor_map(const void* ptr, int rows, int K, int box_rows);
int gemm_bn_for(int M);
int gemm_chunk_kb(int N, int K);
int gemm_chunks(int N, int K);  // chunk count of a weight (rows of a kEpiPartials output)
int gemm_splits_for(int M, int N, int K);
size_t gemm_ws_floats(int M, int N, int K);
void gemm_run(const GemmWeight& w, const GemmAct& x, int M, const GemmEpi& epi, const GemmWorkspace& ws,
              cudaStream_t st, int force_splits = 0);

}  // namespace sgb
