// Row-wise kernels of the decode forward: embedding + LayerNorm, split-K reduction with
// fused residual/LayerNorm, GELU or Q/K/V-scatter epilogues, draft fuse-input gather,
// and the weight-layout conversion used at upload.
//
// Reference loops replaced (include/sgrpo/...):
//   tinylm.hpp:442-448  x = tok_emb[t] + pos_emb[p]                 -> embed_ln_kernel
//   nn.hpp:70-98        layernorm_fwd (pop. var, eps 1e-5)          -> block_ln (all kernels)
//   tinylm.hpp:396-403  residual adds after wo / w2                  -> reduce_residual_ln_kernel
//   nn.hpp:128-133      gelu (tanh form)                             -> reduce_gelu_kernel
//   tinylm.hpp:405-412  KV append                                    -> reduce_qkv_kernel (scatter)
//   tinylm.hpp:519-533  draft fuse concat(tok_emb, feature)          -> gather_fuse_kernel
// Every kernel is row-local with a fixed reduction order, so a row's bits do not depend
// on how many rows share the launch (batch invariance, SURVEY.md §7 hard part 1).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kRowThreads = 256;
constexpr int kMaxPerThread = 32;  // d <= 8192

// Fixed-order block sum (warp butterfly, then warp partials summed in warp order).
__device__ float block_sum(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kRowThreads / 32; ++i) s += red[i];
    return s;
}

// LayerNorm of one row held in registers (xs[i] = x[threadIdx.x + i*256]).
template <int PER>
__device__ void block_ln(const float* xs, int d, const float* __restrict__ g, const float* __restrict__ b,
                         __nv_bfloat16* out_bf, float* out_f, float* red) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * kRowThreads;
        if (e < d) s += xs[i];
    }
    const float mu = block_sum(s, red) / static_cast<float>(d);
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * kRowThreads;
        if (e < d) {
            const float dv = xs[i] - mu;
            v += dv * dv;
        }
    }
    const float var = block_sum(v, red) / static_cast<float>(d);
    const float rstd = 1.0f / sqrtf(var + 1e-5f);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * kRowThreads;
        if (e < d) {
            const float y = g[e] * (xs[i] - mu) * rstd + b[e];
            if (out_bf) out_bf[e] = __float2bfloat16(y);
            if (out_f) out_f[e] = y;
        }
    }
}

// Same, gamma/beta already in registers (gs[i] = g[threadIdx.x + i*256]); identical bits.
template <int PER>
__device__ void block_ln_regs(const float* xs, int d, const float* gs, const float* bs, __nv_bfloat16* out_bf,
                              float* out_f, float* red) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * kRowThreads;
        if (e < d) s += xs[i];
    }
    const float mu = block_sum(s, red) / static_cast<float>(d);
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * kRowThreads;
        if (e < d) {
            const float dv = xs[i] - mu;
            v += dv * dv;
        }
    }
    const float var = block_sum(v, red) / static_cast<float>(d);
    const float rstd = 1.0f / sqrtf(var + 1e-5f);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * kRowThreads;
        if (e < d) {
            const float y = gs[i] * (xs[i] - mu) * rstd + bs[i];
            if (out_bf) out_bf[e] = __float2bfloat16(y);
            if (out_f) out_f[e] = y;
        }
    }
}

template <int PER>
__global__ void __launch_bounds__(kRowThreads) embed_ln_kernel(const int* __restrict__ tokens,
                                                             const int* __restrict__ positions, int d,
                                                             const float* __restrict__ tok_emb,
                                                             const float* __restrict__ pos_emb,
                                                             const float* __restrict__ g, const float* __restrict__ b,
                                                             float* __restrict__ x, __nv_bfloat16* __restrict__ a) {
    pdl_wait();
    pdl_trigger();
    __shared__ float red[kRowThreads / 32];
    const int r = blockIdx.x;
    const float* te = tok_emb + static_cast<size_t>(tokens[r]) * d;
    const float* pe = pos_emb + static_cast<size_t>(positions[r]) * d;
    float xs[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = threadIdx.x + i * kRowThreads;
        xs[i] = e < d ? te[e] + pe[e] : 0.f;
        if (e < d) x[static_cast<size_t>(r) * d + e] = xs[i];
    }
    block_ln<PER>(xs, d, g, b, a + static_cast<size_t>(r) * d, nullptr, red);
}

// x = (mode==0 ? 0 : x) + sum_s P[s][r] (+ pos_emb[pos[r]]); then LN -> a (bf16) / y (fp32).
// FR: chunks loaded in the first round (with the residual row); CPR per later round.
// LATE: gamma / beta read at the end (block_ln, identical bits) instead of held in registers from
// before the PDL wait, and two CTAs per SM: for launches of many waves of rows at d >= 3584, where
// the register-resident variant (142-167 registers) runs one CTA per SM
template <int PER, int FR = 4, bool LATE = false>
__global__ void __launch_bounds__(kRowThreads, LATE ? 2 : 1)
    reduce_residual_ln_kernel(const float* __restrict__ P, int S, int M, int d, float* __restrict__ x, int accumulate,
                              const float* __restrict__ pos_emb, const int* __restrict__ positions,
                              const float* __restrict__ g, const float* __restrict__ b, __nv_bfloat16* __restrict__ a,
                              float* __restrict__ y) {
    __shared__ float red[kRowThreads / 32];
    // LN parameters are weights, never written by the previous kernel: load them before the
    // PDL wait, so that a one-row launch (the decode tail) pays one dependent round trip for
    // partials + residual instead of four
    float gs[LATE ? 1 : PER], bs[LATE ? 1 : PER];
    if (g && !LATE) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = threadIdx.x + i * kRowThreads;
            gs[i] = e < d ? g[e] : 0.f;
            bs[i] = e < d ? b[e] : 0.f;
        }
    }
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    float xs[PER];
    const float* pe = pos_emb ? pos_emb + static_cast<size_t>(positions[r]) * d : nullptr;
    const size_t row = static_cast<size_t>(r) * d;
    if (P) {
        // chunk partials, strictly in chunk order per element: acc = P0, acc += P1, ... The
        // first round loads chunks 0..CPR-1 together with the residual row; later rounds load
        // CPR chunks at a time (w2 at the c2 shape has 12 chunks: 3 round trips; eight per
        // round measured slower)
        const size_t st = static_cast<size_t>(M) * d;
        constexpr int CPR = 4;
        float acc[PER], xr[PER];
        {
            const int n0 = min(S, FR);
            float pp[FR][PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = threadIdx.x + i * kRowThreads;
                xr[i] = (accumulate && e < d) ? x[row + e] : 0.f;
            }
#pragma unroll
            for (int c = 0; c < FR; ++c)
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int e = threadIdx.x + i * kRowThreads;
                    pp[c][i] = (c < n0 && e < d) ? P[c * st + row + e] : 0.f;
                }
#pragma unroll
            for (int i = 0; i < PER; ++i) acc[i] = pp[0][i];
#pragma unroll
            for (int c = 1; c < FR; ++c)
                if (c < n0) {
#pragma unroll
                    for (int i = 0; i < PER; ++i) acc[i] += pp[c][i];
                }
        }
        int s = min(S, FR);
        for (; s + CPR <= S; s += CPR) {
            float pp[CPR][PER];
#pragma unroll
            for (int c = 0; c < CPR; ++c)
#pragma unroll
                for (int i = 0; i < PER; ++i) {
                    const int e = threadIdx.x + i * kRowThreads;
                    pp[c][i] = e < d ? P[(s + c) * st + row + e] : 0.f;
                }
#pragma unroll
            for (int c = 0; c < CPR; ++c)
#pragma unroll
                for (int i = 0; i < PER; ++i) acc[i] += pp[c][i];
        }
        for (; s + 2 <= S; s += 2) {
            float p1[PER], p2[PER];
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = threadIdx.x + i * kRowThreads;
                p1[i] = e < d ? P[s * st + row + e] : 0.f;
                p2[i] = e < d ? P[(s + 1) * st + row + e] : 0.f;
            }
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                acc[i] += p1[i];
                acc[i] += p2[i];
            }
        }
        if (s < S) {
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const int e = threadIdx.x + i * kRowThreads;
                acc[i] += e < d ? P[s * st + row + e] : 0.f;
            }
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = threadIdx.x + i * kRowThreads;
            if (e < d) {
                float v = accumulate ? xr[i] + acc[i] : acc[i];
                if (pe) v += pe[e];
                x[row + e] = v;
                xs[i] = v;
            } else {
                xs[i] = 0.f;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int e = threadIdx.x + i * kRowThreads;
            xs[i] = e < d ? x[row + e] : 0.f;  // plain LayerNorm of the residual stream
        }
    }
    if (g) {
        if constexpr (LATE)
            block_ln<PER>(xs, d, g, b, a ? a + static_cast<size_t>(r) * d : nullptr,
                          y ? y + static_cast<size_t>(r) * d : nullptr, red);
        else
            block_ln_regs<PER>(xs, d, gs, bs, a ? a + static_cast<size_t>(r) * d : nullptr,
                               y ? y + static_cast<size_t>(r) * d : nullptr, red);
    }
}

__device__ __forceinline__ float gelu_tanh(float x) {
    const float c = 0.7978845608028654f;
    const float u = c * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.0f + tanhf(u));
}

__global__ void reduce_gelu_kernel(const float* __restrict__ P, int S, int M, int N, __nv_bfloat16* __restrict__ out) {
    const size_t total = static_cast<size_t>(M) * N;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float acc = P[i];
        for (int s = 1; s < S; ++s) acc += P[static_cast<size_t>(s) * total + i];
        out[i] = __float2bfloat16(gelu_tanh(acc));
    }
}

__global__ void reduce_plain_kernel(const float* __restrict__ P, int S, int M, int N, float* __restrict__ out) {
    const size_t total = static_cast<size_t>(M) * N;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float acc = P[i];
        for (int s = 1; s < S; ++s) acc += P[static_cast<size_t>(s) * total + i];
        out[i] = acc;
    }
}

// qkv partials [S][M][3d] -> q fp32 [M][d]; K, V bf16 into cache slots kv_dst[r].
__global__ void reduce_qkv_kernel(const float* __restrict__ P, int S, int M, int d, float* __restrict__ q,
                                  __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                                  const long long* __restrict__ kv_dst) {
    const int N = 3 * d;
    const size_t total = static_cast<size_t>(M) * N;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        float acc = P[i];
        for (int s = 1; s < S; ++s) acc += P[static_cast<size_t>(s) * total + i];
        const int r = static_cast<int>(i / N);
        const int c = static_cast<int>(i - static_cast<size_t>(r) * N);
        if (c < d) {
            q[static_cast<size_t>(r) * d + c] = acc;
        } else if (c < 2 * d) {
            kc[kv_dst[r] * d + (c - d)] = __float2bfloat16(acc);
        } else {
            vc[kv_dst[r] * d + (c - 2 * d)] = __float2bfloat16(acc);
        }
    }
}

// Draft fuse input (tinylm.hpp:519-527): out[r] = bf16(concat(tok_emb[tok[r]], feat_ptr[r])).
__global__ void gather_fuse_kernel(const int* __restrict__ tokens, const long long* __restrict__ feat_off,
                                   const float* __restrict__ feat_base, const float* __restrict__ tok_emb, int d,
                                   __nv_bfloat16* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    const float* te = tok_emb + static_cast<size_t>(tokens[r]) * d;
    const float* fe = feat_base + feat_off[r];
    __nv_bfloat16* o = out + static_cast<size_t>(r) * 2 * d;
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
        o[e] = __float2bfloat16(te[e]);
        o[d + e] = __float2bfloat16(fe[e]);
    }
}

// Reference [in][out] fp32 -> device [out][in] bf16 at row offset (tiled transpose).
__global__ void transpose_to_bf16_kernel(const float* __restrict__ src, int in, int out_dim,
                                         __nv_bfloat16* __restrict__ dst, int dst_ld) {
    __shared__ float tile[32][33];
    const int i0 = blockIdx.y * 32, o0 = blockIdx.x * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = i0 + k, o = o0 + threadIdx.x;
        tile[k][threadIdx.x] = (i < in && o < out_dim) ? src[static_cast<size_t>(i) * out_dim + o] : 0.f;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int o = o0 + k, i = i0 + threadIdx.x;
        if (o < out_dim && i < in) dst[static_cast<size_t>(o) * dst_ld + i] = __float2bfloat16(tile[threadIdx.x][k]);
    }
}

__global__ void gather_rows_bf16_kernel(const __nv_bfloat16* __restrict__ src, const int* __restrict__ idx, int d,
                                        __nv_bfloat16* __restrict__ dst) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    const __nv_bfloat16* s = src + static_cast<size_t>(idx[r]) * d;
    for (int e = threadIdx.x; e < d; e += blockDim.x) dst[static_cast<size_t>(r) * d + e] = s[e];
}

// Random-normal fill (benchmark weights; splitmix64 counter + Box-Muller, deterministic).
__global__ void init_normal_kernel(float* __restrict__ out, size_t n, unsigned long long seed, float std_) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        uint64_t s = seed ^ (0x632BE59BD9B4E019ULL * (i >> 1));
        const double u1 = (static_cast<double>(splitmix64_next(s) >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(splitmix64_next(s) >> 11) * 0x1.0p-53;
        const double r = sqrt(-2.0 * log(u1));
        const double th = 6.283185307179586 * u2;
        out[i] = static_cast<float>(std_ * ((i & 1) ? r * sin(th) : r * cos(th)));
    }
}

__global__ void fill_kernel(float* __restrict__ out, size_t n, float v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = v;
}

int grid_for(size_t n, int threads) {
    size_t b = (n + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

#define SGB_PER_DISPATCH(d, KERNEL, ...)                                                 \
    do {                                                                                 \
        if ((d) <= 256) KERNEL<1><<<__VA_ARGS__>>>;                                      \
        else if ((d) <= 1024) KERNEL<4><<<__VA_ARGS__>>>;                                \
        else if ((d) <= 1536) KERNEL<6><<<__VA_ARGS__>>>;                                \
        else if ((d) <= 2048) KERNEL<8><<<__VA_ARGS__>>>;                                \
        else if ((d) <= 3584) KERNEL<14><<<__VA_ARGS__>>>;                               \
        else if ((d) <= 4096) KERNEL<16><<<__VA_ARGS__>>>;                               \
        else KERNEL<kMaxPerThread><<<__VA_ARGS__>>>;                                     \
    } while (0)

void launch_embed_ln(const int* tokens, const int* positions, int M, int d, const float* tok_emb, const float* pos_emb,
                     const float* g, const float* b, float* x, __nv_bfloat16* a, cudaStream_t st) {
    if (M <= 0) return;
    if (d > kMaxPerThread * kRowThreads) throw std::invalid_argument("d_model too large");
#define ARGS , dim3(M), dim3(kRowThreads), 0, st, tokens, positions, d, tok_emb, pos_emb, g, b, x, a
    if (d <= 256) launch_pdl(embed_ln_kernel<1> ARGS);
    else if (d <= 1024) launch_pdl(embed_ln_kernel<4> ARGS);
    else if (d <= 1536) launch_pdl(embed_ln_kernel<6> ARGS);  // exact per-thread counts: fewer registers
    else if (d <= 2048) launch_pdl(embed_ln_kernel<8> ARGS);
    else if (d <= 3584) launch_pdl(embed_ln_kernel<14> ARGS);
    else if (d <= 4096) launch_pdl(embed_ln_kernel<16> ARGS);
    else launch_pdl(embed_ln_kernel<kMaxPerThread> ARGS);
#undef ARGS
    SGB_KCHECK();
}

void launch_reduce_residual_ln(const float* P, int S, int M, int d, float* x, bool accumulate, const float* pos_emb,
                               const int* positions, const float* g, const float* b, __nv_bfloat16* a, float* y,
                               cudaStream_t st) {
    if (M <= 0) return;
#define ARGS , dim3(M), dim3(kRowThreads), 0, st, P, S, M, d, x, accumulate ? 1 : 0, pos_emb, positions, g, b, a, y
    if (d <= 256) launch_pdl(reduce_residual_ln_kernel<1> ARGS);
    else if (d <= 1024) launch_pdl(reduce_residual_ln_kernel<4> ARGS);
    else if (d <= 1536) {  // exact per-thread counts: fewer registers
        static const int fr = [] {
            // A/B: chunks in the first load round. Measured at c2 (profiles/r01_row_fr_c2.txt):
            // 6 -> 45.1 k tok/s, rowops 682 ms/step; 4 -> 44.9 k, 798 ms; 12 -> 43.6 k (162
            // registers: one CTA per SM)
            const char* v = getenv("SGB_ROW_FR");
            return v ? atoi(v) : 6;
        }();
        if (fr >= 12) launch_pdl(reduce_residual_ln_kernel<6, 12> ARGS);
        else if (fr >= 6) launch_pdl(reduce_residual_ln_kernel<6, 6> ARGS);
        else launch_pdl(reduce_residual_ln_kernel<6> ARGS);
    }
    else if (d <= 2048) launch_pdl(reduce_residual_ln_kernel<8> ARGS);
    else if (d <= 4096) {
        // many waves of rows (prefill chunks): the two-CTA-per-SM LATE variant (same bits).
        // Measured (profiles/r02_row_late_ab.txt, c5 width): 2,048 rows 66.5 -> 51.2 us, but
        // 151-256 rows 10.7-11.6 -> 14.1-14.5 us, so it starts at 1,024 rows
        static const int late_env = [] {
            const char* v = getenv("SGB_ROW_LATE");  // A/B: 0 = never, N = from N rows
            return v ? atoi(v) : 1024;
        }();
        const bool late = late_env > 0 && M >= late_env;
        if (d <= 3584) {
            static const int fr14 = [] {
                const char* v = getenv("SGB_ROW_FR14");  // A/B: 5 = the 7B wo / w2 partials in one trip
                return v ? atoi(v) : 4;
            }();
            if (late) launch_pdl(reduce_residual_ln_kernel<14, 4, true> ARGS);
            else if (fr14 >= 5) launch_pdl(reduce_residual_ln_kernel<14, 5> ARGS);
            else launch_pdl(reduce_residual_ln_kernel<14> ARGS);
        } else {
            if (late) launch_pdl(reduce_residual_ln_kernel<16, 4, true> ARGS);
            else launch_pdl(reduce_residual_ln_kernel<16> ARGS);
        }
    }
    else launch_pdl(reduce_residual_ln_kernel<kMaxPerThread> ARGS);
#undef ARGS
    SGB_KCHECK();
}

void launch_reduce_gelu(const float* P, int S, int M, int N, __nv_bfloat16* out, cudaStream_t st) {
    if (M <= 0) return;
    reduce_gelu_kernel<<<grid_for(static_cast<size_t>(M) * N, 256), 256, 0, st>>>(P, S, M, N, out);
    SGB_KCHECK();
}

void launch_reduce_plain(const float* P, int S, int M, int N, float* out, cudaStream_t st) {
    if (M <= 0) return;
    reduce_plain_kernel<<<grid_for(static_cast<size_t>(M) * N, 256), 256, 0, st>>>(P, S, M, N, out);
    SGB_KCHECK();
}

void launch_reduce_qkv(const float* P, int S, int M, int d, float* q, __nv_bfloat16* kc, __nv_bfloat16* vc,
                       const long long* kv_dst, cudaStream_t st) {
    if (M <= 0) return;
    reduce_qkv_kernel<<<grid_for(static_cast<size_t>(M) * 3 * d, 256), 256, 0, st>>>(P, S, M, d, q, kc, vc, kv_dst);
    SGB_KCHECK();
}

void launch_gather_fuse(const int* tokens, const long long* feat_off, const float* feat_base, const float* tok_emb,
                        int R, int d, __nv_bfloat16* out, cudaStream_t st) {
    if (R <= 0) return;
    launch_pdl(gather_fuse_kernel, dim3(R), dim3(256), 0, st, tokens, feat_off, feat_base, tok_emb, d, out);
    SGB_KCHECK();
}

void launch_transpose_to_bf16(const float* src, int in, int out_dim, __nv_bfloat16* dst, int dst_ld,
                              cudaStream_t st) {
    dim3 grid((out_dim + 31) / 32, (in + 31) / 32);
    transpose_to_bf16_kernel<<<grid, dim3(32, 8), 0, st>>>(src, in, out_dim, dst, dst_ld);
    SGB_KCHECK();
}

void launch_gather_rows_bf16(const __nv_bfloat16* src, const int* idx, int R, int d, __nv_bfloat16* dst,
                             cudaStream_t st) {
    if (R <= 0) return;
    launch_pdl(gather_rows_bf16_kernel, dim3(R), dim3(256), 0, st, src, idx, d, dst);
    SGB_KCHECK();
}

void launch_init_normal(float* out, size_t n, unsigned long long seed, float std_, cudaStream_t st) {
    init_normal_kernel<<<grid_for(n, 256), 256, 0, st>>>(out, n, seed, std_);
    SGB_KCHECK();
}

void launch_fill(float* out, size_t n, float v, cudaStream_t st) {
    fill_kernel<<<grid_for(n, 256), 256, 0, st>>>(out, n, v);
    SGB_KCHECK();
}

}  // namespace sgb
