// Acceptance-side sampling and draft top-k over materialised fp32 logit rows.
//
// emit_kernel      -- sample_token (include/sgrpo/tinylm.hpp:591-628): T=0 argmax with the
//                     lowest index on ties (bit-exact given identical logits); T>0 fp64
//                     inverse CDF of exp((l-max)/T) with u = Rng(key).uniform()*sum, key
//                     mix_key(seq_seed, position) derived on device (drafttree.cpp:184-190).
//                     Also flags NaN / all -inf / non-finite rows (tinylm.hpp:460-461,597,601).
// topk_lsm_kernel  -- log_softmax_row<double> (nn.hpp:172-180) + topk_tokens
//                     (drafttree.cpp:20-30): top-k by (value desc, index asc), log-probs in fp64.
// One 256-thread CTA per row; all reductions are in a fixed order.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kT = 256;

struct VI {
    float v;
    int i;
};
__device__ __forceinline__ bool better(const VI& a, const VI& b) { return a.v > b.v || (a.v == b.v && a.i < b.i); }

__device__ VI block_argmax(VI x, VI* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        VI y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o)};
        if (better(y, x)) x = y;
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = x;
    __syncthreads();
    VI b = sh[0];
    for (int i = 1; i < kT / 32; ++i)
        if (better(sh[i], b)) b = sh[i];
    return b;
}

__device__ double block_sum_d(double v, double* sh) {
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kT / 32; ++i) s += sh[i];
    return s;
}

__global__ void __launch_bounds__(kT) emit_kernel(const float* __restrict__ logits, int V,
                                                  const int* __restrict__ row_idx, const unsigned long long* __restrict__ seeds,
                                                  const int* __restrict__ key_pos, double temperature,
                                                  int* __restrict__ out, int* __restrict__ err) {
    pdl_wait();
    pdl_trigger();
    __shared__ VI shv[kT / 32];
    __shared__ double shd[kT / 32];
    __shared__ double chunk_sum[kT];
    const int r = blockIdx.x;
    const float* L = logits + static_cast<size_t>(row_idx ? row_idx[r] : r) * V;
    VI best{-INFINITY, 0x7fffffff};
    bool nan = false, nonfinite = false;
    for (int i = threadIdx.x; i < V; i += kT) {
        const float x = L[i];
        if (x != x) nan = true;
        if (!isfinite(x)) nonfinite = true;
        VI c{x, i};
        if (better(c, best)) best = c;
    }
    const int any_nonfinite = __syncthreads_or(nonfinite);
    const int any_nan = __syncthreads_or(nan);
    if (any_nonfinite && threadIdx.x == 0) atomicOr(err, any_nan ? 3 : 1);
    best = block_argmax(best, shv);
    if (best.v == -INFINITY) {
        if (threadIdx.x == 0) {
            atomicOr(err, 4);
            out[r] = 0;
        }
        return;
    }
    if (temperature == 0.0) {
        if (threadIdx.x == 0) out[r] = best.i;
        return;
    }
    // T > 0: contiguous chunk per thread, sequential fp64 inside, chunks in order.
    const double mx = static_cast<double>(best.v);
    const int C = (V + kT - 1) / kT;
    const int lo = threadIdx.x * C, hi = min(V, lo + C);
    double s = 0.0;
    for (int i = lo; i < hi; ++i) s += exp((static_cast<double>(L[i]) - mx) / temperature);
    chunk_sum[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int t = 0; t < kT; ++t) {
            const double c = chunk_sum[t];
            chunk_sum[t] = acc;  // exclusive prefix
            acc += c;
        }
        const uint64_t key = mix_key(seeds[r], static_cast<uint64_t>(key_pos[r]));
        shd[0] = rng_first_uniform(key) * acc;
    }
    __syncthreads();
    const double u = shd[0];
    // The winner is the last non-empty chunk whose exclusive prefix is <= u; it walks its
    // chunk sequentially (like the reference's single loop) and falls back to its last
    // element if fp rounding leaves u above its walked sum.
    const int cand = (lo < hi && chunk_sum[threadIdx.x] <= u) ? static_cast<int>(threadIdx.x) : -1;
    VI cv{static_cast<float>(cand), cand};
    cv = block_argmax(cv, shv);
    if (static_cast<int>(threadIdx.x) == cv.i) {
        double acc = chunk_sum[threadIdx.x];
        int tok = hi - 1;
        for (int i = lo; i < hi; ++i) {
            acc += exp((static_cast<double>(L[i]) - mx) / temperature);
            if (u < acc) {
                tok = i;
                break;
            }
        }
        out[r] = tok;
    } else if (cv.i < 0 && threadIdx.x == 0) {
        out[r] = V - 1;
    }
}

// Fused log-softmax (fp64) + top-k, k <= 16.
__global__ void __launch_bounds__(kT) topk_lsm_kernel(const float* __restrict__ logits, int V, int k,
                                                      int* __restrict__ out_tok, double* __restrict__ out_lp) {
    pdl_wait();
    pdl_trigger();
    constexpr int KM = 16;
    __shared__ VI cand[kT][KM];
    __shared__ VI shv[kT / 32];
    __shared__ double shd[kT / 32];
    const int r = blockIdx.x;
    const float* L = logits + static_cast<size_t>(r) * V;
    VI loc[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) loc[j] = VI{-INFINITY, 0x7fffffff};
    VI best{-INFINITY, 0x7fffffff};
    for (int i = threadIdx.x; i < V; i += kT) {
        VI c{L[i], i};
        if (better(c, best)) best = c;
        if (better(c, loc[k - 1])) {
            int j = k - 1;
            while (j > 0 && better(c, loc[j - 1])) {
                loc[j] = loc[j - 1];
                --j;
            }
            loc[j] = c;
        }
    }
    best = block_argmax(best, shv);
    const double mx = static_cast<double>(best.v);
    double s = 0.0;
    for (int i = threadIdx.x; i < V; i += kT) s += exp(static_cast<double>(L[i]) - mx);
    const double lse = mx + log(block_sum_d(s, shd));
    for (int j = 0; j < k; ++j) cand[threadIdx.x][j] = loc[j];
    __syncthreads();
    if (threadIdx.x < 32) {
        // k rounds of selection over the 256 sorted lists (8 per lane)
        int head[kT / 32];
#pragma unroll
        for (int t = 0; t < kT / 32; ++t) head[t] = 0;
        for (int j = 0; j < k; ++j) {
            VI b{-INFINITY, 0x7fffffff};
            int bt = -1;
#pragma unroll
            for (int t = 0; t < kT / 32; ++t) {
                const int owner = threadIdx.x + 32 * t;
                if (head[t] < k) {
                    const VI c = cand[owner][head[t]];
                    if (better(c, b)) {
                        b = c;
                        bt = t;
                    }
                }
            }
            VI x = b;
            int xo = bt >= 0 ? static_cast<int>(threadIdx.x) + 32 * bt : -1;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                VI y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o)};
                const int yo = __shfl_xor_sync(0xffffffffu, xo, o);
                if (better(y, x)) {
                    x = y;
                    xo = yo;
                }
            }
            if (xo >= 0 && (xo & 31) == static_cast<int>(threadIdx.x)) head[xo >> 5]++;
            if (threadIdx.x == 0) {
                out_tok[static_cast<size_t>(r) * k + j] = x.i;
                out_lp[static_cast<size_t>(r) * k + j] = static_cast<double>(x.v) - lse;
            }
        }
    }
}

}  // namespace

void launch_emit(const float* logits, int V, const int* row_idx, const unsigned long long* seeds, const int* key_pos,
                 int R, double temperature, int* out, int* err, cudaStream_t st) {
    if (R <= 0) return;
    launch_pdl(emit_kernel, dim3(R), dim3(kT), 0, st, logits, V, row_idx, seeds, key_pos, temperature, out, err);
    SGB_KCHECK();
}

void launch_topk_lsm(const float* logits, int V, int R, int k, int* out_tok, double* out_lp, cudaStream_t st) {
    if (R <= 0) return;
    if (k < 1 || k > 16) throw std::invalid_argument("top-k must be in [1, 16]");
    launch_pdl(topk_lsm_kernel, dim3(R), dim3(kT), 0, st, logits, V, k, out_tok, out_lp);
    SGB_KCHECK();
}

}  // namespace sgb
