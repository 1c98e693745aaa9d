// Acceptance-side sampling and draft top-k over materialised fp32 logit rows.
//
// emit_*_kernel  -- sample_token (include/sgrpo/tinylm.hpp:591-628): T=0 argmax with the
//                   lowest index on ties (bit-exact given identical logits); T>0 fp64 inverse
//                   CDF of exp((l-max)/T) with u = Rng(key).uniform()*sum, key
//                   mix_key(seq_seed, position) derived on device (drafttree.cpp:184-190).
//                   Also flags NaN / all -inf / non-finite rows (tinylm.hpp:460-461,597,601).
// topk_kernel    -- log_softmax_row<double> (nn.hpp:172-180) + topk_tokens
//                   (drafttree.cpp:20-30): top-k by (value desc, index asc), log-probs in fp64.
//
// A row of V logits (608 KB at V=152k) is cut into fixed chunks of kCH = 8192 logits, one
// 256-thread CTA per (chunk, row), so a single row streams at HBM rate instead of one SM's
// bandwidth. Each CTA reduces its chunk and publishes a record; the last CTA of the row to
// arrive (atomic ticket) merges the records in chunk order. Chunking depends only on V,
// never on the number of rows, so every row's result is independent of the batch it is in
// (the speculative and AR rollouts call these with different row counts).
#include <cfloat>

#include "common.cuh"
#include "glibc_exp.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kT = 256;
constexpr int kCH = 8192;          // logits per CTA
constexpr int kPer = kCH / kT;     // 32 per thread
constexpr int kMaxK = 16;
constexpr int kMaxChunks = 64;     // V <= 524288

struct VI {
    float v;
    int i;
};
__device__ __forceinline__ bool better(const VI& a, const VI& b) { return a.v > b.v || (a.v == b.v && a.i < b.i); }

__device__ __forceinline__ VI warp_best(VI x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        VI y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o)};
        if (better(y, x)) x = y;
    }
    return x;
}

__device__ VI block_best(VI x, VI* sh) {
    x = warp_best(x);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = x;
    __syncthreads();
    VI b = sh[0];
#pragma unroll
    for (int i = 1; i < kT / 32; ++i)
        if (better(sh[i], b)) b = sh[i];
    return b;
}

// fixed-order block sum: warp trees, then warps 0..7 in order
__device__ double block_sum_d(double v, double* sh) {
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) sh[w] = v;
    __syncthreads();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kT / 32; ++i) s += sh[i];
    return s;
}

// Last-arriver ticket: true in every thread of the CTA that completes row r.
__device__ __forceinline__ bool last_of_row(int* ctr, int r, int P, int* flag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int old = atomicAdd(&ctr[r], 1);
        *flag = (old == P - 1);
        if (old == P - 1) ctr[r] = 0;  // re-armed for the next launch
    }
    __syncthreads();
    const bool last = *flag;
    if (last) __threadfence();
    return last;
}

// Coalesced chunk load: element j of thread t is logit base + j*kT + t (-inf / INT_MAX pad).
__device__ __forceinline__ void load_chunk(const float* L, int V, int base, float (&v)[kPer]) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int i = base + j * kT + static_cast<int>(threadIdx.x);
        v[j] = i < V ? __ldcs(L + i) : -INFINITY;
    }
}

// ------------------------------------------------------------------ top-k + log-softmax
struct TopkRec {
    double m, s;        // chunk max, sum exp(l - m)
    VI top[kMaxK];      // chunk top-k, best first
};

__global__ void __launch_bounds__(kT) topk_kernel(const float* __restrict__ logits, int V, int k, int P,
                                                  TopkRec* __restrict__ rec, int* __restrict__ ctr,
                                                  int* __restrict__ out_tok, double* __restrict__ out_lp) {
    pdl_wait();
    pdl_trigger();
    __shared__ VI shv[kT / 32];
    __shared__ double shd[kT / 32];
    __shared__ int flag;
    const int p = blockIdx.x, r = blockIdx.y;
    const int base = p * kCH;
    const float* L = logits + static_cast<size_t>(r) * V;
    float v[kPer];
    load_chunk(L, V, base, v);
    // chunk max
    float m = -INFINITY;
#pragma unroll
    for (int j = 0; j < kPer; ++j) m = fmaxf(m, v[j]);
    VI mb = block_best(VI{m, 0}, shv);
    const double md = static_cast<double>(mb.v);
    double s = 0.0;
    if (mb.v != -INFINITY) {
#pragma unroll
        for (int j = 0; j < kPer; ++j) s += exp(static_cast<double>(v[j]) - md);
    }
    s = block_sum_d(s, shd);
    TopkRec* my = rec + static_cast<size_t>(r) * P + p;
    // chunk top-k: k rounds of block argmax; the owner retires its element (a bit mask, so
    // -inf logits are taken in index order like any other value)
    unsigned taken = 0u;
    for (int t = 0; t < k; ++t) {
        VI b{-INFINITY, 0x7fffffff};
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int i = base + j * kT + static_cast<int>(threadIdx.x);
            const VI c{v[j], i};
            if (i < V && !((taken >> j) & 1u) && better(c, b)) b = c;
        }
        b = block_best(b, shv);
        if (b.i != 0x7fffffff && ((b.i - base) & (kT - 1)) == static_cast<int>(threadIdx.x))
            taken |= 1u << ((b.i - base) / kT);
        if (threadIdx.x == 0) my->top[t] = b;
    }
    if (threadIdx.x == 0) {
        my->m = md;
        my->s = s;
    }
    if (!last_of_row(ctr, r, P, &flag)) return;
    if (threadIdx.x >= 32) return;
    // merge: lane l owns chunks l and l+32
    const TopkRec* rr = rec + static_cast<size_t>(r) * P;
    double M = -INFINITY;
    for (int q = 0; q < P; ++q) M = fmax(M, __ldcg(&rr[q].m));
    double S = 0.0;
    if (threadIdx.x == 0)
        for (int q = 0; q < P; ++q) {
            const double mq = __ldcg(&rr[q].m);
            if (mq != -INFINITY) S += __ldcg(&rr[q].s) * exp(mq - M);
        }
    S = __shfl_sync(0xffffffffu, S, 0);
    const double lse = M + log(S);
    int h0 = 0, h1 = 0;
    const int l = threadIdx.x;
    for (int t = 0; t < k; ++t) {
        VI b{-INFINITY, 0x7fffffff};
        int src = -1;
        if (l < P && h0 < k) {
            const VI c{__ldcg(&rr[l].top[h0].v), __ldcg(&rr[l].top[h0].i)};
            if (better(c, b)) {
                b = c;
                src = 0;
            }
        }
        if (l + 32 < P && h1 < k) {
            const VI c{__ldcg(&rr[l + 32].top[h1].v), __ldcg(&rr[l + 32].top[h1].i)};
            if (better(c, b)) {
                b = c;
                src = 1;
            }
        }
        const VI w = warp_best(b);
        if (src >= 0 && w.i == b.i && w.v == b.v) {
            if (src == 0) ++h0;
            else ++h1;
        }
        if (l == 0) {
            out_tok[static_cast<size_t>(r) * k + t] = w.i;
            out_lp[static_cast<size_t>(r) * k + t] = static_cast<double>(w.v) - lse;
        }
    }
}

// ------------------------------------------------------------------ emission
struct EmitRec {
    VI best;
    int flags;  // 1 non-finite, 2 NaN
    double s;   // T>0: chunk sum of exp((l - max)/T)
};

// Max / argmax is order-free, so a CTA takes kCPC chunks (32 K logits, float4 loads) and
// the row's last CTA merges ceil(P / kCPC) records.
constexpr int kCPC = 4;

__global__ void __launch_bounds__(kT) emit_max_kernel(const float* __restrict__ logits, int V, int Pc,
                                                      const int* __restrict__ row_idx, double temperature,
                                                      EmitRec* __restrict__ rec, int* __restrict__ ctr,
                                                      float* __restrict__ rowmax, int* __restrict__ out,
                                                      int* __restrict__ err) {
    pdl_wait();
    pdl_trigger();
    __shared__ VI shv[kT / 32];
    __shared__ int flag;
    const int q = blockIdx.x, r = blockIdx.y;
    const int lo = q * kCPC * kCH, hi = min(V, lo + kCPC * kCH);
    const float* L = logits + static_cast<size_t>(row_idx ? row_idx[r] : r) * V;
    VI best{-INFINITY, 0x7fffffff};
    bool nan = false, nonfinite = false;
    auto see = [&](float x, int i) {
        if (x != x) nan = true;
        if (!isfinite(x)) nonfinite = true;
        const VI c{x, i};
        if (better(c, best)) best = c;
    };
    if ((V & 3) == 0) {
        const float4* L4 = reinterpret_cast<const float4*>(L);
#pragma unroll 4
        for (int i4 = lo / 4 + static_cast<int>(threadIdx.x); i4 < hi / 4; i4 += kT) {
            const float4 x = __ldcs(L4 + i4);
            see(x.x, 4 * i4);
            see(x.y, 4 * i4 + 1);
            see(x.z, 4 * i4 + 2);
            see(x.w, 4 * i4 + 3);
        }
    } else {
#pragma unroll 8
        for (int i = lo + static_cast<int>(threadIdx.x); i < hi; i += kT) see(__ldcs(L + i), i);
    }
    const int any_nonfinite = __syncthreads_or(nonfinite);
    const int any_nan = __syncthreads_or(nan);
    best = block_best(best, shv);
    if (threadIdx.x == 0) {
        EmitRec* my = rec + static_cast<size_t>(r) * (Pc * kCPC) + q;
        my->best = best;
        my->flags = (any_nonfinite ? 1 : 0) | (any_nan ? 2 : 0);
    }
    if (!last_of_row(ctr, r, Pc, &flag)) return;
    if (threadIdx.x != 0) return;
    const EmitRec* rr = rec + static_cast<size_t>(r) * (Pc * kCPC);
    VI b{-INFINITY, 0x7fffffff};
    int fl = 0;
    for (int k = 0; k < Pc; ++k) {
        const VI c{__ldcg(&rr[k].best.v), __ldcg(&rr[k].best.i)};
        fl |= __ldcg(&rr[k].flags);
        if (better(c, b)) b = c;
    }
    if (fl) atomicOr(err, (fl & 2) ? 3 : 1);
    if (b.v == -INFINITY) {
        atomicOr(err, 4);
        out[r] = 0;
        rowmax[r] = -INFINITY;
        return;
    }
    rowmax[r] = b.v;
    if (temperature == 0.0) out[r] = b.i;
}

// T > 0. Every CDF term is glibc's exp of (l - max) / T, bit for bit (glibc_exp.cuh), so the
// only difference to the reference's sequential fp64 sum is the summation ORDER: thread t of
// chunk p sums its kPer contiguous logits sequentially, then threads in order, then chunks in
// order. Summing n non-negative terms in any order is within (n - 1) * 2^-53 * S of the exact
// sum, so the reference's prefixes P'_i and u' = U * S' differ from ours by less than
// (2V + 1024) * 2^-53 * S (first order). The draw is taken from the fast path only when u lies
// more than kMarginUlps(V) * 2^-53 * S (twice that bound) inside the chosen token's interval
// [P_{i-1}, P_i); otherwise the row is flagged and emit_exact_kernel redoes it with the
// reference's own sequential order (tinylm.hpp:614-627), which then gives the same bits.
__device__ __forceinline__ double margin_bound(int V, double S) { return (4.0 * V + 4096.0) * 0x1p-53 * S; }

__device__ const uint64_t kExpTab[256] = SGB_GLIBC_EXP_TAB;

__device__ __forceinline__ void load_exp_tab(uint64_t* sh) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = kExpTab[i];
    __syncthreads();
}

__device__ __forceinline__ double thread_expsum(const float* L, int V, int lo, double mx, double temperature,
                                                const uint64_t* tab) {
    double s = 0.0;
    const int hi = min(V, lo + kPer);
    for (int i = lo; i < hi; ++i) s = __dadd_rn(s, gx::cdf_term(L[i], mx, temperature, tab));
    return s;
}

__device__ __forceinline__ double row_uniform(const unsigned long long* seeds, const int* key_pos,
                                              const double* uniforms, int r) {
    if (uniforms) return uniforms[r];
    return rng_first_uniform(mix_key(seeds[r], static_cast<uint64_t>(key_pos[r])));
}

__global__ void __launch_bounds__(kT) emit_sample_kernel(const float* __restrict__ logits, int V, int P,
                                                         const int* __restrict__ row_idx,
                                                         const unsigned long long* __restrict__ seeds,
                                                         const int* __restrict__ key_pos,
                                                         const double* __restrict__ uniforms, double temperature,
                                                         EmitRec* __restrict__ rec, int* __restrict__ ctr,
                                                         const float* __restrict__ rowmax, int* __restrict__ out,
                                                         int* __restrict__ exact) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint64_t tab[256];
    __shared__ double ts[kT];
    __shared__ VI shv[kT / 32];
    __shared__ int flag;
    __shared__ double sh_u, sh_S;
    __shared__ int sh_p;
    const int p = blockIdx.x, r = blockIdx.y;
    const float mxf = rowmax[r];
    if (mxf == -INFINITY) {  // emit_max flagged the row (domain_error)
        if (p == 0 && threadIdx.x == 0) exact[r] = 0;
        return;
    }
    load_exp_tab(tab);
    const double mx = static_cast<double>(mxf);
    const float* L = logits + static_cast<size_t>(row_idx ? row_idx[r] : r) * V;
    const int lo = p * kCH + static_cast<int>(threadIdx.x) * kPer;
    ts[threadIdx.x] = thread_expsum(L, V, lo, mx, temperature, tab);
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int t = 0; t < kT; ++t) acc = __dadd_rn(acc, ts[t]);
        rec[static_cast<size_t>(r) * (((P + kCPC - 1) / kCPC) * kCPC) + p].s = acc;
    }
    if (!last_of_row(ctr, r, P, &flag)) return;
    const EmitRec* rr = rec + static_cast<size_t>(r) * (((P + kCPC - 1) / kCPC) * kCPC);
    if (threadIdx.x == 0) {
        // chunk prefixes in order; the winner chunk is the last non-empty one whose
        // exclusive prefix is <= u
        double acc = 0.0;
        for (int q = 0; q < P; ++q) acc = __dadd_rn(acc, __ldcg(&rr[q].s));
        const double u = __dmul_rn(row_uniform(seeds, key_pos, uniforms, r), acc);
        double pre = 0.0;
        int win = 0;
        for (int q = 0; q < P; ++q) {
            if (pre <= u) win = q;
            pre = __dadd_rn(pre, __ldcg(&rr[q].s));
        }
        double wpre = 0.0;
        for (int q = 0; q < win; ++q) wpre = __dadd_rn(wpre, __ldcg(&rr[q].s));
        sh_u = u;
        sh_S = acc;
        ts[0] = wpre;  // reused below after the barrier
        sh_p = win;
    }
    __syncthreads();
    const double u = sh_u;
    const int win = sh_p;
    const double cpre = ts[0];
    __syncthreads();
    // recompute the winner chunk's per-thread sums (same arithmetic, same bits)
    const int wlo = win * kCH + static_cast<int>(threadIdx.x) * kPer;
    ts[threadIdx.x] = thread_expsum(L, V, wlo, mx, temperature, tab);
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = cpre;
        for (int t = 0; t < kT; ++t) {
            const double c = ts[t];
            ts[t] = acc;  // exclusive prefix of thread t (chunk prefix included)
            acc = __dadd_rn(acc, c);
        }
    }
    __syncthreads();
    const bool nonempty = wlo < V;
    const int cand = (nonempty && ts[threadIdx.x] <= u) ? static_cast<int>(threadIdx.x) : -1;
    VI cv{static_cast<float>(cand), cand};
    cv = block_best(cv, shv);
    if (static_cast<int>(threadIdx.x) == cv.i) {
        double acc = ts[threadIdx.x];
        const int hi = min(V, wlo + kPer);
        int tok = -1;
        double margin = 0.0;
        for (int i = wlo; i < hi; ++i) {
            const double before = acc;
            acc = __dadd_rn(acc, gx::cdf_term(L[i], mx, temperature, tab));
            if (u < acc) {
                tok = i;
                margin = fmin(u - before, acc - u);
                break;
            }
        }
        const bool sure = tok >= 0 && margin > margin_bound(V, sh_S);
        out[r] = tok >= 0 ? tok : V - 1;
        exact[r] = sure ? 0 : 1;
    } else if (cv.i < 0 && threadIdx.x == 0) {
        out[r] = V - 1;
        exact[r] = 1;
    }
}

// The rows flagged above, redone exactly as sample_token does (tinylm.hpp:614-627): the
// terms in index order into ONE sequential fp64 sum, u = uniform * sum, then the sequential
// walk to the first prefix above u. Terms are computed by the whole CTA into shared memory,
// the additions (the only order-sensitive step) by one thread. Rare by construction (the
// probability that u lands inside the margin is ~1e-10 per row), so its serial cost is moot;
// unflagged rows exit at once.
constexpr int kExT = 256;
constexpr int kExChunk = 4096;

__global__ void __launch_bounds__(kExT) emit_exact_kernel(const float* __restrict__ logits, int V,
                                                          const int* __restrict__ row_idx,
                                                          const unsigned long long* __restrict__ seeds,
                                                          const int* __restrict__ key_pos,
                                                          const double* __restrict__ uniforms, double temperature,
                                                          const float* __restrict__ rowmax, int* __restrict__ out,
                                                          int* __restrict__ exact,
                                                          unsigned long long* __restrict__ n_exact) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    if (!exact[r]) return;
    __shared__ uint64_t tab[256];
    __shared__ double e[kExChunk];
    __shared__ double sh_acc;
    __shared__ int sh_tok;
    load_exp_tab(tab);
    const double mx = static_cast<double>(rowmax[r]);
    const float* L = logits + static_cast<size_t>(row_idx ? row_idx[r] : r) * V;
    double sum = 0.0;  // thread 0's running sum
    for (int base = 0; base < V; base += kExChunk) {
        const int n = min(kExChunk, V - base);
        for (int j = threadIdx.x; j < n; j += kExT) e[j] = gx::cdf_term(L[base + j], mx, temperature, tab);
        __syncthreads();
        if (threadIdx.x == 0)
            for (int j = 0; j < n; ++j) sum = __dadd_rn(sum, e[j]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sh_acc = __dmul_rn(row_uniform(seeds, key_pos, uniforms, r), sum);  // u
        sh_tok = -1;
    }
    __syncthreads();
    const double u = sh_acc;
    double acc = 0.0;
    for (int base = 0; base < V; base += kExChunk) {
        const int n = min(kExChunk, V - base);
        for (int j = threadIdx.x; j < n; j += kExT) e[j] = gx::cdf_term(L[base + j], mx, temperature, tab);
        __syncthreads();
        if (threadIdx.x == 0)
            for (int j = 0; j < n; ++j) {
                acc = __dadd_rn(acc, e[j]);
                if (u < acc) {
                    sh_tok = base + j;
                    break;
                }
            }
        __syncthreads();
        if (sh_tok >= 0) break;
    }
    if (threadIdx.x == 0) {
        out[r] = sh_tok >= 0 ? sh_tok : V - 1;
        atomicAdd(n_exact, 1ull);
    }
}

__global__ void debug_exp_kernel(const double* __restrict__ x, size_t n, double* __restrict__ y) {
    __shared__ uint64_t tab[256];
    load_exp_tab(tab);
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        y[i] = gx::exp(x[i], tab);
}

int chunks_for(int V) {
    const int P = (V + kCH - 1) / kCH;
    if (P > kMaxChunks) throw std::invalid_argument("vocab too large for the sampling kernels");
    return P;
}

}  // namespace

size_t row_scratch_bytes(int rows, int V) {
    return static_cast<size_t>(rows) * chunks_for(V) * sizeof(TopkRec) + 256;
}

void launch_emit(const float* logits, int V, const int* row_idx, const unsigned long long* seeds, const int* key_pos,
                 int R, double temperature, int* out, int* err, const RowScratch& sc, cudaStream_t st,
                 const double* uniforms) {
    if (R <= 0) return;
    const int P = chunks_for(V);
    if (R > sc.rows || static_cast<size_t>(R) * (((P + kCPC - 1) / kCPC) * kCPC) * sizeof(EmitRec) > sc.bytes)
        throw std::invalid_argument("emit: rows exceed the sampling scratch");
    EmitRec* rec = reinterpret_cast<EmitRec*>(sc.buf);
    const int Pc = (P + kCPC - 1) / kCPC;
    launch_pdl(emit_max_kernel, dim3(Pc, R), dim3(kT), 0, st, logits, V, Pc, row_idx, temperature, rec, sc.ctr,
               sc.rowmax, out, err);
    SGB_KCHECK();
    if (temperature != 0.0) {
        launch_pdl(emit_sample_kernel, dim3(P, R), dim3(kT), 0, st, logits, V, P, row_idx, seeds, key_pos, uniforms,
                   temperature, rec, sc.ctr, static_cast<const float*>(sc.rowmax), out, sc.exact);
        SGB_KCHECK();
        launch_pdl(emit_exact_kernel, dim3(R), dim3(kExT), 0, st, logits, V, row_idx, seeds, key_pos, uniforms,
                   temperature, static_cast<const float*>(sc.rowmax), out, sc.exact, sc.n_exact);
        SGB_KCHECK();
    }
}

int emit_launches(double temperature) { return temperature != 0.0 ? 3 : 1; }

void launch_debug_exp(const double* x, size_t n, double* out, cudaStream_t st) {
    if (n == 0) return;
    debug_exp_kernel<<<296, 256, 0, st>>>(x, n, out);
    SGB_KCHECK();
}

void launch_topk_lsm(const float* logits, int V, int R, int k, int* out_tok, double* out_lp, const RowScratch& sc,
                     cudaStream_t st) {
    if (R <= 0) return;
    if (k < 1 || k > kMaxK) throw std::invalid_argument("top-k must be in [1, 16]");
    const int P = chunks_for(V);
    if (R > sc.rows || static_cast<size_t>(R) * P * sizeof(TopkRec) > sc.bytes)
        throw std::invalid_argument("top-k: rows exceed the sampling scratch");
    launch_pdl(topk_kernel, dim3(P, R), dim3(kT), 0, st, logits, V, k, P, reinterpret_cast<TopkRec*>(sc.buf), sc.ctr,
               out_tok, out_lp);
    SGB_KCHECK();
}

}  // namespace sgb
