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

// T > 0: thread t of chunk p owns the kPer contiguous logits base + t*kPer ...; sums are
// sequential in fp64 inside a thread, then in thread order, then in chunk order.
__device__ __forceinline__ double thread_expsum(const float* L, int V, int lo, double mx, double temperature) {
    double s = 0.0;
    const int hi = min(V, lo + kPer);
    for (int i = lo; i < hi; ++i) s += exp((static_cast<double>(L[i]) - mx) / temperature);
    return s;
}

__global__ void __launch_bounds__(kT) emit_sample_kernel(const float* __restrict__ logits, int V, int P,
                                                         const int* __restrict__ row_idx,
                                                         const unsigned long long* __restrict__ seeds,
                                                         const int* __restrict__ key_pos, double temperature,
                                                         EmitRec* __restrict__ rec, int* __restrict__ ctr,
                                                         const float* __restrict__ rowmax, int* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    __shared__ double ts[kT];
    __shared__ VI shv[kT / 32];
    __shared__ int flag;
    __shared__ double sh_u;
    __shared__ int sh_p;
    const int p = blockIdx.x, r = blockIdx.y;
    const float mxf = rowmax[r];
    if (mxf == -INFINITY) return;  // emit_max flagged the row (domain_error)
    const double mx = static_cast<double>(mxf);
    const float* L = logits + static_cast<size_t>(row_idx ? row_idx[r] : r) * V;
    const int lo = p * kCH + static_cast<int>(threadIdx.x) * kPer;
    ts[threadIdx.x] = thread_expsum(L, V, lo, mx, temperature);
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int t = 0; t < kT; ++t) acc += ts[t];
        rec[static_cast<size_t>(r) * (((P + kCPC - 1) / kCPC) * kCPC) + p].s = acc;
    }
    if (!last_of_row(ctr, r, P, &flag)) return;
    const EmitRec* rr = rec + static_cast<size_t>(r) * (((P + kCPC - 1) / kCPC) * kCPC);
    if (threadIdx.x == 0) {
        // chunk prefixes in order; the winner chunk is the last non-empty one whose
        // exclusive prefix is <= u
        double acc = 0.0;
        for (int q = 0; q < P; ++q) acc += __ldcg(&rr[q].s);
        const uint64_t key = mix_key(seeds[r], static_cast<uint64_t>(key_pos[r]));
        const double u = rng_first_uniform(key) * acc;
        double pre = 0.0;
        int win = 0;
        for (int q = 0; q < P; ++q) {
            if (pre <= u) win = q;
            pre += __ldcg(&rr[q].s);
        }
        double wpre = 0.0;
        for (int q = 0; q < win; ++q) wpre += __ldcg(&rr[q].s);
        sh_u = u;
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
    ts[threadIdx.x] = thread_expsum(L, V, wlo, mx, temperature);
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = cpre;
        for (int t = 0; t < kT; ++t) {
            const double c = ts[t];
            ts[t] = acc;  // exclusive prefix of thread t (chunk prefix included)
            acc += c;
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
        int tok = hi - 1;
        for (int i = wlo; i < hi; ++i) {
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
                 int R, double temperature, int* out, int* err, const RowScratch& sc, cudaStream_t st) {
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
        launch_pdl(emit_sample_kernel, dim3(P, R), dim3(kT), 0, st, logits, V, P, row_idx, seeds, key_pos, temperature,
                   rec, sc.ctr, static_cast<const float*>(sc.rowmax), out);
        SGB_KCHECK();
    }
}

int emit_launches(double temperature) { return temperature != 0.0 ? 2 : 1; }

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
