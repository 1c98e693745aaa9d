// tcgen05 + TMA GEMM for sm_100a: persistent, warp-specialised, fused epilogues and a
// batch-invariant split-K.
//
//   Y[t][o] = sum_k X[t][k] * W[o][k]      (X = token rows, W = weight, both K-major bf16)
//
// Replaces the reference's scalar i-k-j nn::matmul (include/sgrpo/nn.hpp:15-29) for every
// projection of the decode forward: q/k/v (tinylm.hpp:325-327), wo (:396), w1 (:400),
// w2 (:402), lm_head (:458) and the draft fuse (:528). Weights are stored K-major
// ([out][in], bf16), so the reference's y = x.W is a "TN" GEMM whose UMMA A operand is
// the weight tile (M = 128 output features) and whose B operand is the token tile
// (N = BN in {16,32,64,128,256} tokens): the swap-AB mapping that keeps tcgen05 busy at
// decode batch sizes, where the kernel streams weight tiles at HBM rate.
//
// Persistent: one CTA per SM walks work units (m_tile, n_tile, k_split) round-robin; the
// smem stage ring and the two TMEM accumulator buffers run continuously across units, so
// the epilogue of one tile overlaps the MMAs of the next.
// Roles (320 threads): warp 0 = TMA producer, warp 1 = MMA issuer (+TMEM owner),
// warps 2-9 = epilogue (TMEM lane quarter = warp % 4 -> one output feature per thread;
// two warps per quarter split the token columns).
//
// Batch invariance (SURVEY.md §7 hard part 1). K is cut into fixed chunks whose width is
// a property of the WEIGHT (chosen once from N and K so that a one-token GEMM still spans
// the 148 SMs, never from the token count). Every chunk is accumulated separately in TMEM,
// read out, and the chunk sums are added in fp32 registers strictly in chunk order:
// ((c0 + c1) + c2) + ... A K split only decides WHICH CTA computes which chunks: split 0
// keeps the running prefix, later splits publish their raw chunk sums, and the last-
// arriving CTA continues the same sequential sum. The bits of an output element are
// therefore independent of M, of the token tile BN and of the split count, which makes the
// speculative and the AR rollouts bit-identical.
//
// Streaming: a pipeline stage carries kSub 64-wide k-boxes (up to 64 KB of weight) on one
// mbarrier -- measured on B200, per-SM TMA throughput grows with the bytes per stage, not
// with the stage count (scripts/probes/probe_bw.cu). With PDL the producer issues the
// weight boxes of its first stages BEFORE griddepcontrol.wait (weights never depend on the
// previous kernel), so the first HBM round trip overlaps the predecessor's tail.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "gemm.h"

namespace sgb {

int g_gemm_sm_cap = 0;

namespace {

#ifndef SGB_KSUB32
#define SGB_KSUB32 4
#endif
#ifndef SGB_KSUB64
#define SGB_KSUB64 2
#endif
#ifndef SGB_KSUB128
#define SGB_KSUB128 2
#endif
#ifndef SGB_GEMM_SMEM_KB
#define SGB_GEMM_SMEM_KB 220  // stage ring budget: 3 x 72 KB stages for 16-32-token tiles
#endif
#ifndef SGB_CHUNK_MIN
#define SGB_CHUNK_MIN 4
#endif
constexpr int kBK = 64;       // 64 bf16 = 128 B = one swizzle row
constexpr int kBM = 128;      // output features per tile (UMMA M)
constexpr int kABytes = kBM * kBK * 2;
// TMA warp, MMA warp, then 4*CQ epilogue warps: CQ column parts per TMEM lane quarter, so
// every epilogue thread owns one output feature and BN/CQ <= 64 token columns
constexpr int cq_for(int BN) { return BN >= 256 ? 4 : 2; }
constexpr int threads_for(int BN) { return 64 + 128 * cq_for(BN); }
constexpr int kNumSMs = 148;

// PAIR: the CTA pair (cta_group::2) form -- a 256-feature tile per 2-CTA cluster, each CTA
// holding its 128 weight rows and half of the token rows (BN / 2) in shared memory
template <int BN, bool PAIR = false>
struct GemmCfg {
    static constexpr int kSub = BN <= 32 ? SGB_KSUB32 : (BN == 64 ? SGB_KSUB64 : (BN == 128 ? SGB_KSUB128 : 1));
    static constexpr int kBRows = PAIR ? BN / 2 : BN;
    static constexpr int kBBytes = kBRows * kBK * 2;
    static constexpr int kStage = kSub * (kABytes + kBBytes);
    static constexpr int kStages = (SGB_GEMM_SMEM_KB * 1024) / kStage > 8 ? 8 : (SGB_GEMM_SMEM_KB * 1024) / kStage;
    static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int kSmem = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/;
    static constexpr int kCQ = cq_for(BN);
    static constexpr int kEpiThreads = 128 * kCQ;
    static constexpr int kThreads = threads_for(BN);
};

__device__ __forceinline__ float gelu_tanh(float x) {
    const float c = 0.7978845608028654f;
    return 0.5f * x * (1.0f + tanhf(c * (x + 0.044715f * x * x * x)));
}

// Element-wise epilogue (split-K finisher path).
__device__ __forceinline__ void epi_store(const GemmEpi& e, int t, int o, float v) {
    const size_t i = static_cast<size_t>(t) * e.ld + o;
    switch (e.kind) {
        case kEpiF32: e.f32[i] = v; break;
        case kEpiBF16: e.b16[i] = __float2bfloat16(v); break;
        case kEpiGeluBF16: e.b16[i] = __float2bfloat16(gelu_tanh(v)); break;
        case kEpiResid: e.f32[i] += v; break;
        case kEpiQKV:
            if (o < e.d) e.f32[static_cast<size_t>(t) * e.d + o] = v;
            else if (o < 2 * e.d) e.K[e.kv_dst[t] * e.d + (o - e.d)] = __float2bfloat16(v);
            else e.V[e.kv_dst[t] * e.d + (o - 2 * e.d)] = __float2bfloat16(v);
            break;
        case kEpiFusePos: e.f32[i] = v + e.pos_emb[static_cast<size_t>(e.pos[t]) * e.ld + o]; break;
    }
}

// Tile epilogue from registers: one branch on the (uniform) kind, then a tight loop over
// this thread's token columns. Stores are coalesced along the feature dimension o.
template <int HB>
__device__ __forceinline__ void epi_store_run(const GemmEpi& e, int t0, int n, int o, const float* run) {
    switch (e.kind) {
        case kEpiF32:
#pragma unroll
            for (int j = 0; j < HB; ++j)
                if (j < n) e.f32[static_cast<size_t>(t0 + j) * e.ld + o] = run[j];
            break;
        case kEpiBF16:
#pragma unroll
            for (int j = 0; j < HB; ++j)
                if (j < n) e.b16[static_cast<size_t>(t0 + j) * e.ld + o] = __float2bfloat16(run[j]);
            break;
        case kEpiGeluBF16:
#pragma unroll
            for (int j = 0; j < HB; ++j)
                if (j < n) e.b16[static_cast<size_t>(t0 + j) * e.ld + o] = __float2bfloat16(gelu_tanh(run[j]));
            break;
        case kEpiResid:
#pragma unroll
            for (int j = 0; j < HB; ++j)
                if (j < n) e.f32[static_cast<size_t>(t0 + j) * e.ld + o] += run[j];
            break;
        case kEpiQKV:
            if (o < e.d) {
#pragma unroll
                for (int j = 0; j < HB; ++j)
                    if (j < n) e.f32[static_cast<size_t>(t0 + j) * e.d + o] = run[j];
            } else {
                __nv_bfloat16* base = o < 2 * e.d ? e.K + (o - e.d) : e.V + (o - 2 * e.d);
#pragma unroll
                for (int j = 0; j < HB; ++j)
                    if (j < n) base[e.kv_dst[t0 + j] * e.d] = __float2bfloat16(run[j]);
            }
            break;
        case kEpiFusePos:
#pragma unroll
            for (int j = 0; j < HB; ++j)
                if (j < n)
                    e.f32[static_cast<size_t>(t0 + j) * e.ld + o] =
                        run[j] + e.pos_emb[static_cast<size_t>(e.pos[t0 + j]) * e.ld + o];
            break;
    }
}

template <int NT>
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

struct Unit {
    int m0, n0, split, tile;
};

// Units are tile-major (the K splits of a tile are adjacent), so the splits of a tile run
// concurrently and the finisher work is spread over the launch instead of its last wave.
// tw: features per tile (128, or 256 for a CTA pair), noff: this CTA's offset inside it
__device__ __forceinline__ Unit decode_unit(int u, int m_tiles, int S, int BN, int tw = kBM, int noff = 0) {
    Unit r;
    r.tile = u / S;
    r.split = u - r.tile * S;
    const int mt = r.tile % m_tiles;
    const int nt = r.tile / m_tiles;
    r.m0 = mt * BN;
    r.n0 = nt * tw + noff;
    return r;
}

// MMA width of a token tile: its valid rows rounded up to 16 (32 for a pair: each CTA's half
// of B stays a multiple of 16 rows)
__device__ __forceinline__ int mma_width(int rows, int BN, bool pair) {
    const int g = pair ? 32 : 16;
    return min(BN, max(g, (rows + g - 1) / g * g));
}

// The stage sequence of a CTA: units u = blockIdx.x + k*gridDim.x, each unit's chunks in
// order, each chunk in stages of up to kSub k-blocks (a stage never straddles a chunk).
struct StageSeq {
    int u, c, c_end, kb, hi;
    int n_units, stride, S, cps, nc, ckb, kbt, m_tiles, BN;
    __device__ void start_unit() {
        const Unit un = decode_unit(u, m_tiles, S, BN);
        c = un.split * cps;
        c_end = min(nc, c + cps);
        kb = c * ckb;
        hi = min(kbt, kb + ckb);
    }
    __device__ bool valid() const { return u < n_units; }
    __device__ void next(int ksub) {
        kb += ksub;
        if (kb < hi) return;
        if (++c < c_end) {
            kb = c * ckb;
            hi = min(kbt, kb + ckb);
            return;
        }
        u += stride;
        if (u < n_units) start_unit();
    }
};

template <int BN, bool PART, bool PAIR>
__global__ void __launch_bounds__(threads_for(BN), 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX, int M,
                        int N, int kb_total, int n_chunks, int ckb, int cps, int S, int m_tiles, int n_tiles, GemmEpi epi,
                        float* __restrict__ ws, int* __restrict__ ctr, int pf_boxes) {
    using Cfg = GemmCfg<BN, PAIR>;
    constexpr int TW = PAIR ? 2 * kBM : kBM;
    constexpr int SUB = Cfg::kSub;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStage);
    uint64_t* empty = full + Cfg::kStages;
    uint64_t* tfull = empty + Cfg::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_units = m_tiles * n_tiles * S;
    // pair: rank 0 (leader) issues the MMAs; full / tempty barriers live in the leader
    const int rank = PAIR ? static_cast<int>(cluster_rank()) : 0;
    const int noff = rank * kBM;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapW);
        tma_prefetch(&mapX);
        for (int s = 0; s < Cfg::kStages; ++s) {
            mbar_init(&full[s], PAIR ? 2 : 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], (PAIR ? 2 : 1) * Cfg::kEpiThreads / 32);
        }
        fence_barrier_init();
    }
    if constexpr (PAIR) {
        if (warp == 1) tmem_alloc_pair<Cfg::kTmemCols>(tmem_slot);
        tc_fence_before();
        cluster_sync_all();
    } else {
        if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
        tc_fence_before();
        __syncthreads();
    }
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    StageSeq seq0;
    seq0.u = PAIR ? blockIdx.x / 2 : blockIdx.x;
    seq0.n_units = n_units;
    seq0.stride = PAIR ? gridDim.x / 2 : gridDim.x;
    seq0.S = S;
    seq0.cps = cps;
    seq0.nc = n_chunks;
    seq0.ckb = ckb;
    seq0.kbt = kb_total;
    seq0.m_tiles = m_tiles;
    seq0.BN = BN;
    if (seq0.valid()) seq0.start_unit();

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first();
            // (1) weight boxes of the first stages: independent of the previous kernel
            StageSeq sq = seq0;
            int npre = 0;
            int pre_kb[Cfg::kStages], pre_ns[Cfg::kStages], pre_m0[Cfg::kStages];
            for (; npre < Cfg::kStages && sq.valid(); ++npre) {
                const int ns = min(SUB, sq.hi - sq.kb);
                const Unit un = decode_unit(sq.u, m_tiles, S, BN, TW, noff);
                uint8_t* a = smem + npre * Cfg::kStage;
                if constexpr (PAIR) {
                    const uint32_t fb = mapa_u32(&full[npre], 0);
                    mbar_arrive_expect_tx_remote(fb, ns * (kABytes + Cfg::kBBytes));
                    for (int j = 0; j < ns; ++j)
                        tma_load_2d_pair_hint(a + j * kABytes, &mapW, fb, (sq.kb + j) * kBK, un.n0, pol_w);
                    pre_m0[npre] = un.m0 + rank * (mma_width(M - un.m0, BN, true) / 2);
                } else {
                    mbar_arrive_expect_tx(&full[npre], ns * (kABytes + Cfg::kBBytes));
                    for (int j = 0; j < ns; ++j)
                        tma_load_2d_hint(a + j * kABytes, &mapW, &full[npre], (sq.kb + j) * kBK, un.n0, pol_w);
                    pre_m0[npre] = un.m0;
                }
                pre_kb[npre] = sq.kb;
                pre_ns[npre] = ns;
                sq.next(SUB);
            }
            // (1b) HBM-bound token tiles: the following weight boxes go to L2 as well, so the
            // weight stream keeps running while the previous kernel drains (pf_boxes per CTA,
            // sized by the host to a fraction of L2; the smem loads then hit in L2)
            {
                StageSeq pq = sq;
                for (int n = 0; n < pf_boxes && pq.valid(); pq.next(SUB)) {
                    const int ns = min(SUB, pq.hi - pq.kb);
                    const Unit un = decode_unit(pq.u, m_tiles, S, BN, TW, noff);
                    for (int j = 0; j < ns; ++j, ++n) tma_prefetch_l2_2d(&mapW, (pq.kb + j) * kBK, un.n0);
                }
            }
            // (2) activations are produced by the previous kernel
            pdl_wait();
            pdl_trigger();
            for (int s = 0; s < npre; ++s) {
                uint8_t* b = smem + s * Cfg::kStage + SUB * kABytes;
                for (int j = 0; j < pre_ns[s]; ++j) {
                    if constexpr (PAIR)
                        tma_load_2d_pair(b + j * Cfg::kBBytes, &mapX, mapa_u32(&full[s], 0), (pre_kb[s] + j) * kBK,
                                         pre_m0[s]);
                    else
                        tma_load_2d(b + j * Cfg::kBBytes, &mapX, &full[s], (pre_kb[s] + j) * kBK, pre_m0[s]);
                }
            }
            // (3) steady state
            for (int i = npre; sq.valid(); ++i, sq.next(SUB)) {
                const int s = i % Cfg::kStages;
                mbar_wait(&empty[s], ((i / Cfg::kStages) & 1) ^ 1);
                const int ns = min(SUB, sq.hi - sq.kb);
                const Unit un = decode_unit(sq.u, m_tiles, S, BN, TW, noff);
                uint8_t* a = smem + s * Cfg::kStage;
                if constexpr (PAIR) {
                    const uint32_t fb = mapa_u32(&full[s], 0);
                    const int xm = un.m0 + rank * (mma_width(M - un.m0, BN, true) / 2);
                    mbar_arrive_expect_tx_remote(fb, ns * (kABytes + Cfg::kBBytes));
                    for (int j = 0; j < ns; ++j) {
                        tma_load_2d_pair_hint(a + j * kABytes, &mapW, fb, (sq.kb + j) * kBK, un.n0, pol_w);
                        tma_load_2d_pair(a + SUB * kABytes + j * Cfg::kBBytes, &mapX, fb, (sq.kb + j) * kBK, xm);
                    }
                } else {
                    mbar_arrive_expect_tx(&full[s], ns * (kABytes + Cfg::kBBytes));
                    for (int j = 0; j < ns; ++j) {
                        tma_load_2d_hint(a + j * kABytes, &mapW, &full[s], (sq.kb + j) * kBK, un.n0, pol_w);
                        tma_load_2d(a + SUB * kABytes + j * Cfg::kBBytes, &mapX, &full[s], (sq.kb + j) * kBK, un.m0);
                    }
                }
            }
        } else {
            pdl_wait();
            pdl_trigger();
        }
    } else if (warp == 1) {
        pdl_wait();
        pdl_trigger();
        if (lane == 0 && rank == 0) {
            // MMA width = the tile's valid token rows rounded up to 16 (tcgen05 N granularity):
            // a 211-row tile issues 224-wide MMAs, not 256. Output columns are independent, so
            // the width never changes an element's bits (test_gemm_batch_invariance).
            uint32_t idesc = PAIR ? idesc_bf16_m256(BN) : idesc_bf16_m128(BN);
            StageSeq sq = seq0;
            int i = 0, it = -1, cur_c = -1, cur_u = -1;
            for (; sq.valid(); ++i) {
                const bool chunk_start = (sq.u != cur_u || sq.c != cur_c);
                if (chunk_start) {
                    if (sq.u != cur_u) {
                        const int n_eff = mma_width(M - decode_unit(sq.u, m_tiles, S, BN).m0, BN, PAIR);
                        idesc = PAIR ? idesc_bf16_m256(static_cast<uint32_t>(n_eff))
                                     : idesc_bf16_m128(static_cast<uint32_t>(n_eff));
                    }
                    cur_u = sq.u;
                    cur_c = sq.c;
                    ++it;
                    if (it >= 2) mbar_wait(&tempty[it & 1], ((it >> 1) - 1) & 1);
                    tc_fence_after();
                }
                const int buf = it & 1;
                const int ns = min(SUB, sq.hi - sq.kb);
                const bool first = sq.kb == sq.c * ckb;
                const bool chunk_end = sq.kb + ns >= sq.hi;
                const int s = i % Cfg::kStages;
                mbar_wait(&full[s], (i / Cfg::kStages) & 1);
                tc_fence_after();
                const uint32_t a = smem_u32(smem + s * Cfg::kStage);
                const uint32_t b = a + SUB * kABytes;
                for (int j = 0; j < ns; ++j) {
                    const uint64_t adesc = sw128_desc(a + j * kABytes), bdesc = sw128_desc(b + j * Cfg::kBBytes);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        if constexpr (PAIR)
                            umma_bf16_pair(tmem + buf * BN, adesc + 2 * k, bdesc + 2 * k, idesc,
                                           (!first || j != 0 || k != 0));
                        else
                            umma_bf16(tmem + buf * BN, adesc + 2 * k, bdesc + 2 * k, idesc,
                                      (!first || j != 0 || k != 0));
                    }
                }
                if constexpr (PAIR) {
                    umma_commit_pair(&empty[s], 0x3);
                    if (chunk_end) umma_commit_pair(&tfull[buf], 0x3);
                } else {
                    umma_commit(&empty[s]);
                    if (chunk_end) umma_commit(&tfull[buf]);
                }
                sq.next(SUB);
            }
        }
    } else {
        pdl_wait();
        pdl_trigger();
        // ---------------- epilogue warps: TMEM lane quarter q (output feature o), column part h
        constexpr int HB = BN / Cfg::kCQ;
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        const int r = 32 * q + lane;
        const int j0 = h * HB;
        int it = 0;
        for (int u = seq0.u; u < n_units; u += seq0.stride) {
            const Unit un = decode_unit(u, m_tiles, S, BN, TW, noff);
            const int ctile = PAIR ? 2 * un.tile + rank : un.tile;  // 128-feature tile: finisher state
            const int o = un.n0 + r;
            const int ncols = min(BN, M - un.m0);
            const int nmine = max(0, min(HB, ncols - j0));
            const int c_begin = un.split * cps, c_end = min(n_chunks, c_begin + cps);
            float* wst = ws ? ws + static_cast<size_t>(ctile) * n_chunks * BN * kBM : nullptr;
            // 256-token tiles run only single-chunk weights (gemm_run), so their pieces are final
            constexpr bool kOneChunk = (BN == 256);
            float run[(PART || kOneChunk) ? 1 : HB];  // the chunk-ordered running sum
            for (int c = c_begin; c < c_end; ++c, ++it) {
                const int buf = it & 1;
                mbar_wait(&tfull[buf], (it >> 1) & 1);
                tc_fence_after();
                // read the chunk out of TMEM in pieces of <= 64 columns (register budget)
                constexpr int PC = HB < 64 ? HB : (HB == 64 ? 64 : 32);
#pragma unroll
                for (int p0 = 0; p0 < HB; p0 += PC) {
                    float v[PC];
                    tmem_ld<PC>(tmem + (static_cast<uint32_t>(32 * q) << 16) + buf * BN + j0 + p0, v);
                    if constexpr (PART) {
                        float* dst = epi.f32 + (static_cast<size_t>(c) * M + un.m0 + j0 + p0) * epi.ld + o;
#pragma unroll
                        for (int j = 0; j < PC; ++j)
                            if (p0 + j < nmine && o < N) dst[static_cast<size_t>(j) * epi.ld] = v[j];
                    } else if constexpr (kOneChunk) {
                        if (o < N && p0 < nmine) epi_store_run<PC>(epi, un.m0 + j0 + p0, nmine - p0, o, v);
                    } else if (un.split == 0) {
                        if (c == c_begin) {
#pragma unroll
                            for (int j = 0; j < PC; ++j) run[p0 + j] = v[j];
                        } else {
#pragma unroll
                            for (int j = 0; j < PC; ++j) run[p0 + j] += v[j];
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < PC; ++j)
                            if (p0 + j < nmine) wst[(static_cast<size_t>(c) * BN + j0 + p0 + j) * kBM + r] = v[j];
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR) mbar_arrive_remote(mapa_u32(&tempty[buf], 0));
                    else mbar_arrive(&tempty[buf]);
                }
            }
            if constexpr (PART || kOneChunk) {
                // raw chunk sums / single-chunk results already stored
            } else if (S == 1) {
                if (o < N) epi_store_run<HB>(epi, un.m0 + j0, nmine, o, run);
            } else {
                if (un.split == 0)
#pragma unroll
                    for (int j = 0; j < HB; ++j)
                        if (j < nmine) wst[static_cast<size_t>(j0 + j) * kBM + r] = run[j];
                __threadfence();
                epi_bar<Cfg::kEpiThreads>();
                if (threadIdx.x == 64) {
                    const int old = atomicAdd(&ctr[ctile], 1);
                    *last_flag = (old == S - 1);
                }
                epi_bar<Cfg::kEpiThreads>();
                const int last = *last_flag;
                if (last) {
                    __threadfence();
                    if (o < N) {
                        // The finisher continues the sequential chunk sum. Columns are
                        // independent: 8 columns x FB chunks of loads are in flight at once,
                        // then added strictly in chunk order per column.
                        constexpr int FB = HB <= 8 ? 8 : 4;
                        for (int jb = j0; jb < j0 + nmine; jb += 8) {
                            float v[8];
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                v[t] = (jb + t < j0 + nmine) ? __ldcg(&wst[static_cast<size_t>(jb + t) * kBM + r]) : 0.f;
                            for (int c0 = cps; c0 < n_chunks; c0 += FB) {
                                float a[FB][8];
#pragma unroll
                                for (int cc = 0; cc < FB; ++cc)
#pragma unroll
                                    for (int t = 0; t < 8; ++t)
                                        a[cc][t] = (c0 + cc < n_chunks && jb + t < j0 + nmine)
                                                       ? __ldcg(&wst[(static_cast<size_t>(c0 + cc) * BN + jb + t) * kBM + r])
                                                       : 0.f;
#pragma unroll
                                for (int cc = 0; cc < FB; ++cc)
                                    if (c0 + cc < n_chunks)
#pragma unroll
                                        for (int t = 0; t < 8; ++t) v[t] += a[cc][t];
                            }
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                if (jb + t < j0 + nmine) epi_store(epi, un.m0 + jb + t, o, v[t]);
                        }
                    }
                    if (threadIdx.x == 64) ctr[ctile] = 0;
                }
                epi_bar<Cfg::kEpiThreads>();  // last_flag is reused by the next unit
            }
        }
    }
    tc_fence_before();
    if constexpr (PAIR) {
        cluster_sync_all();  // the leader's MMAs read the peer's shared memory / write its TMEM
        if (warp == 1) tmem_dealloc_pair<Cfg::kTmemCols>(tmem);
    } else {
        __syncthreads();
        if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <int BN, bool PART, bool PAIR = false>
void launch_bn(const CUtensorMap& w, const CUtensorMap& x, int M, int N, int kbt, int n_chunks, int ckb, int S, int cps,
               const GemmEpi& epi, float* ws, int* ctr, cudaStream_t st) {
    using Cfg = GemmCfg<BN, PAIR>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN, PART, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Cfg::kSmem);
        attr = true;
    }
    constexpr int TW = PAIR ? 2 * kBM : kBM;
    const int m_tiles = (M + BN - 1) / BN, n_tiles = (N + TW - 1) / TW;
    const int units = m_tiles * n_tiles * S;
    if constexpr (PAIR) {
        // one unit per CTA pair per round; the 2-CTA cluster maps onto one TPC
        const int grid = 2 * std::min(units, kNumSMs / 2);
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(Cfg::kThreads);
        cfg.dynamicSmemBytes = Cfg::kSmem;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 2;
        cudaLaunchKernelEx(&cfg, gemm_bf16_tn_kernel<BN, PART, true>, w, x, M, N, kbt, n_chunks, ckb, cps, S, m_tiles,
                           n_tiles, epi, ws, ctr, 0);
        return;
    }
    const int grid = std::min(units, g_gemm_sm_cap > 0 ? g_gemm_sm_cap : kNumSMs);
    // L2 prefetch budget for the weight stream of HBM-bound (<= 32-token) tiles, in MB over
    // the whole grid. A/B switch only, off by default: measured at the 7B shape, 48 MB made
    // the one-token QKV GEMM 17.4 -> 19.6 us and the B = 1 AR step 3.19 -> 3.50 ms
    // (profiles/r01_tail_b1_c3.txt)
    static const int pf_mb = [] {
        const char* v = getenv("SGB_L2_PF_MB");
        return v ? atoi(v) : 0;
    }();
    const int pf_boxes = BN <= 32 ? static_cast<int>((static_cast<long long>(pf_mb) << 20) / grid / kABytes) : 0;
    launch_pdl(gemm_bf16_tn_kernel<BN, PART, false>, dim3(grid), dim3(Cfg::kThreads), Cfg::kSmem, st, w, x, M, N, kbt, n_chunks, ckb,
               cps, S, m_tiles, n_tiles, epi, ws, ctr, pf_boxes);
}

}  // namespace

// Chunk width (in 64-wide k-blocks) of a weight [N][K]: enough chunks that a one-token
// GEMM has ~one unit per SM, at least 4 k-blocks (one full stage) per chunk. A function
// of the weight shape only -- never of the token count -- so the fp32 association of
// every output is fixed per weight.
int gemm_chunk_kb(int N, int K) {
    const int kbt = (K + kBK - 1) / kBK;
    const int n_tiles = (N + kBM - 1) / kBM;
    // weights wider than 64 tiles are never K-split (gemm_splits_for): one chunk, which also
    // lets their >128-row GEMMs take 256-token tiles
    static const int max_split_tiles = [] {
        const char* v = getenv("SGB_CHUNK_TILES_MAX");  // A/B switch (0 = chunk every weight)
        return v ? atoi(v) : 64;  // measured: c2 +1.3 %, c3 speculative steps 3-5 % cheaper
    }();
    if (max_split_tiles > 0 && n_tiles > max_split_tiles) return ((kbt + 3) / 4) * 4;
    // at most floor(148 / n_tiles) splits fit one wave (gemm_splits_for), so the chunk count
    // aims at that: a ceil here gave the 7B w2 six chunks, which only split 3 ways (84 CTAs,
    // 104 k-blocks each); five chunks split 5 ways (140 CTAs, 60 k-blocks): M = 1 w2 31 -> ~22 us
    const int want = std::max(1, kNumSMs / n_tiles);
    int ckb = (kbt + want - 1) / want;
    ckb = ((ckb + 3) / 4) * 4;
    ckb = std::max(ckb, SGB_CHUNK_MIN);
    return std::min(ckb, ((kbt + 3) / 4) * 4);
}

int gemm_chunks(int N, int K) {
    const int kbt = (K + kBK - 1) / kBK;
    const int ckb = gemm_chunk_kb(N, K);
    return (kbt + ckb - 1) / ckb;
}

static int chunks_of(int N, int K) {
    const int kbt = (K + kBK - 1) / kBK;
    const int ckb = gemm_chunk_kb(N, K);
    return (kbt + ckb - 1) / ckb;
}

CUtensorMap make_kmajor_map(const void* ptr, int rows, int K, int box_rows) {
    if (K % 8) throw std::invalid_argument("GEMM K must be a multiple of 8");
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

int gemm_bn_for(int M) {
    if (M <= 16) return 16;
    // BN=32 measured slower than BN=64 for 17..32 tokens at the c2 shapes
    // (profiles/hw_profile_c2.json latency curve); BN=32 stays instantiated for tests
    if (M <= 64) return 64;
    if (M <= 128) return 128;
    // 256-token tiles (16 epilogue warps, 64 columns each): every weight tile is streamed
    // once per 256 rows -- the 129..256-row verify forwards read the weights once, not twice
    static const int max_bn = [] {
        const char* v = getenv("SGB_GEMM_MAXBN");  // tuning experiments only
        return v ? atoi(v) : 256;
    }();
    // 257..384 rows: three 128-token tiles beat two 256-token ones (M = 384 at the c5 QKV shape:
    // 45.6 vs 57.3 us, profiles/r02_gemm_c5_ab.jsonl); 129..256 rows keep one 256-token tile
    if (M > 256 && M <= 384) return 128;
    return max_bn >= 256 ? 256 : 128;
}

// CTA-pair (cta_group::2) tiles for 128- and 256-token tiles: each SM receives half of the
// token tile (the operand bytes per MMA flop drop by a third). Bit-identical to the 1-CTA
// kernel (test_gemm_batch_invariance, spec == AR rollouts) but not faster: measured
// (profiles/r02_gemm_pair_sweep.jsonl, ncu in profiles/README.md) the producer waits on free
// stages, i.e. the MMA issue rate -- not the TMA delivery -- bounds these shapes, and the pair
// is 0-8 % slower at the c2 shapes. Off by default; SGB_GEMM_PAIR=1 selects it.
bool gemm_pair() {
    static const bool on = [] {
        const char* v = getenv("SGB_GEMM_PAIR");
        return v ? atoi(v) != 0 : false;
    }();
    return on;
}

// K split: which CTA computes which chunks. Any choice gives identical bits.
int gemm_splits_for(int M, int N, int K) {
    const int bn = gemm_bn_for(M);
    const int tiles = ((M + bn - 1) / bn) * ((N + kBM - 1) / kBM);
    const int nc = chunks_of(N, K);
    if (nc <= 1) return 1;
    int S = 1;
    if (bn <= 32) {
        // HBM-bound decode regime: up to one unit per SM; with more than ~64 weight tiles a
        // split only adds finisher latency (measured, scripts/gemm_sweep.py)
        if (tiles <= 64) S = std::min(nc, kNumSMs / tiles);
    }
    // token tiles of 64-128: the in-kernel finisher would read (nc - cps) raw chunk partials
    // of BN x 128 fp32 each; those GEMMs run unsplit, or in kEpiPartials mode when a row
    // kernel follows (wo, w2, draft fuse)
    S = std::max(1, S);
    const int cps = (nc + S - 1) / S;
    return (nc + cps - 1) / cps;
}

size_t gemm_ws_floats(int M, int N, int K) {
    const int bn = gemm_bn_for(M);
    // 128-feature tiles, rounded up to whole CTA pairs
    const size_t tiles = static_cast<size_t>((M + bn - 1) / bn) * (2 * ((N + 2 * kBM - 1) / (2 * kBM)));
    return tiles * chunks_of(N, K) * bn * kBM;
}

void gemm_run(const GemmWeight& w, const GemmAct& x, int M, const GemmEpi& epi, const GemmWorkspace& ws,
              cudaStream_t st, int force_splits) {
    if (M <= 0) return;
    if (M > x.cap_rows) throw std::invalid_argument("gemm: rows exceed activation capacity");
    const int kbt = (w.K + kBK - 1) / kBK;
    const int ckb = w.chunk_kb;
    const int nc = (kbt + ckb - 1) / ckb;
    int S = force_splits > 0 ? std::min(force_splits, nc) : gemm_splits_for(M, w.N, w.K);
    const int bn = gemm_bn_for(M);
    const int tiles = ((M + bn - 1) / bn) * ((w.N + kBM - 1) / kBM);
    if (epi.kind == kEpiPartials) {
        // one unit per (tile, chunk), no in-kernel finisher. Token tile: 128 up to 384 rows
        // (more units), 256 above (each weight tile read once per 256 tokens); measured with
        // scripts/gemm_part.py at the c2/c3 residual shapes
        static const int part_bn = [] {
            const char* v = getenv("SGB_PART_BN");  // tuning experiments only
            return v ? atoi(v) : 0;
        }();
        const int pbn = part_bn > 0 && M > 128 ? part_bn : (M > 384 ? 256 : std::max(64, bn));
        if (gemm_pair() && pbn >= 128) {
            const CUtensorMap& xm = x.map_for_bn(pbn / 2);
            if (pbn == 256) launch_bn<256, true, true>(w.map, xm, M, w.N, kbt, nc, ckb, nc, 1, epi, nullptr, nullptr, st);
            else launch_bn<128, true, true>(w.map, xm, M, w.N, kbt, nc, ckb, nc, 1, epi, nullptr, nullptr, st);
            return;
        }
        const CUtensorMap& xm = x.map_for_bn(pbn);
        if (pbn == 256) launch_bn<256, true>(w.map, xm, M, w.N, kbt, nc, ckb, nc, 1, epi, nullptr, nullptr, st);
        else if (pbn == 128) launch_bn<128, true>(w.map, xm, M, w.N, kbt, nc, ckb, nc, 1, epi, nullptr, nullptr, st);
        else launch_bn<64, true>(w.map, xm, M, w.N, kbt, nc, ckb, nc, 1, epi, nullptr, nullptr, st);
        return;
    }
    if (S > 1 && (ws.buf == nullptr || gemm_ws_floats(M, w.N, w.K) > ws.cap_floats || tiles > ws.ctr_cap)) S = 1;
    const int cps = (nc + S - 1) / S;
    S = (nc + cps - 1) / cps;
    const int bn_run = (bn == 256 && (nc > 1 || S > 1)) ? 128 : bn;  // 256-token tiles: single-chunk weights
    if (gemm_pair() && bn_run >= 128) {
        const CUtensorMap& xp = x.map_for_bn(bn_run / 2);
        if (bn_run == 256) launch_bn<256, false, true>(w.map, xp, M, w.N, kbt, nc, ckb, S, cps, epi, ws.buf, ws.ctr, st);
        else launch_bn<128, false, true>(w.map, xp, M, w.N, kbt, nc, ckb, S, cps, epi, ws.buf, ws.ctr, st);
        return;
    }
    const CUtensorMap& xm = x.map_for_bn(bn_run);
    switch (bn_run) {
        case 16: launch_bn<16, false>(w.map, xm, M, w.N, kbt, nc, ckb, S, cps, epi, ws.buf, ws.ctr, st); break;
        case 64: launch_bn<64, false>(w.map, xm, M, w.N, kbt, nc, ckb, S, cps, epi, ws.buf, ws.ctr, st); break;
        case 128: launch_bn<128, false>(w.map, xm, M, w.N, kbt, nc, ckb, S, cps, epi, ws.buf, ws.ctr, st); break;
        default: launch_bn<256, false>(w.map, xm, M, w.N, kbt, nc, ckb, S, cps, epi, ws.buf, ws.ctr, st); break;
    }
}

void GemmWeight::init(const __nv_bfloat16* p, int n, int k, int chunk_kb_override) {
    ptr = p;
    N = n;
    K = k;
    chunk_kb = chunk_kb_override > 0 ? chunk_kb_override : gemm_chunk_kb(n, k);
    map = make_kmajor_map(p, n, k, kBM);
}

void GemmAct::init(const __nv_bfloat16* p, int rows, int k) {
    ptr = p;
    cap_rows = rows;
    K = k;
    const int bns[5] = {16, 32, 64, 128, 256};
    for (int i = 0; i < 5; ++i) maps[i] = make_kmajor_map(p, rows, k, bns[i]);
}

const CUtensorMap& GemmAct::map_for_bn(int bn) const {
    switch (bn) {
        case 16: return maps[0];
        case 32: return maps[1];
        case 64: return maps[2];
        case 128: return maps[3];
        default: return maps[4];
    }
}

}  // namespace sgb
