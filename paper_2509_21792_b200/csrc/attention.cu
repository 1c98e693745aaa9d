// Tree-masked paged-KV attention (decode / tree verify / draft expansion / prefill).
//
// Replaces the per-row, per-head scalar loop of the reference decode block
// (include/sgrpo/tinylm.hpp:335-395): scores over [cache | ancestor pool | masked new
// rows], softmax (nn.hpp:157-169), then P.V.
//
// Device formulation. Every query row carries a *virtual key sequence*: virtual index
// v < ctx_len maps to the contiguous cache slots ctx_base+v (the committed prefix), and
// ctx_len <= v < ctx_len+chain_len maps to chain_slots[v-ctx_len] (the row's own tree
// path: ancestors root-first, then itself). The virtual index equals the absolute
// position (target) or position-1 (draft cache), so a tree row and the AR row for the
// same token see the *same* key sequence in the same order -- the tree mask of
// build_tree_mask (drafttree.cpp:145-168) is exactly "keys = ancestors-or-self".
//
// Kernel (B200): one CTA per (row, run of 64-key blocks), ALL heads of the row. The K and
// V rows of a 16-key chunk are contiguous in the store ([slot][d], heads interleaved as
// in the reference), so one elected thread moves each chunk with a single bulk DMA
// (cp.async.bulk, mbarrier completion) into a 2-stage shared-memory ring: the kernel is a
// pure HBM stream with no per-lane address math on the load side. Tree-path keys come
// from the scratch slots with one bulk copy per key. One consumer warp per head (two
// heads per warp above 16 heads) computes coalesced conflict-free dot products from
// smem, an online softmax per chunk, and P.V with each lane owning DH/32 dims.
//
// Determinism / batch invariance (SURVEY.md §7 hard part 1): every 64-key block yields
// its own partial (m, l, acc) from a fresh state, with chunk boundaries fixed in virtual
// index; attn_combine_kernel merges a row's block partials strictly in block order. How
// many blocks a CTA walks (a launch-shape choice) never changes the bits, so the AR
// and the tree rows of the same token produce identical outputs.
//
// Roofline: HBM-bound on K/V reads, 4*d bytes per key per layer.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kBlock = 64;  // keys per softmax partial (fixed: part of the numerics)
constexpr int kStages = 2;

SGB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// KPC keys per chunk (fixed per d), HPW heads per consumer warp.
template <int DH, int KPC, int HPW>
__global__ void __launch_bounds__(1024, 1)
    attn_block_kernel(const float* __restrict__ q, const __nv_bfloat16* __restrict__ K,
                      const __nv_bfloat16* __restrict__ V, AttnRowsDev rows, int H, int d, int nb_max,
                      int blocks_per_cta, float scale, float* __restrict__ part_acc, float* __restrict__ part_ml) {
    pdl_wait();
    pdl_trigger();
    constexpr int PL = DH / 32;      // P.V dims per lane
    constexpr int LPR = DH / 8;      // lanes per key row in the score pass (16 B each)
    constexpr int RPI = 32 / LPR;    // key rows per score instruction
    constexpr int NIT = KPC / RPI;   // score instructions per chunk
    constexpr int CPB = kBlock / KPC;
    extern __shared__ __align__(128) uint8_t smem[];
    const size_t stage_bytes = static_cast<size_t>(KPC) * d * 2;  // one of K or V
    __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* Vs = reinterpret_cast<__nv_bfloat16*>(smem + kStages * stage_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kStages * stage_bytes);
    uint64_t* empty = full + kStages;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_cons = (H + HPW - 1) / HPW;
    const int r = blockIdx.y;
    const int ctx_len = rows.ctx_len[r];
    const int Lv = ctx_len + rows.chain_len[r];
    const long long ctx_base = rows.ctx_base[r];
    const long long* chain = rows.chain_slots + static_cast<size_t>(r) * kMaxChain;
    const int nb_row = (Lv + kBlock - 1) / kBlock;
    const int b0 = blockIdx.x * blocks_per_cta;
    const int b1 = min(nb_row, b0 + blocks_per_cta);
    if (b0 >= nb_row) return;
    const int k_begin = b0 * kBlock, k_end = min(Lv, b1 * kBlock);
    const int n_chunks = (k_end - k_begin + KPC - 1) / KPC;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], n_cons);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp == n_cons) {
        // ---------------- producer: bulk DMA of K/V chunks into the smem ring
        if (lane == 0) {
            for (int i = 0; i < n_chunks; ++i) {
                const int s = i % kStages;
                if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
                const int v0 = k_begin + i * KPC;
                const int v1 = min(k_end, v0 + KPC);
                const int nctx = max(0, min(v1, ctx_len) - v0);
                const int nch = (v1 - v0) - nctx;
                const uint32_t row_bytes = static_cast<uint32_t>(d) * 2;
                mbar_arrive_expect_tx(&full[s], 2u * row_bytes * (nctx + nch));
                __nv_bfloat16* kd = Ks + static_cast<size_t>(s) * KPC * d;
                __nv_bfloat16* vd = Vs + static_cast<size_t>(s) * KPC * d;
                if (nctx > 0) {
                    const size_t src = static_cast<size_t>(ctx_base + v0) * d;
                    bulk_g2s(kd, K + src, row_bytes * nctx, &full[s]);
                    bulk_g2s(vd, V + src, row_bytes * nctx, &full[s]);
                }
                for (int j = 0; j < nch; ++j) {
                    const size_t src = static_cast<size_t>(chain[v0 + nctx + j - ctx_len]) * d;
                    bulk_g2s(kd + static_cast<size_t>(nctx + j) * d, K + src, row_bytes, &full[s]);
                    bulk_g2s(vd + static_cast<size_t>(nctx + j) * d, V + src, row_bytes, &full[s]);
                }
            }
        }
        return;
    }
    if (warp > n_cons) return;

    // ---------------- consumers: warp `warp` owns heads warp*HPW .. +HPW-1
    const int piece = lane % LPR, sub = lane / LPR;
    float qreg[HPW][8];
    float m[HPW], l[HPW], acc[HPW][PL];
#pragma unroll
    for (int hh = 0; hh < HPW; ++hh) {
        const int h = warp * HPW + hh;
        const float* qrow = q + static_cast<size_t>(r) * d + min(h, H - 1) * DH;
#pragma unroll
        for (int t = 0; t < 8; ++t) qreg[hh][t] = qrow[piece * 8 + t];
    }
    for (int i = 0; i < n_chunks; ++i) {
        const int s = i % kStages;
        const int v0 = k_begin + i * KPC;
        const int nvalid = min(KPC, k_end - v0);
        const bool block_start = ((v0 - k_begin) % kBlock) == 0;
        mbar_wait(&full[s], (i / kStages) & 1);
        const __nv_bfloat16* kc = Ks + static_cast<size_t>(s) * KPC * d;
        const __nv_bfloat16* vc = Vs + static_cast<size_t>(s) * KPC * d;
#pragma unroll
        for (int hh = 0; hh < HPW; ++hh) {
            const int h = warp * HPW + hh;
            if (h >= H) break;
            if (block_start) {
                m[hh] = -INFINITY;
                l[hh] = 0.f;
#pragma unroll
                for (int e = 0; e < PL; ++e) acc[hh][e] = 0.f;
            }
            // scores: RPI rows per LDS.128 instruction, LPR-lane butterfly per row
            float sc = -INFINITY;
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
                const int key = it * RPI + sub;
                const uint4 u = *reinterpret_cast<const uint4*>(kc + static_cast<size_t>(key) * d + h * DH + piece * 8);
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
                float dot = 0.f;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 f = __bfloat1622float2(b2[t]);
                    dot = fmaf(qreg[hh][2 * t], f.x, dot);
                    dot = fmaf(qreg[hh][2 * t + 1], f.y, dot);
                }
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
#pragma unroll
                for (int rr = 0; rr < RPI; ++rr) {
                    const float dr = __shfl_sync(0xffffffffu, dot, rr * LPR);
                    if (lane == it * RPI + rr && lane < nvalid) sc = dr * scale;
                }
            }
            const float cm = warp_max(sc);
            const float nm = fmaxf(m[hh], cm);
            const float alpha = (m[hh] == -INFINITY) ? 0.f : expf(m[hh] - nm);
            const float p = (lane < nvalid) ? expf(sc - nm) : 0.f;
            l[hh] = l[hh] * alpha + warp_sum(p);
#pragma unroll
            for (int e = 0; e < PL; ++e) acc[hh][e] *= alpha;
            m[hh] = nm;
#pragma unroll
            for (int j = 0; j < KPC; ++j) {
                const float pj = __shfl_sync(0xffffffffu, p, j);
                if (j < nvalid) {
                    const __nv_bfloat16* vr = vc + static_cast<size_t>(j) * d + h * DH + lane * PL;
                    if constexpr (PL == 4) {
                        const uint2 u = *reinterpret_cast<const uint2*>(vr);
                        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
                        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
                        acc[hh][0] = fmaf(pj, a.x, acc[hh][0]);
                        acc[hh][1] = fmaf(pj, a.y, acc[hh][1]);
                        acc[hh][2] = fmaf(pj, b.x, acc[hh][2]);
                        acc[hh][3] = fmaf(pj, b.y, acc[hh][3]);
                    } else {
#pragma unroll
                        for (int e = 0; e < PL; e += 2) {
                            const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr + e));
                            acc[hh][e] = fmaf(pj, a.x, acc[hh][e]);
                            acc[hh][e + 1] = fmaf(pj, a.y, acc[hh][e + 1]);
                        }
                    }
                }
            }
            // end of a 64-key block (or of the row): publish the block partial
            const bool block_end = (((v0 + KPC - k_begin) % kBlock) == 0) || (v0 + KPC >= k_end);
            if (block_end) {
                const int b = v0 / kBlock;
                const size_t pidx = (static_cast<size_t>(r) * nb_max + b) * H + h;
                float* pa = part_acc + pidx * DH + lane * PL;
#pragma unroll
                for (int e = 0; e < PL; ++e) pa[e] = acc[hh][e];
                if (lane == 0) {
                    part_ml[2 * pidx] = m[hh];
                    part_ml[2 * pidx + 1] = l[hh];
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

// Merge a row's 64-key block partials strictly in block order -> bf16 attention output.
template <int DH>
__global__ void attn_combine_kernel(const float* __restrict__ part_acc, const float* __restrict__ part_ml,
                                    AttnRowsDev rows, int H, int nb_max, __nv_bfloat16* __restrict__ out, int d) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x, h = blockIdx.y;
    const int Lv = rows.ctx_len[r] + rows.chain_len[r];
    const int nb = (Lv + kBlock - 1) / kBlock;
    for (int e = threadIdx.x; e < DH; e += blockDim.x) {
        size_t pidx = static_cast<size_t>(r) * nb_max * H + h;
        float M = part_ml[2 * pidx], L = part_ml[2 * pidx + 1], A = part_acc[pidx * DH + e];
        for (int b = 1; b < nb; ++b) {
            pidx = (static_cast<size_t>(r) * nb_max + b) * H + h;
            const float mb = part_ml[2 * pidx], lb = part_ml[2 * pidx + 1], ab = part_acc[pidx * DH + e];
            const float Mn = fmaxf(M, mb);
            const float ca = expf(M - Mn), cb = expf(mb - Mn);
            L = L * ca + lb * cb;
            A = A * ca + ab * cb;
            M = Mn;
        }
        out[static_cast<size_t>(r) * d + h * DH + e] = __float2bfloat16(A / L);
    }
}

template <int DH, int KPC, int HPW>
void launch_impl(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, int M,
                 int H, int d, int nb_max, float* part_acc, float* part_ml, __nv_bfloat16* out, cudaStream_t st) {
    const size_t smem = 2 * kStages * static_cast<size_t>(KPC) * d * 2 + 64;
    static size_t attr = 0;
    if (attr < smem) {
        cudaFuncSetAttribute(attn_block_kernel<DH, KPC, HPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        attr = smem;
    }
    // enough CTAs for ~4 waves on 148 SMs; the blocks-per-CTA choice does not affect results
    const long long total_blocks = static_cast<long long>(M) * nb_max;
    int bpc = static_cast<int>((total_blocks + 148 * 4 - 1) / (148 * 4));
    bpc = std::max(1, std::min(bpc, nb_max));
    const int n_cons = (H + HPW - 1) / HPW;
    dim3 grid((nb_max + bpc - 1) / bpc, M);
    launch_pdl(attn_block_kernel<DH, KPC, HPW>, grid, dim3(32 * (n_cons + 1)), smem, st, q, K, V, rows, H, d, nb_max, bpc,
                                                                         1.0f / sqrtf(static_cast<float>(DH)),
                                                                         part_acc, part_ml);
    SGB_KCHECK();
    launch_pdl(attn_combine_kernel<DH>, dim3(M, H), dim3(DH), 0, st, part_acc, part_ml, rows, H, nb_max, out, d);
}

}  // namespace

int attn_splits_for(int max_virtual_len) { return (max_virtual_len + kBlock - 1) / kBlock; }

void launch_attention(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, int M,
                      int H, int d, int max_virtual_len, float* part_acc, float* part_ml, __nv_bfloat16* out,
                      cudaStream_t st) {
    if (M <= 0) return;
    const int dh = d / H;
    const int nb = attn_splits_for(max_virtual_len);
    // chunk size KPC is fixed per model width (2 stages x (K+V) must fit in shared memory);
    // it is part of the numerics, never a function of the batch
    if (H > 32) throw std::invalid_argument("attention: at most 32 heads");
    const int kpc = d <= 1664 ? 16 : (d <= 3328 ? 8 : 4);
    const bool two = H > 16;
#define SGB_ATT(DH_, KPC_, HPW_) launch_impl<DH_, KPC_, HPW_>(q, K, V, rows, M, H, d, nb, part_acc, part_ml, out, st)
    if (dh == 128 && kpc == 16) { if (two) SGB_ATT(128, 16, 2); else SGB_ATT(128, 16, 1); }
    else if (dh == 128 && kpc == 8) { if (two) SGB_ATT(128, 8, 2); else SGB_ATT(128, 8, 1); }
    else if (dh == 128 && kpc == 4) { if (two) SGB_ATT(128, 4, 2); else SGB_ATT(128, 4, 1); }
    else if (dh == 64 && kpc == 16) { if (two) SGB_ATT(64, 16, 2); else SGB_ATT(64, 16, 1); }
    else if (dh == 64 && kpc == 8) { if (two) SGB_ATT(64, 8, 2); else SGB_ATT(64, 8, 1); }
#undef SGB_ATT
    else throw std::invalid_argument("attention: head dim must be 64 or 128");
    SGB_KCHECK();
}

}  // namespace sgb
