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
// Kernel (B200): persistent and flat. The work of a launch is the list of items
// (row, head group, 64-key block), rows in order; CTA c takes the contiguous slice
// [c*T/G, (c+1)*T/G) of it, so every CTA streams the same number of blocks (+-1) whatever
// the mix of context lengths, and its shared-memory ring never drains between rows. The K
// and V rows of a KPC-key chunk are contiguous in the store ([slot][d], heads interleaved
// as in the reference): with all heads in one item a chunk is ONE bulk DMA
// (cp.async.bulk, mbarrier completion); at small batch the heads are split into groups so
// the launch still covers the SMs, and each key row of the group is its own bulk copy.
// Tree-path keys come from the scratch slots with one bulk copy per key. One consumer warp
// per head (two heads per warp above 12 heads) computes dot products from smem, an online
// softmax per chunk, and P.V with each lane owning DH/32 dims. The CTA that completes the
// last block of a (row, head group) -- an atomic ticket per row -- merges the row's block
// partials in block order and writes the bf16 output: no separate combine launch.
//
// Determinism / batch invariance (SURVEY.md §7 hard part 1): every 64-key block yields
// its own partial (m, l, acc) from a fresh state, with chunk boundaries fixed in virtual
// index; the merge runs strictly in block order. How the blocks are spread over CTAs and
// heads over groups (launch-shape choices) never changes the bits, so the AR and the tree
// rows of the same token produce identical outputs.
//
// Roofline: HBM-bound on K/V reads, 4*d bytes per key per layer.
#include <algorithm>
#include <cstdlib>
#include <cfloat>

#include "attn_numerics.cuh"
#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kBlock = kAttnBlock;

SGB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int kMaxScanRows = 1 << 20;
constexpr int kSmemBudget = 227 * 1024;

struct ItemIt {
    int r, g, b, nb;
};

__device__ __forceinline__ int row_blocks(const AttnRowsDev& rows, int r) {
    return (rows.ctx_len[r] + rows.chain_len[r] + kBlock - 1) / kBlock;
}

// KPC keys per chunk (fixed per d), HPW heads per consumer warp.
template <int DH, int KPC, int HPW>
__global__ void __launch_bounds__(HPW == 1 ? 416 : 544, HPW == 1 ? 2 : 1)  // consumers + producer
    attn_kernel(const float* __restrict__ q, const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
                AttnRowsDev rows, int M, int H, int d, int G, int nst, int nb_max, float scale,
                float* __restrict__ part_acc, float* __restrict__ part_ml, int* __restrict__ row_ctr,
                __nv_bfloat16* __restrict__ out) {
    constexpr int PL = DH / 32;      // P.V dims per lane
    constexpr int LPR = DH / 16;     // lanes per key row in the score pass (16 dims = 32 B each)
    constexpr int RPI = 32 / LPR;    // key rows per score instruction
    constexpr int NIT = KPC / RPI;   // score instructions per chunk
    extern __shared__ __align__(128) uint8_t smem[];
    const int HG = H / G;            // heads per item
    const int wd = HG * DH;          // item width (elements)
    const size_t kv_bytes = static_cast<size_t>(KPC) * wd * 2;  // one of K or V per stage
    __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem);
    __nv_bfloat16* Vs = reinterpret_cast<__nv_bfloat16*>(smem + nst * kv_bytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * nst * kv_bytes);
    uint64_t* empty = full + nst;
    int* flag = reinterpret_cast<int*>(empty + nst);
    int* tsum = flag + 4;                 // [blockDim.x + 1]
    int* loc = tsum + blockDim.x + 1;     // [2] start row, start block offset

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_cons = (HG + HPW - 1) / HPW;
    const int nthr = blockDim.x;

    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], n_cons);
        }
        fence_barrier_init();
    }
    // PDL: barrier setup overlapped the previous kernel; row metadata is produced by it
    pdl_wait();
    pdl_trigger();
    // ---- block counts per thread slice of rows [t*per, (t+1)*per), exclusive scan over slices
    const int per = (M + nthr - 1) / nthr;
    const int r0 = min(M, static_cast<int>(threadIdx.x) * per), r1 = min(M, r0 + per);
    int own = 0;
    for (int r = r0; r < r1; ++r) own += row_blocks(rows, r);
    tsum[threadIdx.x] = own;
    __syncthreads();
    if (warp == 0) {
        const int run = (nthr + 31) / 32;
        int lsum = 0;
        for (int t = lane * run; t < min(nthr, (lane + 1) * run); ++t) lsum += tsum[t];
        int inc = lsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        int off = inc - lsum;
        for (int t = lane * run; t < min(nthr, (lane + 1) * run); ++t) {
            const int v = tsum[t];
            tsum[t] = off;
            off += v;
        }
        if (lane == 31) tsum[nthr] = inc;
    }
    __syncthreads();
    const long long T = static_cast<long long>(G) * tsum[nthr];
    const long long i0 = T * blockIdx.x / gridDim.x, i1 = T * (blockIdx.x + 1) / gridDim.x;
    if (i0 >= i1) return;
    {
        // the slice holding item i0 walks its rows to find it
        const long long s0 = static_cast<long long>(G) * tsum[threadIdx.x];
        if (own > 0 && s0 <= i0 && i0 < s0 + static_cast<long long>(G) * own) {
            long long c = s0;
            for (int r = r0; r < r1; ++r) {
                const long long n = static_cast<long long>(G) * row_blocks(rows, r);
                if (i0 < c + n) {
                    loc[0] = r;
                    loc[1] = static_cast<int>(i0 - c);
                    break;
                }
                c += n;
            }
        }
    }
    __syncthreads();
    ItemIt it0;
    it0.r = loc[0];
    it0.nb = row_blocks(rows, it0.r);
    it0.g = loc[1] / it0.nb;
    it0.b = loc[1] % it0.nb;
    const int n_items = static_cast<int>(i1 - i0);
    auto advance = [&](ItemIt& x) {
        if (++x.b == x.nb) {
            x.b = 0;
            if (++x.g == G) {
                x.g = 0;
                ++x.r;
                if (x.r < M) x.nb = row_blocks(rows, x.r);
            }
        }
    };

    if (warp == n_cons) {
        // ---------------- producer warp: bulk DMA of K/V chunks into the smem ring
        ItemIt x = it0;
        int i = 0;
        const uint32_t row_bytes = static_cast<uint32_t>(wd) * 2;
        for (int n = 0; n < n_items; ++n, advance(x)) {
            const int ctx_len = rows.ctx_len[x.r];
            const int Lv = ctx_len + rows.chain_len[x.r];
            const long long ctx_base = rows.ctx_base[x.r];
            const long long* chain = rows.chain_slots + static_cast<size_t>(x.r) * kMaxChain;
            const int pre_len = rows.pre_len ? rows.pre_len[x.r] : 0;
            const long long pre_base = rows.pre_len ? rows.pre_base[x.r] : 0;
            const int kb = x.b * kBlock, ke = min(Lv, kb + kBlock);
            const size_t col = static_cast<size_t>(x.g) * wd;
            for (int v0 = kb; v0 < ke; v0 += KPC, ++i) {
                const int s = i % nst;
                if (i >= nst) mbar_wait(&empty[s], ((i / nst) & 1) ^ 1);
                const int v1 = min(ke, v0 + KPC);
                const int nk = v1 - v0;
                const int nctx = max(0, min(v1, ctx_len) - v0);
                if (lane == 0) mbar_arrive_expect_tx(&full[s], 2u * row_bytes * nk);
                __syncwarp();
                __nv_bfloat16* kd = Ks + static_cast<size_t>(s) * KPC * wd;
                __nv_bfloat16* vd = Vs + static_cast<size_t>(s) * KPC * wd;
                if (G == 1) {
                    if (lane == 0 && nctx > 0) {
                        // prompt keys from the group's shared copy, the rest from the row's region
                        const int npre = max(0, min(nctx, pre_len - v0));
                        if (npre > 0) {
                            const size_t src = static_cast<size_t>(pre_base + v0) * d;
                            bulk_g2s(kd, K + src, row_bytes * npre, &full[s]);
                            bulk_g2s(vd, V + src, row_bytes * npre, &full[s]);
                        }
                        if (nctx > npre) {
                            const size_t src = static_cast<size_t>(ctx_base + v0 + npre) * d;
                            bulk_g2s(kd + static_cast<size_t>(npre) * wd, K + src, row_bytes * (nctx - npre), &full[s]);
                            bulk_g2s(vd + static_cast<size_t>(npre) * wd, V + src, row_bytes * (nctx - npre), &full[s]);
                        }
                    }
                    if (lane >= nctx && lane < nk) {
                        const size_t src = static_cast<size_t>(chain[v0 + lane - ctx_len]) * d;
                        bulk_g2s(kd + static_cast<size_t>(lane) * wd, K + src, row_bytes, &full[s]);
                        bulk_g2s(vd + static_cast<size_t>(lane) * wd, V + src, row_bytes, &full[s]);
                    }
                } else if (lane < nk) {
                    const long long slot = lane < nctx ? (v0 + lane < pre_len ? pre_base : ctx_base) + v0 + lane
                                                       : chain[v0 + lane - ctx_len];
                    const size_t src = static_cast<size_t>(slot) * d + col;
                    bulk_g2s(kd + static_cast<size_t>(lane) * wd, K + src, row_bytes, &full[s]);
                    bulk_g2s(vd + static_cast<size_t>(lane) * wd, V + src, row_bytes, &full[s]);
                }
            }
        }
        return;
    }
    if (warp > n_cons) return;

    // ---------------- consumer warps: warp w owns local heads w*HPW .. +HPW-1 of the group
    const int piece = lane % LPR, sub = lane / LPR;
    float qreg[HPW][16];
    float m[HPW], l[HPW], acc[HPW][PL];
    ItemIt x = it0;
    int i = 0, seg_blocks = 0;
    int cur_r = -1, cur_g = -1;
    for (int n = 0; n < n_items; ++n) {
        const int ctx_len = rows.ctx_len[x.r];
        const int Lv = ctx_len + rows.chain_len[x.r];
        const int kb = x.b * kBlock, ke = min(Lv, kb + kBlock);
        if (x.r != cur_r || x.g != cur_g) {
            cur_r = x.r;
            cur_g = x.g;
            seg_blocks = 0;
#pragma unroll
            for (int hh = 0; hh < HPW; ++hh) {
                const int hl = min(warp * HPW + hh, HG - 1);
                const float* qrow = q + static_cast<size_t>(x.r) * d + x.g * wd + hl * DH;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float4 a = *reinterpret_cast<const float4*>(qrow + piece * 16 + 4 * t);
                    qreg[hh][4 * t] = a.x;
                    qreg[hh][4 * t + 1] = a.y;
                    qreg[hh][4 * t + 2] = a.z;
                    qreg[hh][4 * t + 3] = a.w;
                }
            }
        }
#pragma unroll
        for (int hh = 0; hh < HPW; ++hh) {
            m[hh] = -INFINITY;
            l[hh] = 0.f;
#pragma unroll
            for (int e = 0; e < PL; ++e) acc[hh][e] = 0.f;
        }
        for (int v0 = kb; v0 < ke; v0 += KPC, ++i) {
            const int s = i % nst;
            const int nvalid = min(KPC, ke - v0);
            mbar_wait(&full[s], (i / nst) & 1);
            const __nv_bfloat16* kc = Ks + static_cast<size_t>(s) * KPC * wd;
            const __nv_bfloat16* vc = Vs + static_cast<size_t>(s) * KPC * wd;
#pragma unroll
            for (int hh = 0; hh < HPW; ++hh) {
                const int hl = warp * HPW + hh;
                if (hl >= HG) break;
                // scores: RPI key rows per iteration, each lane a 16-dim slice (two LDS.128),
                // LPR-lane butterfly, one shuffle hands key j's score to lane j
                float sc = -INFINITY;
#pragma unroll
                for (int t = 0; t < NIT; ++t) {
                    const int key = t * RPI + sub;
                    const __nv_bfloat16* kr = kc + static_cast<size_t>(key) * wd + hl * DH + piece * 16;
                    const uint4 u0 = *reinterpret_cast<const uint4*>(kr);
                    const uint4 u1 = *reinterpret_cast<const uint4*>(kr + 8);
                    const __nv_bfloat162* b0 = reinterpret_cast<const __nv_bfloat162*>(&u0);
                    const __nv_bfloat162* b1 = reinterpret_cast<const __nv_bfloat162*>(&u1);
                    float dot = 0.f;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = __bfloat1622float2(b0[e]);
                        dot = fmaf(qreg[hh][2 * e], f.x, dot);
                        dot = fmaf(qreg[hh][2 * e + 1], f.y, dot);
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 f = __bfloat1622float2(b1[e]);
                        dot = fmaf(qreg[hh][8 + 2 * e], f.x, dot);
                        dot = fmaf(qreg[hh][8 + 2 * e + 1], f.y, dot);
                    }
#pragma unroll
                    for (int o = LPR / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                    const float dr = __shfl_sync(0xffffffffu, dot, (lane % RPI) * LPR);
                    if (lane / RPI == t && lane < nvalid) sc = attn_scale(dr, scale);
                }
                const float cm = warp_max(sc);
                const float nm = fmaxf(m[hh], cm);
                const float alpha = attn_alpha(m[hh], nm);
                const float p = (lane < nvalid) ? attn_p(sc, nm) : 0.f;
                l[hh] = attn_l(l[hh], alpha, warp_sum(p));
#pragma unroll
                for (int e = 0; e < PL; ++e) acc[hh][e] = __fmul_rn(acc[hh][e], alpha);
                m[hh] = nm;
#pragma unroll
                for (int j = 0; j < KPC; ++j) {
                    const float pj = __shfl_sync(0xffffffffu, p, j);
                    if (j < nvalid) {
                        const __nv_bfloat16* vr = vc + static_cast<size_t>(j) * wd + hl * DH + lane * PL;
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
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        // end of the 64-key block: publish its partial
#pragma unroll
        for (int hh = 0; hh < HPW; ++hh) {
            const int hl = warp * HPW + hh;
            if (hl >= HG) break;
            const size_t pidx = (static_cast<size_t>(x.r) * nb_max + x.b) * H + x.g * HG + hl;
            float* pa = part_acc + pidx * DH + lane * PL;
#pragma unroll
            for (int e = 0; e < PL; ++e) pa[e] = acc[hh][e];
            if (lane == 0) {
                part_ml[2 * pidx] = m[hh];
                part_ml[2 * pidx + 1] = l[hh];
            }
        }
        ++seg_blocks;
        const ItemIt done = x;
        advance(x);
        const bool seg_end = (n + 1 == n_items) || x.r != done.r || x.g != done.g;
        if (!seg_end) continue;
        // ---- segment end: ticket on (row, group); the completing CTA merges the row
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"r"(n_cons * 32) : "memory");
        if (threadIdx.x == 0) {
            int* c = row_ctr + static_cast<size_t>(done.r) * G + done.g;
            const int old = atomicAdd(c, seg_blocks);
            const int last = (old + seg_blocks == done.nb);
            if (last) *c = 0;  // re-armed for the next launch
            *flag = last;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(n_cons * 32) : "memory");
        if (!*flag) continue;
        __threadfence();
#pragma unroll
        for (int hh = 0; hh < HPW; ++hh) {
            const int hl = warp * HPW + hh;
            if (hl >= HG) break;
            const int h = done.g * HG + hl;
            // merge from the identity (-inf, 0, 0): the first merge reproduces partial 0
            // exactly, so this equals "start from block 0"; loads are batched 8 blocks at
            // a time so the serial tail is the arithmetic, not 8 L2 round trips
            float Mx = -INFINITY, Lx = 0.f, A[PL];
#pragma unroll
            for (int e0 = 0; e0 < PL; ++e0) A[e0] = 0.f;
            constexpr int kMB = 4;
            for (int b0 = 0; b0 < done.nb; b0 += kMB) {
                float mb[kMB], lb[kMB], ab[kMB][PL];
#pragma unroll
                for (int u = 0; u < kMB; ++u) {
                    const int b = min(b0 + u, done.nb - 1);
                    const size_t pidx = (static_cast<size_t>(done.r) * nb_max + b) * H + h;
                    mb[u] = __ldcg(part_ml + 2 * pidx);
                    lb[u] = __ldcg(part_ml + 2 * pidx + 1);
                    if constexpr (PL == 4) {
                        const float4 t = __ldcg(reinterpret_cast<const float4*>(part_acc + pidx * DH + lane * PL));
                        ab[u][0] = t.x; ab[u][1] = t.y; ab[u][2] = t.z; ab[u][3] = t.w;
                    } else {
#pragma unroll
                        for (int e0 = 0; e0 < PL; ++e0) ab[u][e0] = __ldcg(part_acc + pidx * DH + lane * PL + e0);
                    }
                }
#pragma unroll
                for (int u = 0; u < kMB; ++u) {
                    if (b0 + u < done.nb) attn_merge<PL>(Mx, Lx, A, mb[u], lb[u], ab[u]);
                }
            }
#pragma unroll
            for (int e0 = 0; e0 < PL; ++e0) {
                const int e = lane * PL + e0;
                out[static_cast<size_t>(done.r) * d + h * DH + e] = __float2bfloat16(__fdiv_rn(A[e0], Lx));
            }
        }
    }
}

template <int DH, int KPC, int HPW>
void launch_impl(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, int M,
                 int H, int d, int G, int nb_max, long long est_items, const AttnScratch& sc, __nv_bfloat16* out,
                 cudaStream_t st) {
    const int HG = H / G;
    const int wd = HG * DH;
    const int n_cons = (HG + HPW - 1) / HPW;
    const int threads = 32 * (n_cons + 1);
    const size_t fixed = static_cast<size_t>(8 * 4 + 16 + 4 * (threads + 3)) + 128;
    const size_t stage = 2 * static_cast<size_t>(KPC) * wd * 2;
    // two CTAs per SM when two 2-stage rings fit (more warps to hide the consumers'
    // shuffle / shared-memory latency), else one CTA with up to 4 stages
    const int per_sm = (2 * (2 * stage + fixed) <= static_cast<size_t>(kSmemBudget)) ? 2 : 1;
    const int nst = static_cast<int>(std::min<size_t>(4, (kSmemBudget / per_sm - fixed) / stage));
    if (nst < 2) throw std::invalid_argument("attention: shared memory too small for the model width");
    const size_t smem = nst * stage + fixed;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_kernel<DH, KPC, HPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemBudget));
        attr = true;
    }
    const int fit = std::max(1, std::min(8, static_cast<int>(kSmemBudget / smem)));
    const long long grid = std::max(1LL, std::min<long long>(est_items, 148LL * fit));
    launch_pdl(attn_kernel<DH, KPC, HPW>, dim3(static_cast<unsigned>(grid)), dim3(threads), smem, st, q, K, V, rows, M,
               H, d, G, nst, nb_max, 1.0f / sqrtf(static_cast<float>(DH)), sc.part_acc, sc.part_ml, sc.row_ctr, out);
}

}  // namespace

int attn_splits_for(int max_virtual_len) { return (max_virtual_len + kBlock - 1) / kBlock; }

void launch_attention(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, int M,
                      int H, int d, int max_virtual_len, double total_keys, const AttnScratch& sc, __nv_bfloat16* out,
                      cudaStream_t st) {
    if (M <= 0) return;
    if (M > kMaxScanRows) throw std::invalid_argument("attention: too many rows in one launch");
    const int dh = d / H;
    const int nb = attn_splits_for(max_virtual_len);
    if (H > 32) throw std::invalid_argument("attention: at most 32 heads");
    if (static_cast<long long>(M) * H > sc.ctr_cap) throw std::invalid_argument("attention: row tickets too small");
    // chunk size KPC is fixed per model width; it is part of the numerics, never a
    // function of the batch
    const int kpc = d <= 3328 ? 8 : 4;
    // head groups: split the heads only when the launch has too few blocks to cover the SMs
    const long long blocks = static_cast<long long>(total_keys / kBlock) + M;
    int G = 1;
    while (G < H && blocks * G < 2 * 148) {
        int g2 = G + 1;
        while (H % g2) ++g2;
        G = g2;
    }
    static const int g_force = [] {
        const char* v = getenv("SGB_ATTN_G");  // tuning experiments only
        return v ? atoi(v) : 0;
    }();
    if (g_force > 0 && H % g_force == 0) G = g_force;
    const int HG = H / G;
    const bool two = HG > 12;  // one head per warp up to 12 heads (two CTAs per SM fit)
    const long long est = blocks * G;
#define SGB_ATT(DH_, KPC_, HPW_) \
    launch_impl<DH_, KPC_, HPW_>(q, K, V, rows, M, H, d, G, nb, est, sc, out, st)
    if (dh == 128 && kpc == 8) { if (two) SGB_ATT(128, 8, 2); else SGB_ATT(128, 8, 1); }
    else if (dh == 128 && kpc == 4) { if (two) SGB_ATT(128, 4, 2); else SGB_ATT(128, 4, 1); }
    else if (dh == 64 && kpc == 8) { if (two) SGB_ATT(64, 8, 2); else SGB_ATT(64, 8, 1); }
#undef SGB_ATT
    else throw std::invalid_argument("attention: head dim must be 64 or 128");
    SGB_KCHECK();
}

}  // namespace sgb
