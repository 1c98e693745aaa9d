// Tree-verify attention: the rows of one sequence's draft tree against its committed prefix
// plus each row's own ancestor path -- the verify forward of a speculative step and the batched
// draft-level forwards (decode_blocks, include/sgrpo/tinylm.hpp:335-395, with the tree mask of
// build_tree_mask, drafttree.cpp:145-168).
//
// Why a separate kernel. attention.cu serves every row shape through one persistent work list
// of (tile <= 16 rows, head group, 64-key block) items whose block partials are merged through
// global memory; for ~200 tree rows over a few hundred prefix keys that list is thousands of
// tiny items and the kernel is latency-bound (ncu: DRAM 0.8 %, 23 % occupancy,
// profiles/r01_verify_attn_c3_m211.txt). Here one CTA owns (sequence, head, tile of up to 64
// rows) for the WHOLE key range: the prefix streams once per tile through a TMA ring (16-key x
// 64-dim SWIZZLE_128B boxes straight from the paged K/V store), the tree nodes' own K/V rows
// (the keys of every row's path) are loaded once into shared memory, and the per-64-key-block
// partials are merged in registers -- no partials in HBM, no tickets.
//
// Bit-identical to attention.cu (batch invariance): a row's virtual key sequence
// is [prefix 0..P) then its path (ancestors root-first, then itself), chunked in 16-key steps
// of 64-key blocks at the same virtual offsets; the chunk arithmetic (mma.sync S^T = K.Q^T with
// keys in M, online softmax with the same explicit-rounding steps and shuffle trees, P^T via
// movmatrix, O^T += V^T.P^T) and the in-order block merge (attn_merge from the identity) are
// the same operations on the same operands. Chunks wholly inside the prefix are shared by all
// rows of the tile (every column live); a chunk that reaches past P is run once per row with
// only that row's query column live (-inf scores on the others are exact no-ops, as in
// attention.cu's boundary tiles), its key rows gathered per lane by ldmatrix addresses: prefix
// keys from the staged ring, path keys from the node table.
#include <algorithm>
#include <array>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <cfloat>

#include <cooperative_groups.h>

#include "attn_numerics.cuh"
#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace cg = cooperative_groups;

namespace {

constexpr int kTBlock = kAttnBlock;  // 64 keys per softmax partial
constexpr int kTChunk = 16;          // keys per staged chunk
constexpr int kTMaxWarps = 8;        // consumer warps (8 query rows each)
constexpr int kTSmem = 227 * 1024;
#ifndef SGB_TREE_ONE_WARP_CTAS
#define SGB_TREE_ONE_WARP_CTAS 7
#endif
constexpr int kTOneWarpCtas = SGB_TREE_ONE_WARP_CTAS;  // CTAs per SM of the one-warp tree kernel

SGB_DEV void ldsm_x4(uint32_t addr, uint32_t* r) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
SGB_DEV void ldsm_x4_t(uint32_t addr, uint32_t* r) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
SGB_DEV uint32_t movm_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
SGB_DEV void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
SGB_DEV uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}
SGB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// smem address of dims [dd, dd+8) of key row kr in a staged chunk: DH/64 SWIZZLE_128B boxes of
// 16 rows x 128 B (16-byte unit u of row r stored at unit u ^ (r & 7))
SGB_DEV uint32_t ring_addr(uint32_t stage, int kr, int dd) {
    const int box = dd >> 6, u = (dd & 63) >> 3;
    return stage + static_cast<uint32_t>(box * 2048 + kr * 128 + ((u ^ (kr & 7)) << 4));
}

// MAXW: the consumer warps a launch may use. The one-warp instantiation (tiles of <= 8 rows, the
// c5 verify shape: 4 rows per sequence) is register-capped so that 7 CTAs fit an SM (with 168
// registers 6 did, and 1,024 CTAs took 1.15 waves); the code and so the bits are the same
template <int DH, int MAXW>
__global__ void __launch_bounds__(32 * (MAXW + 1), MAXW == 1 ? kTOneWarpCtas : 1)
    tree_attn_kernel(const float* __restrict__ q, const __grid_constant__ CUtensorMap kmap,
                     const __grid_constant__ CUtensorMap vmap, long long layer_row0, const __nv_bfloat16* __restrict__ K,
                     const __nv_bfloat16* __restrict__ V, AttnRowsDev rows, const TreeGroupDev* __restrict__ groups,
                     const TreeTileDev* __restrict__ tiles, int d, int nst, int tbl_cap, float scale,
                     __nv_bfloat16* __restrict__ out) {
    constexpr int NK = DH / 16;
    constexpr uint32_t kStageK = static_cast<uint32_t>(kTChunk) * DH * 2;  // one of K or V per stage
    constexpr int kRowB = DH * 2 + 16;                                    // padded node-table row
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // SWIZZLE_128B TMA destinations need 1024-byte alignment
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int W = static_cast<int>(blockDim.x >> 5) - 1;  // consumer warps
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const TreeTileDev tt = tiles[blockIdx.x];
    const TreeGroupDev gr = groups[tt.group];
    const int h = blockIdx.y;
    const int P = gr.ctx_len;
    uint8_t* ringK = smem;                                    // [nst][16][DH] swizzled
    uint8_t* ringV = smem + static_cast<size_t>(nst) * kStageK;
    uint8_t* tblK = ringV + static_cast<size_t>(nst) * kStageK;  // [tbl_cap][kRowB]
    uint8_t* tblV = tblK + static_cast<size_t>(tbl_cap) * kRowB;
    uint64_t* full = reinterpret_cast<uint64_t*>(tblV + static_cast<size_t>(tbl_cap) * kRowB);
    uint64_t* empty = full + nst;
    uint64_t* tbar = empty + nst;
    int* chains = reinterpret_cast<int*>(tbar + 1);  // [W][8 rows][lv + 8 path node indices]
    const int n_prefix_chunks = (P + kTChunk - 1) / kTChunk;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], W);
        }
        mbar_init(tbar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    pdl_wait();  // q and this layer's K/V (incl. the tree rows') come from the previous kernels
    pdl_trigger();

    if (warp == W) {
        // ---------------- producer: node table (bulk rows), then the prefix chunks (TMA ring)
        const int nn = gr.n_nodes;
        const uint32_t rowbytes = DH * 2;
        if (lane == 0) mbar_arrive_expect_tx(tbar, 2u * rowbytes * nn);
        __syncwarp();
        for (int i = lane; i < nn; i += 32) {
            const size_t src = static_cast<size_t>(gr.node_base + i) * d + static_cast<size_t>(h) * DH;
            bulk_g2s(tblK + static_cast<size_t>(i) * kRowB, K + src, rowbytes, tbar);
            bulk_g2s(tblV + static_cast<size_t>(i) * kRowB, V + src, rowbytes, tbar);
        }
        if (lane == 0) {
            int s = 0, ph = 0;  // ring stage and its phase (no integer division in the loop)
            for (int c = 0; c < n_prefix_chunks; ++c, s = s + 1 == nst ? 0 : s + 1, ph ^= s == 0) {
                if (c >= nst) mbar_wait(&empty[s], ph ^ 1);
                const int v0 = c * kTChunk;
                // the shared prompt copy (identical values) while the whole box lies in it
                const long long slot0 = (v0 + kTChunk <= gr.pre_len ? gr.pre_base : gr.ctx_base) + v0;
                const int row = static_cast<int>(layer_row0 + slot0);
                mbar_arrive_expect_tx(&full[s], 2 * kStageK);
#pragma unroll
                for (int b = 0; b < DH / 64; ++b) {
                    tma_load_2d(ringK + static_cast<size_t>(s) * kStageK + b * 2048, &kmap, &full[s], h * DH + 64 * b, row);
                    tma_load_2d(ringV + static_cast<size_t>(s) * kStageK + b * 2048, &vmap, &full[s], h * DH + 64 * b, row);
                }
            }
        }
        return;
    }

    // ---------------- consumers: warp w owns tile rows [8w, 8w + 8) as the 8 query columns
    const int g8 = lane >> 2, t4 = lane & 3;
    const int li = lane >> 3, lr = lane & 7;
    const int row0 = gr.row0 + tt.r0 + 8 * warp;
    const int nrows = max(0, min(8, tt.nr - 8 * warp));
    uint32_t qf[NK][2];
    {
        const int qrow = nrows > 0 ? row0 + min(g8, nrows - 1) : gr.row0;
        const float* qr = q + static_cast<size_t>(qrow) * d + h * DH + 2 * t4;
#pragma unroll
        for (int ks = 0; ks < NK; ++ks) {
            const float2 a = __ldg(reinterpret_cast<const float2*>(qr + 16 * ks));
            const float2 b = __ldg(reinterpret_cast<const float2*>(qr + 16 * ks + 8));
            qf[ks][0] = pack_bf16(a.x, a.y);
            qf[ks][1] = pack_bf16(b.x, b.y);
        }
    }
    // the warp's rows: virtual length and path node indices (shared memory, read per chunk)
    int* wchain = chains + warp * 72;
    for (int x = lane; x < 72; x += 32) {
        const int j = x / 9, f = x % 9;
        int val = 0;
        if (j < nrows) {
            const int cl = rows.chain_len[row0 + j];
            val = f == 0 ? P + cl
                         : (f - 1 < cl ? static_cast<int>(rows.chain_slots[static_cast<size_t>(row0 + j) * kMaxChain + f - 1] -
                                                          gr.node_base)
                                       : 0);
        }
        wchain[x] = val;
    }
    __syncwarp();
    // virtual lengths of this lane's two query columns, and of the warp's rows
    const int c0 = 2 * t4, c1 = 2 * t4 + 1;
    const int lv0 = c0 < nrows ? P + rows.chain_len[row0 + c0] : 0;
    const int lv1 = c1 < nrows ? P + rows.chain_len[row0 + c1] : 0;
    int lvmax = max(lv0, lv1);
#pragma unroll
    for (int o2 = 1; o2 < 4; o2 <<= 1) lvmax = max(lvmax, __shfl_xor_sync(0xffffffffu, lvmax, o2));
    const uint32_t ringK0 = smem_u32(ringK), ringV0 = smem_u32(ringV);
    const uint32_t tblK0 = smem_u32(tblK), tblV0 = smem_u32(tblV);
    // merged state of the two columns (attn_merge from the identity), o layout as attention.cu
    float M0 = -INFINITY, M1 = -INFINITY, L0 = 0.f, L1 = 0.f;
    float A[NK][4];
#pragma unroll
    for (int mt = 0; mt < NK; ++mt) A[mt][0] = A[mt][1] = A[mt][2] = A[mt][3] = 0.f;
    bool tbl_ready = false;
    int i = 0, si = 0, ph = 0;  // staged chunk counter, its ring stage and phase
    const int nb = (lvmax + kTBlock - 1) / kTBlock;
    const int nbp = (P + kTBlock - 1) / kTBlock;  // blocks holding prefix keys: every warp runs them
    for (int b = 0; b < max(nb, nbp); ++b) {
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        float o[NK][4];
#pragma unroll
        for (int mt = 0; mt < NK; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
        // one chunk: kaddr / vaddr give the smem row of key slot kr; e0 / e1 = key end of the
        // lane's two query columns
        auto chunk = [&](auto kaddr, auto vaddr, int v0, int e0, int e1) {
            float sc[4] = {0.f, 0.f, 0.f, 0.f};
            const int kr_k = lr + 8 * (li & 1);
#pragma unroll
            for (int ks = 0; ks < NK; ++ks) {
                uint32_t a[4];
                ldsm_x4(kaddr(kr_k, 16 * ks + 8 * (li >> 1)), a);
                mma16816(sc, a, qf[ks][0], qf[ks][1]);
            }
            const bool va0 = v0 + g8 < e0, va1 = v0 + g8 < e1, vb0 = v0 + g8 + 8 < e0, vb1 = v0 + g8 + 8 < e1;
            const float s0 = va0 ? attn_scale(sc[0], scale) : -INFINITY;
            const float s1 = va1 ? attn_scale(sc[1], scale) : -INFINITY;
            const float s2 = vb0 ? attn_scale(sc[2], scale) : -INFINITY;
            const float s3 = vb1 ? attn_scale(sc[3], scale) : -INFINITY;
            float x0 = fmaxf(s0, s2), x1 = fmaxf(s1, s3);
#pragma unroll
            for (int o2 = 4; o2 < 32; o2 <<= 1) {
                x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, o2));
                x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o2));
            }
            const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);
            const float a0 = attn_alpha(m0, n0), a1 = attn_alpha(m1, n1);
            const float p0 = va0 ? attn_p(s0, n0) : 0.f, p1 = va1 ? attn_p(s1, n1) : 0.f;
            const float p2 = vb0 ? attn_p(s2, n0) : 0.f, p3 = vb1 ? attn_p(s3, n1) : 0.f;
            float ps0 = __fadd_rn(p0, p2), ps1 = __fadd_rn(p1, p3);
#pragma unroll
            for (int o2 = 4; o2 < 32; o2 <<= 1) {
                ps0 = __fadd_rn(ps0, __shfl_xor_sync(0xffffffffu, ps0, o2));
                ps1 = __fadd_rn(ps1, __shfl_xor_sync(0xffffffffu, ps1, o2));
            }
            l0 = attn_l(l0, a0, ps0);
            l1 = attn_l(l1, a1, ps1);
            m0 = n0;
            m1 = n1;
            uint32_t va4[NK][4];
            const int kr_v = lr + 8 * (li >> 1);
#pragma unroll
            for (int mt = 0; mt < NK; ++mt) ldsm_x4_t(vaddr(kr_v, 16 * mt + 8 * (li & 1)), va4[mt]);
            const uint32_t b0 = movm_t(pack_bf16(p0, p1)), b1 = movm_t(pack_bf16(p2, p3));
#pragma unroll
            for (int mt = 0; mt < NK; ++mt) {
                o[mt][0] = __fmul_rn(o[mt][0], a0);
                o[mt][1] = __fmul_rn(o[mt][1], a1);
                o[mt][2] = __fmul_rn(o[mt][2], a0);
                o[mt][3] = __fmul_rn(o[mt][3], a1);
                mma16816(o[mt], va4[mt], b0, b1);
            }
        };
        for (int c = 0; c < kTBlock / kTChunk; ++c) {
            const int v0 = b * kTBlock + c * kTChunk;
            if (v0 >= max(lvmax, P)) break;
            const bool staged = v0 < P;
            uint32_t sK = 0, sV = 0;
            int s = 0;
            if (staged) {
                s = si;
                mbar_wait(&full[s], ph);
                sK = ringK0 + static_cast<uint32_t>(s) * kStageK;
                sV = ringV0 + static_cast<uint32_t>(s) * kStageK;
            }
            if (v0 + kTChunk <= P) {
                // shared prefix chunk: every query column live
                auto ka = [&](int kr, int dd) { return ring_addr(sK, kr, dd); };
                auto vaa = [&](int kr, int dd) { return ring_addr(sV, kr, dd); };
                chunk(ka, vaa, v0, lv0, lv1);
            } else if (nrows > 0) {
                // past the prefix: once per row, its own path keys gathered from the node table
                if (!tbl_ready) {
                    mbar_wait(tbar, 0);
                    tbl_ready = true;
                }
                for (int j = 0; j < nrows; ++j) {
                    const int* wc = wchain + j * 9;  // [lv, node of path key 0..7]
                    const int lvj = wc[0];
                    if (lvj <= v0) continue;
                    // this lane's two key slots (K: kr_k, V: kr_v): prefix rows from the ring,
                    // path rows from the node table, past the row's end any finite row (p = 0)
                    const int vk = v0 + lr + 8 * (li & 1), vv = v0 + lr + 8 * (li >> 1);
                    const uint32_t kt = tblK0 + static_cast<uint32_t>((vk >= P && vk < lvj ? wc[1 + vk - P] : 0) * kRowB);
                    const uint32_t vt = tblV0 + static_cast<uint32_t>((vv >= P && vv < lvj ? wc[1 + vv - P] : 0) * kRowB);
                    auto ka = [&](int kr, int dd) { return vk < P ? ring_addr(sK, kr, dd) : kt + static_cast<uint32_t>(dd * 2); };
                    auto vaa = [&](int kr, int dd) { return vv < P ? ring_addr(sV, kr, dd) : vt + static_cast<uint32_t>(dd * 2); };
                    chunk(ka, vaa, v0, c0 == j ? lvj : v0, c1 == j ? lvj : v0);
                }
            }
            if (staged) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                ++i;
                if (++si == nst) {
                    si = 0;
                    ph ^= 1;
                }
            }
        }
        // ordered merge of this block's partial (rows whose keys reach into block b)
        const bool h0 = b * kTBlock < lv0, h1 = b * kTBlock < lv1;
        if (h0) {
            const float Mn = fmaxf(M0, m0);
            const float ca = M0 == -INFINITY ? 0.f : expf(__fsub_rn(M0, Mn));
            const float cb = expf(__fsub_rn(m0, Mn));
            L0 = fmaf(L0, ca, __fmul_rn(l0, cb));
#pragma unroll
            for (int mt = 0; mt < NK; ++mt) {
                A[mt][0] = fmaf(A[mt][0], ca, __fmul_rn(o[mt][0], cb));
                A[mt][2] = fmaf(A[mt][2], ca, __fmul_rn(o[mt][2], cb));
            }
            M0 = Mn;
        }
        if (h1) {
            const float Mn = fmaxf(M1, m1);
            const float ca = M1 == -INFINITY ? 0.f : expf(__fsub_rn(M1, Mn));
            const float cb = expf(__fsub_rn(m1, Mn));
            L1 = fmaf(L1, ca, __fmul_rn(l1, cb));
#pragma unroll
            for (int mt = 0; mt < NK; ++mt) {
                A[mt][1] = fmaf(A[mt][1], ca, __fmul_rn(o[mt][1], cb));
                A[mt][3] = fmaf(A[mt][3], ca, __fmul_rn(o[mt][3], cb));
            }
            M1 = Mn;
        }
    }
    // outputs of the real columns
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
        const int qc = 2 * t4 + cc;
        if (qc >= nrows) continue;
        const float Lx = cc ? L1 : L0;
        __nv_bfloat16* orow = out + static_cast<size_t>(row0 + qc) * d + h * DH;
#pragma unroll
        for (int mt = 0; mt < NK; ++mt) {
            orow[16 * mt + g8] = __float2bfloat16(__fdiv_rn(A[mt][cc], Lx));
            orow[16 * mt + g8 + 8] = __float2bfloat16(__fdiv_rn(A[mt][2 + cc], Lx));
        }
    }
}

// ------------------------------------------------------------------ few-row decode (AR steps)
// One row per group (an AR step: the row's keys are its committed prefix plus its own new key).
// The per-row kernels above stream a row's whole context through one warp; here the 64-key
// blocks of a (row, head) are spread over the S CTAs of a thread-block cluster and their W warps
// (contiguous block ranges per CTA, warp w of a CTA takes every W-th block of the range), each
// block's partial (m, l, o) goes to shared memory, and CTA 0 of the cluster merges the partials
// strictly in block order through distributed shared memory -- the same chunk arithmetic and
// the same ordered merge from the identity as tree_attn_kernel / attention.cu, so the bits are
// those of every other attention path. Each warp streams its own chunks through a private
// NS-stage TMA ring (no producer warp: one lane issues the next chunk when a stage frees up).
// measured (scripts/bench_decode_attn.py): 8 warps x 2 stages pushes the small-B launches to one
// CTA per SM (two waves at B = 1); 4 x 3 keeps two CTAs per SM
constexpr int kDW = 4;   // warps per CTA
constexpr int kDNS = 3;  // ring stages per warp (16 keys of K and V each)

template <int DH>
struct DecodeSmem {
    static constexpr uint32_t kStage = 2u * kTChunk * DH * 2;  // K then V, swizzled boxes
    static constexpr int kRowB = DH * 2 + 16;
    static size_t bytes(int max_blocks) {
        return 1024 + static_cast<size_t>(kDW) * kDNS * kStage + 2 * kRowB +
               static_cast<size_t>(max_blocks) * (DH + 2) * 4 + 8 * (kDW * kDNS + 1);
    }
};

template <class KA, class VA, int NK>
SGB_DEV void decode_chunk(KA kaddr, VA vaddr, int v0, int e0, int e1, const uint32_t (&qf)[NK][2], float scale,
                          float& m0, float& m1, float& l0, float& l1, float (&o)[NK][4], int lane) {
    const int g8 = lane >> 2, li = lane >> 3, lr = lane & 7;
    float sc[4] = {0.f, 0.f, 0.f, 0.f};
    const int kr_k = lr + 8 * (li & 1);
#pragma unroll
    for (int ks = 0; ks < NK; ++ks) {
        uint32_t a[4];
        ldsm_x4(kaddr(kr_k, 16 * ks + 8 * (li >> 1)), a);
        mma16816(sc, a, qf[ks][0], qf[ks][1]);
    }
    const bool va0 = v0 + g8 < e0, va1 = v0 + g8 < e1, vb0 = v0 + g8 + 8 < e0, vb1 = v0 + g8 + 8 < e1;
    const float s0 = va0 ? attn_scale(sc[0], scale) : -INFINITY;
    const float s1 = va1 ? attn_scale(sc[1], scale) : -INFINITY;
    const float s2 = vb0 ? attn_scale(sc[2], scale) : -INFINITY;
    const float s3 = vb1 ? attn_scale(sc[3], scale) : -INFINITY;
    float x0 = fmaxf(s0, s2), x1 = fmaxf(s1, s3);
#pragma unroll
    for (int o2 = 4; o2 < 32; o2 <<= 1) {
        x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, o2));
        x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o2));
    }
    const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);
    const float a0 = attn_alpha(m0, n0), a1 = attn_alpha(m1, n1);
    const float p0 = va0 ? attn_p(s0, n0) : 0.f, p1 = va1 ? attn_p(s1, n1) : 0.f;
    const float p2 = vb0 ? attn_p(s2, n0) : 0.f, p3 = vb1 ? attn_p(s3, n1) : 0.f;
    float ps0 = __fadd_rn(p0, p2), ps1 = __fadd_rn(p1, p3);
#pragma unroll
    for (int o2 = 4; o2 < 32; o2 <<= 1) {
        ps0 = __fadd_rn(ps0, __shfl_xor_sync(0xffffffffu, ps0, o2));
        ps1 = __fadd_rn(ps1, __shfl_xor_sync(0xffffffffu, ps1, o2));
    }
    l0 = attn_l(l0, a0, ps0);
    l1 = attn_l(l1, a1, ps1);
    m0 = n0;
    m1 = n1;
    uint32_t va4[NK][4];
    const int kr_v = lr + 8 * (li >> 1);
#pragma unroll
    for (int mt = 0; mt < NK; ++mt) ldsm_x4_t(vaddr(kr_v, 16 * mt + 8 * (li & 1)), va4[mt]);
    const uint32_t b0 = movm_t(pack_bf16(p0, p1)), b1 = movm_t(pack_bf16(p2, p3));
#pragma unroll
    for (int mt = 0; mt < NK; ++mt) {
        o[mt][0] = __fmul_rn(o[mt][0], a0);
        o[mt][1] = __fmul_rn(o[mt][1], a1);
        o[mt][2] = __fmul_rn(o[mt][2], a0);
        o[mt][3] = __fmul_rn(o[mt][3], a1);
        mma16816(o[mt], va4[mt], b0, b1);
    }
}

template <int DH>
__global__ void __launch_bounds__(32 * kDW)
    decode_attn_kernel(const float* __restrict__ q, const __grid_constant__ CUtensorMap kmap,
                       const __grid_constant__ CUtensorMap vmap, long long layer_row0, const __nv_bfloat16* __restrict__ K,
                       const __nv_bfloat16* __restrict__ V, const TreeGroupDev* __restrict__ groups, int S,
                       int max_blocks, int d, float scale, __nv_bfloat16* __restrict__ out) {
    constexpr int NK = DH / 16;
    using Sm = DecodeSmem<DH>;
    constexpr uint32_t kHalf = kTChunk * DH * 2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x / S, rank = blockIdx.x % S, h = blockIdx.y;
    const TreeGroupDev gr = groups[g];
    const int P = gr.ctx_len, lv = P + 1;  // prefix keys, then the row's own key (node 0)
    const int nb = (lv + kTBlock - 1) / kTBlock;
    const int b_lo = static_cast<int>(static_cast<long long>(rank) * nb / S);
    const int b_hi = static_cast<int>(static_cast<long long>(rank + 1) * nb / S);
    uint8_t* ring = smem + static_cast<size_t>(warp) * kDNS * Sm::kStage;
    uint8_t* nodeK = smem + static_cast<size_t>(kDW) * kDNS * Sm::kStage;
    uint8_t* nodeV = nodeK + Sm::kRowB;
    float* part = reinterpret_cast<float*>(nodeV + Sm::kRowB);  // [max_blocks][DH + 2]: o, m, l
    uint64_t* full = reinterpret_cast<uint64_t*>(part + static_cast<size_t>(max_blocks) * (DH + 2));
    uint64_t* tbar = full + kDW * kDNS;
    uint64_t* wfull = full + warp * kDNS;
    if (threadIdx.x == 0) {
        tma_prefetch(&kmap);
        tma_prefetch(&vmap);
        for (int s = 0; s < kDW * kDNS; ++s) mbar_init(&full[s], 1);
        mbar_init(tbar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) {
        const size_t src = static_cast<size_t>(gr.node_base) * d + static_cast<size_t>(h) * DH;
        mbar_arrive_expect_tx(tbar, 2u * DH * 2);
        bulk_g2s(nodeK, K + src, DH * 2, tbar);
        bulk_g2s(nodeV, V + src, DH * 2, tbar);
    }
    // this warp's staged chunks (keys below P) in order: block b_lo + warp + k * kDW, chunk c
    auto staged_of = [&](int b) { return min(4, max(0, (P - b * kTBlock + kTChunk - 1) / kTChunk)); };
    int ib = b_lo + warp, ic = 0;  // issue cursor
    auto advance = [&]() {
        if (++ic >= staged_of(ib)) {
            ic = 0;
            ib += kDW;
        }
    };
    while (ib < b_hi && staged_of(ib) == 0) ib += kDW;
    auto issue = [&](int st) {
        const int v0 = ib * kTBlock + ic * kTChunk;
        const long long slot0 = (v0 + kTChunk <= gr.pre_len ? gr.pre_base : gr.ctx_base) + v0;
        const int row = static_cast<int>(layer_row0 + slot0);
        uint8_t* dst = ring + static_cast<size_t>(st) * Sm::kStage;
        mbar_arrive_expect_tx(&wfull[st], Sm::kStage);
#pragma unroll
        for (int bx = 0; bx < DH / 64; ++bx) {
            tma_load_2d(dst + bx * 2048, &kmap, &wfull[st], h * DH + 64 * bx, row);
            tma_load_2d(dst + kHalf + bx * 2048, &vmap, &wfull[st], h * DH + 64 * bx, row);
        }
        advance();
        while (ib < b_hi && staged_of(ib) == 0) ib += kDW;
    };
    if (lane == 0)
        for (int st = 0; st < kDNS && ib < b_hi; ++st) issue(st);
    __syncwarp();
    // q fragment: every column reads the row (columns past the first are dead: e = v0)
    const int g8 = lane >> 2, t4 = lane & 3, li = lane >> 3, lr = lane & 7;
    uint32_t qf[NK][2];
    {
        const float* qr = q + static_cast<size_t>(gr.row0) * d + h * DH + 2 * t4;
#pragma unroll
        for (int ks = 0; ks < NK; ++ks) {
            const float2 a = __ldg(reinterpret_cast<const float2*>(qr + 16 * ks));
            const float2 b = __ldg(reinterpret_cast<const float2*>(qr + 16 * ks + 8));
            qf[ks][0] = pack_bf16(a.x, a.y);
            qf[ks][1] = pack_bf16(b.x, b.y);
        }
    }
    const int lv0 = t4 == 0 ? lv : 0;  // query column 0 is the row
    const uint32_t node_k = smem_u32(nodeK), node_v = smem_u32(nodeV);
    int i = 0, si = 0, ph = 0;  // consumed staged chunks, ring stage, phase
    bool node_ready = false;
    for (int b = b_lo + warp; b < b_hi; b += kDW) {
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        float o[NK][4];
#pragma unroll
        for (int mt = 0; mt < NK; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
        for (int c = 0; c < kTBlock / kTChunk; ++c) {
            const int v0 = b * kTBlock + c * kTChunk;
            if (v0 >= lv) break;
            const bool staged = v0 < P;
            uint32_t sK = 0, sV = 0;
            if (staged) {
                mbar_wait(&wfull[si], ph);
                sK = smem_u32(ring) + static_cast<uint32_t>(si) * Sm::kStage;
                sV = sK + kHalf;
            }
            if (v0 + kTChunk <= P) {
                auto ka = [&](int kr, int dd) { return ring_addr(sK, kr, dd); };
                auto vaa = [&](int kr, int dd) { return ring_addr(sV, kr, dd); };
                decode_chunk(ka, vaa, v0, lv0, 0, qf, scale, m0, m1, l0, l1, o, lane);
            } else {
                if (!node_ready) {
                    mbar_wait(tbar, 0);
                    node_ready = true;
                }
                // prefix keys from the ring, the row's own key (v == P) from the node row, past it
                // any finite row (p = 0)
                const int vk = v0 + lr + 8 * (li & 1), vv = v0 + lr + 8 * (li >> 1);
                auto ka = [&](int kr, int dd) { return vk < P ? ring_addr(sK, kr, dd) : node_k + static_cast<uint32_t>(dd * 2); };
                auto vaa = [&](int kr, int dd) { return vv < P ? ring_addr(sV, kr, dd) : node_v + static_cast<uint32_t>(dd * 2); };
                decode_chunk(ka, vaa, v0, t4 == 0 ? lv : v0, v0, qf, scale, m0, m1, l0, l1, o, lane);
            }
            if (staged) {
                __syncwarp();
                if (lane == 0 && ib < b_hi) {
                    fence_proxy_async();  // this stage's ldmatrix reads before the TMA rewrite
                    issue(si);
                }
                __syncwarp();
                ++i;
                if (++si == kDNS) {
                    si = 0;
                    ph ^= 1;
                }
            }
        }
        // block partial of query column 0 (lanes t4 == 0 hold it)
        if (t4 == 0) {
            float* pb = part + static_cast<size_t>(b - b_lo) * (DH + 2);
#pragma unroll
            for (int mt = 0; mt < NK; ++mt) {
                pb[16 * mt + g8] = o[mt][0];
                pb[16 * mt + g8 + 8] = o[mt][2];
            }
            if (g8 == 0) {
                pb[DH] = m0;
                pb[DH + 1] = l0;
            }
        }
    }
    // ordered merge over all blocks of the row (attn_merge from the identity), CTA 0, warp 0
    cg::cluster_group cl = cg::this_cluster();
    if (S > 1) cl.sync();
    else __syncthreads();
    if (rank == 0 && warp == 0 && t4 == 0) {
        float M0 = -INFINITY, L0 = 0.f, A0[NK], A2[NK];
#pragma unroll
        for (int mt = 0; mt < NK; ++mt) A0[mt] = A2[mt] = 0.f;
        // (measured: gathering all partials into CTA 0 first costs occupancy and was slower)
        for (int r = 0; r < S; ++r) {
            const int r_lo = static_cast<int>(static_cast<long long>(r) * nb / S);
            const int r_hi = static_cast<int>(static_cast<long long>(r + 1) * nb / S);
            const float* pr = S > 1 ? cl.map_shared_rank(part, r) : part;
            for (int b = r_lo; b < r_hi; ++b) {
                const float* pb = pr + static_cast<size_t>(b - r_lo) * (DH + 2);
                const float m0 = pb[DH], l0 = pb[DH + 1];
                const float Mn = fmaxf(M0, m0);
                const float ca = M0 == -INFINITY ? 0.f : expf(__fsub_rn(M0, Mn));
                const float cb = expf(__fsub_rn(m0, Mn));
                L0 = fmaf(L0, ca, __fmul_rn(l0, cb));
#pragma unroll
                for (int mt = 0; mt < NK; ++mt) {
                    A0[mt] = fmaf(A0[mt], ca, __fmul_rn(pb[16 * mt + g8], cb));
                    A2[mt] = fmaf(A2[mt], ca, __fmul_rn(pb[16 * mt + g8 + 8], cb));
                }
                M0 = Mn;
            }
        }
        __nv_bfloat16* orow = out + static_cast<size_t>(gr.row0) * d + h * DH;
#pragma unroll
        for (int mt = 0; mt < NK; ++mt) {
            orow[16 * mt + g8] = __float2bfloat16(__fdiv_rn(A0[mt], L0));
            orow[16 * mt + g8 + 8] = __float2bfloat16(__fdiv_rn(A2[mt], L0));
        }
    }
    if (S > 1) cl.sync();  // peers keep their partials until CTA 0 has read them
}

template <int DH>
void launch_decode_impl(const float* q, const CUtensorMap& kmap, const CUtensorMap& vmap, long long layer_row0,
                        const __nv_bfloat16* K, const __nv_bfloat16* V, const TreeGroupDev* groups, int n_groups,
                        int max_ctx, int H, int d, __nv_bfloat16* out, cudaStream_t st) {
    const int nb = (max_ctx + 1 + kTBlock - 1) / kTBlock;
    // cluster size: fill ~2 CTAs per SM, at most 8 (portable), at most one per block
    int S = std::max(1, std::min(8, 296 / std::max(1, n_groups * H)));
    S = std::min(S, nb);
    const int max_blocks = (nb + S - 1) / S;
    const size_t smem = DecodeSmem<DH>::bytes(max_blocks);
    if (smem > static_cast<size_t>(kTSmem)) throw std::invalid_argument("decode attention: context too long");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(decode_attn_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmem);
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_groups * S, H);
    cfg.blockDim = dim3(32 * kDW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = S;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    SGB_CUDA(cudaLaunchKernelEx(&cfg, decode_attn_kernel<DH>, q, kmap, vmap, layer_row0, K, V, groups, S, max_blocks, d,
                                1.0f / sqrtf(static_cast<float>(DH)), out));
}

template <int DH>
void launch_tree_impl(const float* q, const CUtensorMap& kmap, const CUtensorMap& vmap, long long layer_row0,
                      const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, const TreeGroupDev* groups,
                      const TreeTileDev* tiles, int n_tiles, int W, int H, int d, int max_nodes, __nv_bfloat16* out,
                      cudaStream_t st) {
    constexpr size_t stageK = static_cast<size_t>(kTChunk) * DH * 2;
    const size_t tbl = static_cast<size_t>(max_nodes) * (DH * 2 + 16) * 2;
    const size_t fixed = tbl + 8 * 24 + 4 * 72 * 8 + 1024;  // barriers, chain tables, alignment slack
    // ring depth: 3 stages (measured, profiles/r02_tree_nst.jsonl): the per-chunk work of one
    // consumer warp is latency-bound, so CTAs per SM matter more than stages per CTA -- 6 -> 3
    // stages took the c5 verify shape (48 x 4 rows, ctx 2048, 32 heads) from 0.367 to 0.274 ms
    // per layer (the AR launch of the same contexts: 0.277) and 16 x 13 rows from 0.134 to 0.075
    static const int nst_env = [] {
        const char* v = getenv("SGB_TREE_NST");  // tuning experiments only
        return v ? std::max(2, std::min(8, atoi(v))) : 3;
    }();
    int nst = nst_env;
    while (nst > 2 && 2 * stageK * nst + fixed > static_cast<size_t>(kTSmem)) --nst;
    const size_t smem = 2 * stageK * nst + fixed;
    if (smem > static_cast<size_t>(kTSmem)) throw std::invalid_argument("tree attention: tree too large for shared memory");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tree_attn_kernel<DH, kTMaxWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmem);
        cudaFuncSetAttribute(tree_attn_kernel<DH, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTSmem);
        attr = true;
    }
    static const int one_warp = [] {
        const char* v = getenv("SGB_TREE_ONE_WARP");  // A/B: 0 = never, 1 = always (W == 1), -1 = by waves
        return v ? atoi(v) : -1;
    }();
    // the register-capped one-warp variant fits more CTAs per SM but runs each CTA ~1.25-1.5x
    // slower (spills, shared bandwidth): measured (profiles/r02_tree_onewarp_ab.txt) it pays only
    // when it saves a whole wave (c5 verify at B = 32: 1,024 CTAs, 2 waves -> 1: 0.254 -> 0.191 ms
    // per layer; at B = 48, 2 waves either way: 0.275 -> 0.344), so it is taken when it does
    bool use_one = false;
    if (W == 1 && one_warp != 0) {
        use_one = one_warp > 0;
        if (one_warp < 0) {
            static std::mutex mu;
            static std::vector<std::array<int, 3>> occ_cache;  // (smem, CTAs/SM 8-warp, CTAs/SM one-warp)
            std::array<int, 3> occ{0, 0, 0};
            {
                std::lock_guard<std::mutex> lock(mu);
                for (const auto& c : occ_cache)
                    if (c[0] == static_cast<int>(smem)) occ = c;
                if (occ[1] == 0) {
                    int a = 0, b = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, tree_attn_kernel<DH, kTMaxWarps>, 64, smem);
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tree_attn_kernel<DH, 1>, 64, smem);
                    occ = {static_cast<int>(smem), std::max(1, a), std::max(1, b)};
                    occ_cache.push_back(occ);
                }
            }
            const long long ctas = static_cast<long long>(n_tiles) * H;
            const long long wa = (ctas + 148LL * occ[1] - 1) / (148LL * occ[1]);
            const long long wb = (ctas + 148LL * occ[2] - 1) / (148LL * occ[2]);
            use_one = wb < wa;
        }
    }
    auto kern = use_one ? tree_attn_kernel<DH, 1> : tree_attn_kernel<DH, kTMaxWarps>;
    launch_pdl(kern, dim3(n_tiles, H), dim3(32 * (W + 1)), smem, st, q, kmap, vmap, layer_row0, K, V, rows, groups,
               tiles, d, nst, max_nodes, 1.0f / sqrtf(static_cast<float>(DH)), out);
}

}  // namespace

int tree_attn_warps(int max_rows_per_group, int n_groups, int H, int dh, int max_nodes) {
    static const int w_env = [] {
        const char* v = getenv("SGB_TREE_W");  // A/B: consumer warps (8-row groups) per tile
        return v ? atoi(v) : 0;
    }();
    if (w_env > 0) return std::min(kTMaxWarps, std::max(1, std::min(w_env, (max_rows_per_group + 7) / 8)));
    // widest tiles (the prefix streams once per tile) unless narrower ones finish in fewer waves
    // (CTAs resident per SM are bounded by the node table + ring in shared memory)
    const size_t tbl = static_cast<size_t>(max_nodes) * (dh * 2 + 16) * 2;
    const size_t per_cta = tbl + 4 * static_cast<size_t>(kTChunk) * dh * 2 * 2 + 4096;
    const int occ_smem = std::max<int>(1, static_cast<int>(kTSmem / per_cta));
    int best_w = 1;
    long long best_waves = -1;
    for (int w = std::max(1, std::min(kTMaxWarps, (max_rows_per_group + 7) / 8)); w >= 1; w = (w + 1) / 2 - (w == 1)) {
        const int rows_per_tile = 8 * w;
        const long long ctas =
            static_cast<long long>(n_groups) * ((max_rows_per_group + rows_per_tile - 1) / rows_per_tile) * H;
        const int occ = std::max(1, std::min(occ_smem, 2048 / (32 * (w + 1))));
        const long long waves = (ctas + 148LL * occ - 1) / (148LL * occ);
        if (best_waves < 0 || waves < best_waves) {
            best_waves = waves;
            best_w = w;
        }
        if (w == 1) break;
    }
    return best_w;
}

void build_tree_tiles(const std::vector<TreeGroupDev>& groups, int W, std::vector<TreeTileDev>& out) {
    out.clear();
    const int rt = 8 * W;
    for (size_t g = 0; g < groups.size(); ++g)
        for (int r = 0; r < groups[g].nrows; r += rt)
            out.push_back(TreeTileDev{static_cast<int>(g), r, std::min(rt, groups[g].nrows - r)});
}

void launch_attention_tree(const float* q, const CUtensorMap& kmap, const CUtensorMap& vmap, long long layer_row0,
                           const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows,
                           const TreeGroupDev* groups, const TreeTileDev* tiles, int n_tiles, int W, int H, int d,
                           int max_nodes, __nv_bfloat16* out, cudaStream_t st) {
    if (n_tiles <= 0) return;
    if (W < 1 || W > kTMaxWarps) throw std::invalid_argument("tree attention: warps per tile in [1, 8]");
    const int dh = d / H;
    if (dh == 128)
        launch_tree_impl<128>(q, kmap, vmap, layer_row0, K, V, rows, groups, tiles, n_tiles, W, H, d, max_nodes, out, st);
    else if (dh == 64)
        launch_tree_impl<64>(q, kmap, vmap, layer_row0, K, V, rows, groups, tiles, n_tiles, W, H, d, max_nodes, out, st);
    else
        throw std::invalid_argument("tree attention: head dim must be 64 or 128");
    SGB_KCHECK();
}

void launch_attention_decode(const float* q, const CUtensorMap& kmap, const CUtensorMap& vmap, long long layer_row0,
                             const __nv_bfloat16* K, const __nv_bfloat16* V, const TreeGroupDev* groups, int n_groups,
                             int max_ctx, int H, int d, __nv_bfloat16* out, cudaStream_t st) {
    if (n_groups <= 0) return;
    const int dh = d / H;
    if (dh == 128)
        launch_decode_impl<128>(q, kmap, vmap, layer_row0, K, V, groups, n_groups, max_ctx, H, d, out, st);
    else if (dh == 64)
        launch_decode_impl<64>(q, kmap, vmap, layer_row0, K, V, groups, n_groups, max_ctx, H, d, out, st);
    else
        throw std::invalid_argument("decode attention: head dim must be 64 or 128");
    SGB_KCHECK();
}

}  // namespace sgb
