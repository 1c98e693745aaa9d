// Tree-masked paged-KV attention on tensor cores (decode / tree verify / draft expansion /
// prefill), one kernel for every attention row of the engine.
//
// Replaces the per-row, per-head scalar loop of the reference decode block
// (include/sgrpo/tinylm.hpp:335-395): scores over [cache | ancestor pool | masked new
// rows], softmax (nn.hpp:157-169), then P.V.
//
// Rows. Every query row carries a *virtual key sequence*: virtual index v < ctx_len maps to
// the contiguous cache slots ctx_base+v (the committed prefix; v < pre_len reads the group
// leader's shared prompt copy), and ctx_len <= v < ctx_len+chain_len maps to
// chain_slots[v-ctx_len] (the row's own tree path: ancestors root-first, then itself). The
// virtual index equals the absolute position (target) or position-1 (draft cache), so a
// tree row and the AR row of the same token see the same keys in the same order -- the tree
// mask of build_tree_mask (drafttree.cpp:145-168) is exactly "keys = ancestors-or-self".
//
// Tiles. A tile is up to 8 query rows and a range of 64-key blocks. Rows of one tile share
// every key of those blocks: either one row (the AR / prefill / boundary case) or up to 8
// verify rows of one sequence over the blocks that lie entirely inside its committed prefix
// (build_attn_tiles). So the tree rows of a sequence stream its prefix once per 8 rows
// instead of once per row, and the blocks that reach into the tree path run per row.
//
// Kernel (B200): persistent and flat. The work of a launch is the list of items
// (tile, head group, 64-key block), tiles in order; CTA c takes the contiguous slice
// [c*T/G, (c+1)*T/G), so every CTA streams the same number of blocks whatever the context
// mix, and its shared-memory ring never drains between tiles. A producer warp stages each
// 16-key chunk (K and V rows of the head group, one cp.async.bulk per key row into padded
// rows: conflict-free ldmatrix). One consumer warp per head runs the chunk on the tensor
// cores with mma.sync.m16n8k16 (bf16 in, fp32 accumulate):
//   S^T[16 keys][8 queries] = K[16][dh] . Q^T[dh][8]          (dh/16 mma, keys in M)
//   online softmax per query column (running max / sum over the chunk, quad shuffles)
//   P^T -> bf16, transposed in registers with movmatrix into the B fragment
//   O^T[dh][8] += V^T[dh][16] . P^T[16][8]                      (dh/16 mma, ldmatrix.trans)
// Each 64-key block yields its own partial (m, l, O) from a fresh state; the warp that
// completes a (row, head group) -- an atomic ticket per row -- merges the row's block
// partials in block order and writes the bf16 output (no combine launch).
//
// Determinism / batch invariance (SURVEY.md §7 hard part 1). Key slot j of a chunk is
// virtual index 16c+j in every tile; an mma output element depends only on its own row of
// A and column of B (scripts/probes/probe_mma.cu: bit-identical under any permutation of
// the other rows / columns), so a query's scores, probabilities and P.V sums are the same
// bits whichever tile column it occupies and whatever the other queries are. Block
// partials merge strictly in block order. Hence a tree row, the AR row of the same token,
// and a row run alone or in any batch produce identical outputs (spec == AR rollouts).
//
// Roofline: HBM-bound on K/V reads, 4*d bytes per key per layer per tile.
#include <algorithm>
#include <cstdlib>
#include <cfloat>

#include "attn_numerics.cuh"
#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kBlock = kAttnBlock;  // 64 keys per softmax partial
constexpr int kChunk = 16;          // keys per stage = one mma k-step of P.V
constexpr int kQT = kAttnTileRows;  // 8 queries per tile = mma N
constexpr int kSmemBudget = 227 * 1024;
constexpr int kMaxScanTiles = 1 << 20;
constexpr int kMaxCons = 16;                // consumer warps per CTA
constexpr int kMaxTileRows = kQT * kMaxCons;  // rows of one shared tile

SGB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
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

// one tile of the launch: explicit (host-built) or implicit (tile i = row i, all its blocks)
struct TileView {
    const AttnTileDev* tiles;
    const int* ctx_len;
    const int* chain_len;
    __device__ int row_blocks(int r) const { return (ctx_len[r] + chain_len[r] + kBlock - 1) / kBlock; }
    __device__ AttnTileDev get(int t) const {
        if (tiles) return tiles[t];
        return AttnTileDev{t, 1, 0, row_blocks(t), -1};
    }
};

struct ItemIt {
    int t, g, b;
    AttnTileDev tl;
    int lv;  // the longest virtual length among the tile's rows (1-row tiles: the row's key count)
};

// MERGE: a CTA's run of a tile's blocks that starts at block 0 merges its block partials in
// registers (attn_merge in block order, the same arithmetic the finisher would run) instead of
// publishing each of them: a row whose blocks the run covers completely is written straight out
// (no partials, no ticket); otherwise the merged prefix goes into block slot 0 and slots
// 1..k-1 get an m = -inf marker (an exact no-op in the finisher's merge). Used for the shared
// tree-verify / draft-level tiles (many blocks per tile); the per-row decode path keeps the
// 96-register variant.
constexpr int kMaxConsMerge = 8;  // consumer warps of the MERGE variant (its running state needs registers)
template <int DH, bool MERGE>
__global__ void __launch_bounds__(32 * ((MERGE ? kMaxConsMerge : kMaxCons) + 1), 1)
    attn_kernel(const float* __restrict__ q, const __nv_bfloat16* __restrict__ K, const __nv_bfloat16* __restrict__ V,
                AttnRowsDev rows, const AttnTileDev* __restrict__ tiles, int n_tiles, int H, int d, int G, int QW,
                int nst, int nb_max, int balance, float scale, float* __restrict__ part_acc, float* __restrict__ part_ml,
                int* __restrict__ row_ctr, __nv_bfloat16* __restrict__ out) {
    constexpr int NK = DH / 16;   // mma k-steps of S (dims) = m-tiles of O (dims)
    constexpr int DPL = DH / 32;  // merge: dims per lane
    extern __shared__ __align__(128) uint8_t smem[];
    const int HG = H / G;                                            // heads per item
    // consumer warp w: head w % HG, query tile w / HG (8 queries each, QW per item)
    const int rowb = HG * DH * 2 + 16;                               // padded staged key row (bytes)
    const size_t stage_bytes = static_cast<size_t>(kChunk) * rowb;  // one of K or V per stage
    uint8_t* Ks = smem;
    uint8_t* Vs = smem + nst * stage_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * nst * stage_bytes);
    uint64_t* empty = full + nst;
    int* flag = reinterpret_cast<int*>(empty + nst);  // [kMaxTileRows]
    int* tsum = flag + kMaxTileRows;                   // [blockDim.x + 1] item-count scan
    int* loc = tsum + blockDim.x + 1;                  // [4] start tile, head group, block
    long long* wsum = reinterpret_cast<long long*>(  // [blockDim.x + 1] weight scan
        (reinterpret_cast<uintptr_t>(loc + 4) + 7) & ~uintptr_t(7));
    long long* locl = wsum + blockDim.x + 1;          // [2] first item, end item

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_cons = HG * QW;
    const int nthr = blockDim.x;

    // stale smem may hold any bit pattern; key rows past a chunk's end meet p = 0 in the
    // P.V mma, so they must be finite: zero the ring once (later chunks leave real K/V)
    for (size_t o = threadIdx.x * 16; o < 2 * nst * stage_bytes; o += nthr * 16)
        *reinterpret_cast<uint4*>(smem + o) = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], n_cons);
        }
        fence_barrier_init();
    }
    fence_proxy_async();
    // PDL: setup overlapped the previous kernel; row metadata and q are produced by it
    pdl_wait();
    pdl_trigger();
    const TileView tv{tiles, rows.ctx_len, rows.chain_len};
    // ---- work split. Items are (tile, head group, block), tiles in order; an item weighs its
    // 16-key chunks + 1 (shared tiles 5, a tree row's boundary block as few as 2) -- or 1 each
    // (balance == 0) -- and CTA c takes the items whose starting weight lies in
    // [c*W/grid, (c+1)*W/grid).
    const int per = (n_tiles + nthr - 1) / nthr;
    const int t0 = min(n_tiles, static_cast<int>(threadIdx.x) * per), t1 = min(n_tiles, t0 + per);
    auto lv_of = [&](const AttnTileDev& tl) {
        int lv = rows.ctx_len[tl.row0] + rows.chain_len[tl.row0];
        if (tl.bsh >= 0)
            for (int j = 1; j < tl.nrows; ++j) lv = max(lv, rows.ctx_len[tl.row0 + j] + rows.chain_len[tl.row0 + j]);
        return lv;
    };
    auto item_w = [&](const AttnTileDev& tl, int lv, int b) -> int {
        if (!balance) return 1;  // count-based split
        if (tl.nrows > 1 && tl.bsh >= 0 && b == tl.bhi - 1) {
            // boundary block: chunks inside the common prefix once, the rest once per row
            const int kb = b * kBlock, ve = min(kb + kBlock, lv);
            const int nsh = min(max(0, (tl.bsh - kb) / kChunk), (ve - kb + kChunk - 1) / kChunk);
            const int ncp = (ve - kb + kChunk - 1) / kChunk;
            return nsh + (ncp - nsh) * tl.nrows + 1;
        }
        if (tl.nrows > 1) return kBlock / kChunk + 1;
        const int keys = min(kBlock, max(0, lv - b * kBlock));
        return (keys + kChunk - 1) / kChunk + 1;
    };
    auto tile_w = [&](const AttnTileDev& tl, int lv) -> long long {
        long long w = 0;
        for (int b = tl.blo; b < tl.bhi; ++b) w += item_w(tl, lv, b);
        return w;
    };
    int own = 0;
    long long ownw = 0;
    for (int t = t0; t < t1; ++t) {
        const AttnTileDev tl = tv.get(t);
        own += tl.bhi - tl.blo;
        ownw += tile_w(tl, lv_of(tl));
    }
    tsum[threadIdx.x] = own;
    wsum[threadIdx.x] = ownw;
    __syncthreads();
    if (warp == 0) {
        const int run = (nthr + 31) / 32;
        long long lsum = 0, lw = 0;
        for (int t = lane * run; t < min(nthr, (lane + 1) * run); ++t) {
            lsum += tsum[t];
            lw += wsum[t];
        }
        long long inc = lsum, incw = lw;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, inc, o);
            const long long yw = __shfl_up_sync(0xffffffffu, incw, o);
            if (lane >= o) {
                inc += y;
                incw += yw;
            }
        }
        long long off = inc - lsum, offw = incw - lw;
        for (int t = lane * run; t < min(nthr, (lane + 1) * run); ++t) {
            const int v = tsum[t];
            const long long vw = wsum[t];
            tsum[t] = static_cast<int>(off);
            wsum[t] = offw;
            off += v;
            offw += vw;
        }
        if (lane == 31) {
            tsum[nthr] = static_cast<int>(inc);
            wsum[nthr] = incw;
        }
    }
    __syncthreads();
    const long long T = static_cast<long long>(G) * tsum[nthr];
    const long long WT = static_cast<long long>(G) * wsum[nthr];
    const long long w_lo = WT * blockIdx.x / gridDim.x, w_hi = WT * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) locl[1] = T;  // w_hi == WT: the end of the list
    // the item holding weight position w (found by the thread whose tile slice holds it)
    auto find = [&](long long w, bool lo) {
        const long long c0 = static_cast<long long>(G) * wsum[threadIdx.x];
        if (ownw == 0 || w < c0 || w >= c0 + static_cast<long long>(G) * ownw) return;
        long long c = c0, base = static_cast<long long>(G) * tsum[threadIdx.x];
        for (int t = t0; t < t1; ++t) {
            const AttnTileDev tl = tv.get(t);
            const int lv = lv_of(tl);
            const long long wt = tile_w(tl, lv);
            const int nb = tl.bhi - tl.blo;
            if (w < c + static_cast<long long>(G) * wt) {
                const int g = static_cast<int>((w - c) / wt);
                long long rem = (w - c) - g * wt;
                int b = tl.blo;
                while (rem >= item_w(tl, lv, b)) rem -= item_w(tl, lv, b++);
                const long long idx = base + static_cast<long long>(g) * nb + (b - tl.blo);
                if (lo) {
                    loc[0] = t;
                    loc[1] = g;
                    loc[2] = b;
                    locl[0] = idx;
                } else {
                    locl[1] = idx;
                }
                return;
            }
            c += static_cast<long long>(G) * wt;
            base += static_cast<long long>(G) * nb;
        }
    };
    __syncthreads();
    if (w_lo < WT) find(w_lo, true);
    if (w_hi < WT) find(w_hi, false);
    __syncthreads();
    if (w_lo >= WT || locl[1] <= locl[0]) return;
    ItemIt it0;
    it0.t = loc[0];
    it0.tl = tv.get(it0.t);
    it0.lv = lv_of(it0.tl);
    it0.g = loc[1];
    it0.b = loc[2];
    const int n_items = static_cast<int>(locl[1] - locl[0]);
    auto advance = [&](ItemIt& x) {
        if (++x.b == x.tl.bhi) {
            if (++x.g == G) {
                x.g = 0;
                ++x.t;
                if (x.t < n_tiles) {
                    x.tl = tv.get(x.t);
                    x.lv = lv_of(x.tl);
                }
            }
            x.b = x.tl.blo;
        }
    };
    // the keys of item x: virtual [64b, v_end); v_end <= 64b when the row has no such block
    auto item_end = [&](const ItemIt& x) -> int {
        const int kb = x.b * kBlock;
        if (x.tl.nrows > 1 && !(x.tl.bsh >= 0 && x.b == x.tl.bhi - 1))
            return kb + kBlock;  // shared blocks lie inside the committed prefix
        return min(kb + kBlock, x.lv);
    };
    auto nrows_of = [&](const ItemIt& y, int qtile) { return max(0, min(kQT, y.tl.nrows - kQT * qtile)); };
    // a chunk of a boundary block past the common prefix: staged once per tile row
    auto per_row_chunk = [&](const ItemIt& x, int v0) {
        return x.tl.nrows > 1 && x.tl.bsh >= 0 && x.b == x.tl.bhi - 1 && v0 + kChunk > x.tl.bsh;
    };

    if (warp == n_cons) {
        // ---------------- producer warp: one bulk DMA per staged K / V key row
        ItemIt x = it0;
        int i = 0, si = 0, ph = 0;  // staged chunk counter, ring stage, phase
        const uint32_t row_bytes = static_cast<uint32_t>(HG) * DH * 2;
        int cur_r = -1, ctx_len = 0, pre_len = 0;
        long long ctx_base = 0, pre_base = 0;
        const long long* chain = nullptr;
        for (int n = 0; n < n_items; ++n, advance(x)) {
            const int r = x.tl.row0;
            const int ve = item_end(x);
            if (r != cur_r) {
                cur_r = r;
                ctx_len = rows.ctx_len[r];
                ctx_base = rows.ctx_base[r];
                chain = rows.chain_slots + static_cast<size_t>(r) * kMaxChain;
                pre_len = rows.pre_len ? rows.pre_len[r] : 0;
                pre_base = rows.pre_len ? rows.pre_base[r] : 0;
            }
            const size_t col = static_cast<size_t>(x.g) * HG * DH;
            // one stage: keys [v0, v0 + nk) of a row with the given key map
            auto stage = [&](int v0, int nk, int c_len, long long c_base, int p_len, long long p_base,
                             const long long* ch) {
                const int s = si;
                if (i >= nst) mbar_wait(&empty[s], ph ^ 1);
                if (lane == 0) mbar_arrive_expect_tx(&full[s], 2u * row_bytes * nk);
                __syncwarp();
                if (lane < nk) {
                    const int v = v0 + lane;
                    const long long slot = v < c_len ? (v < p_len ? p_base : c_base) + v : ch[v - c_len];
                    const size_t src = static_cast<size_t>(slot) * d + col;
                    bulk_g2s(Ks + static_cast<size_t>(s) * stage_bytes + static_cast<size_t>(lane) * rowb, K + src,
                             row_bytes, &full[s]);
                    bulk_g2s(Vs + static_cast<size_t>(s) * stage_bytes + static_cast<size_t>(lane) * rowb, V + src,
                             row_bytes, &full[s]);
                }
                ++i;
                if (++si == nst) {
                    si = 0;
                    ph ^= 1;
                }
            };
            for (int v0 = x.b * kBlock; v0 < ve; v0 += kChunk) {
                if (!per_row_chunk(x, v0)) {
                    stage(v0, min(kChunk, ve - v0), ctx_len, ctx_base, pre_len, pre_base, chain);
                    continue;
                }
                for (int j = 0; j < x.tl.nrows; ++j) {
                    const int rj = r + j;
                    const int cl = rows.ctx_len[rj];
                    const int nk = max(0, min(kChunk, cl + rows.chain_len[rj] - v0));
                    stage(v0, nk, cl, rows.ctx_base[rj], rows.pre_len ? rows.pre_len[rj] : 0,
                          rows.pre_len ? rows.pre_base[rj] : 0, rows.chain_slots + static_cast<size_t>(rj) * kMaxChain);
                }
            }
        }
        return;
    }
    if (warp > n_cons) return;

    // ---------------- consumer warps: head hl, query tile qt (rows 8qt .. 8qt+7 of the tile)
    const int hl = warp % HG, qt = warp / HG;
    const int g8 = lane >> 2, t4 = lane & 3;
    // ldmatrix lane addresses (bytes within a stage): K as A of S^T (key = lane%8 + 8*(i&1),
    // dim 8*(i>>1)), V as A of O^T via .trans (key = lane%8 + 8*(i>>1), dim 8*(i&1))
    const int li = lane >> 3, lr = lane & 7;
    const uint32_t k_lane = static_cast<uint32_t>((lr + 8 * (li & 1)) * rowb + (hl * DH + 8 * (li >> 1)) * 2);
    const uint32_t v_lane = static_cast<uint32_t>((lr + 8 * (li >> 1)) * rowb + (hl * DH + 8 * (li & 1)) * 2);
    const uint32_t ks_base = smem_u32(Ks), vs_base = smem_u32(Vs);
    uint32_t qf[NK][2];
    ItemIt x = it0;
    int i = 0, si = 0, ph = 0;  // staged chunk counter, ring stage, phase
    int cur_t = -1, cur_g = -1, seg = 0;
    // MERGE: running merged state of this warp's two columns over the current run
    bool run0 = false;
    float RM0 = -INFINITY, RM1 = -INFINITY, RL0 = 0.f, RL1 = 0.f;
    float RA[MERGE ? NK : 1][4];
    for (int n = 0; n < n_items; ++n) {
        const int ve = item_end(x);
        const int kb = x.b * kBlock;
        const int h = x.g * HG + hl;
        const int qrow0 = x.tl.row0 + kQT * qt;                      // this warp's first query row
        const int nrows = max(0, min(kQT, x.tl.nrows - kQT * qt));  // its real query columns
        if (x.t != cur_t || x.g != cur_g) {
            cur_t = x.t;
            cur_g = x.g;
            if constexpr (MERGE) {
                run0 = x.b == 0;
                RM0 = RM1 = -INFINITY;
                RL0 = RL1 = 0.f;
#pragma unroll
                for (int mt = 0; mt < NK; ++mt) RA[mt][0] = RA[mt][1] = RA[mt][2] = RA[mt][3] = 0.f;
            }
            // Q^T as the B operand: query column g8 (tile row, clamped), dims 16ks + {2t, 2t+1, 2t+8, 2t+9}
            const int qrow = nrows > 0 ? qrow0 + min(g8, nrows - 1) : x.tl.row0;
            const float* qr = q + static_cast<size_t>(qrow) * d + h * DH + 2 * t4;
#pragma unroll
            for (int ks = 0; ks < NK; ++ks) {
                const float2 a = __ldg(reinterpret_cast<const float2*>(qr + 16 * ks));
                const float2 b = __ldg(reinterpret_cast<const float2*>(qr + 16 * ks + 8));
                qf[ks][0] = pack_bf16(a.x, a.y);
                qf[ks][1] = pack_bf16(b.x, b.y);
            }
        }
        if (ve > kb) {
            float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // query columns 2t4, 2t4+1
            float o[NK][4];
#pragma unroll
            for (int mt = 0; mt < NK; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.f;
            // one staged chunk; e0 / e1 = key end of this lane's query columns 2t4 / 2t4+1
            auto chunk = [&](int v0, int e0, int e1) {
                const int s = si;
                mbar_wait(&full[s], ph);
                const uint32_t kst = ks_base + static_cast<uint32_t>(s * stage_bytes);
                const uint32_t vst = vs_base + static_cast<uint32_t>(s * stage_bytes);
                // S^T = K . Q^T
                float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int ks = 0; ks < NK; ++ks) {
                    uint32_t a[4];
                    ldsm_x4(kst + k_lane + ks * 32, a);
                    mma16816(sc, a, qf[ks][0], qf[ks][1]);
                }
                const bool va0 = v0 + g8 < e0, va1 = v0 + g8 < e1, vb0 = v0 + g8 + 8 < e0, vb1 = v0 + g8 + 8 < e1;
                const float s0 = va0 ? attn_scale(sc[0], scale) : -INFINITY;  // key g8,   query 2t
                const float s1 = va1 ? attn_scale(sc[1], scale) : -INFINITY;  // key g8,   query 2t+1
                const float s2 = vb0 ? attn_scale(sc[2], scale) : -INFINITY;  // key g8+8, query 2t
                const float s3 = vb1 ? attn_scale(sc[3], scale) : -INFINITY;  // key g8+8, query 2t+1
                float c0 = fmaxf(s0, s2), c1 = fmaxf(s1, s3);
#pragma unroll
                for (int o2 = 4; o2 < 32; o2 <<= 1) {
                    c0 = fmaxf(c0, __shfl_xor_sync(0xffffffffu, c0, o2));
                    c1 = fmaxf(c1, __shfl_xor_sync(0xffffffffu, c1, o2));
                }
                const float n0 = fmaxf(m0, c0), n1 = fmaxf(m1, c1);
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
                // V fragments first: the stage is released before the P.V math
                uint32_t va4[NK][4];
#pragma unroll
                for (int mt = 0; mt < NK; ++mt) ldsm_x4_t(vst + v_lane + mt * 32, va4[mt]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                // P^T as the B operand: [key][query] fragments transposed to [query][key]
                const uint32_t b0 = movm_t(pack_bf16(p0, p1)), b1 = movm_t(pack_bf16(p2, p3));
#pragma unroll
                for (int mt = 0; mt < NK; ++mt) {
                    o[mt][0] = __fmul_rn(o[mt][0], a0);
                    o[mt][1] = __fmul_rn(o[mt][1], a1);
                    o[mt][2] = __fmul_rn(o[mt][2], a0);
                    o[mt][3] = __fmul_rn(o[mt][3], a1);
                    mma16816(o[mt], va4[mt], b0, b1);
                }
                ++i;
                if (++si == nst) {
                    si = 0;
                    ph ^= 1;
                }
            };
            for (int v0 = kb; v0 < ve; v0 += kChunk) {
                if (!per_row_chunk(x, v0)) {
                    chunk(v0, ve, ve);
                    continue;
                }
                // boundary chunk past the common prefix: one stage per tile row, row j's keys.
                // Only row j's query column is live (the others see -inf scores: alpha = 1,
                // p = 0, an exact no-op on their state), so every column runs exactly the
                // chunks its own 1-row item would, in the same order (identical bits).
                for (int j = 0; j < x.tl.nrows; ++j) {
                    const int cj = j - kQT * qt;
                    if (cj < 0 || cj >= kQT) {
                        const int s = si;
                        mbar_wait(&full[s], ph);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty[s]);
                        ++i;
                        if (++si == nst) {
                            si = 0;
                            ph ^= 1;
                        }
                        continue;
                    }
                    const int rj = x.tl.row0 + j;
                    const int lvj = rows.ctx_len[rj] + rows.chain_len[rj];
                    chunk(v0, 2 * t4 == cj ? lvj : v0, 2 * t4 + 1 == cj ? lvj : v0);
                }
            }
            if (MERGE && run0) {
                // ordered in-register merge of this block partial (attn_merge, per column)
                if (x.b == 0) {  // from the identity: reproduces the partial exactly
                    RM0 = m0;
                    RM1 = m1;
                    RL0 = l0;
                    RL1 = l1;
#pragma unroll
                    for (int mt = 0; mt < NK; ++mt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) RA[mt][e] = o[mt][e];
                } else {
                    const float Mn0 = fmaxf(RM0, m0), Mn1 = fmaxf(RM1, m1);
                    const float ca0 = RM0 == -INFINITY ? 0.f : expf(__fsub_rn(RM0, Mn0));
                    const float cb0 = expf(__fsub_rn(m0, Mn0));
                    const float ca1 = RM1 == -INFINITY ? 0.f : expf(__fsub_rn(RM1, Mn1));
                    const float cb1 = expf(__fsub_rn(m1, Mn1));
                    if (m0 != -INFINITY) {  // a column without keys in this block: exact no-op
                        RL0 = fmaf(RL0, ca0, __fmul_rn(l0, cb0));
#pragma unroll
                        for (int mt = 0; mt < NK; ++mt) {
                            RA[mt][0] = fmaf(RA[mt][0], ca0, __fmul_rn(o[mt][0], cb0));
                            RA[mt][2] = fmaf(RA[mt][2], ca0, __fmul_rn(o[mt][2], cb0));
                        }
                        RM0 = Mn0;
                    }
                    if (m1 != -INFINITY) {
                        RL1 = fmaf(RL1, ca1, __fmul_rn(l1, cb1));
#pragma unroll
                        for (int mt = 0; mt < NK; ++mt) {
                            RA[mt][1] = fmaf(RA[mt][1], ca1, __fmul_rn(o[mt][1], cb1));
                            RA[mt][3] = fmaf(RA[mt][3], ca1, __fmul_rn(o[mt][3], cb1));
                        }
                        RM1 = Mn1;
                    }
                }
            } else {
                // publish the block partial of every real query column
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int qc = 2 * t4 + c;
                    if (qc < nrows) {
                        const int r = qrow0 + qc;
                        const size_t pidx = (static_cast<size_t>(r) * nb_max + x.b) * H + h;
                        float* pa = part_acc + pidx * DH;
#pragma unroll
                        for (int mt = 0; mt < NK; ++mt) {
                            pa[16 * mt + g8] = o[mt][c];
                            pa[16 * mt + g8 + 8] = o[mt][2 + c];
                        }
                        if (g8 == 0) {
                            part_ml[2 * pidx] = c ? m1 : m0;
                            part_ml[2 * pidx + 1] = c ? l1 : l0;
                        }
                    }
                }
            }
        }
        if (ve > kb) ++seg;
        const ItemIt done = x;
        advance(x);
        // ---- ticket per (row, head group) at the end of this CTA's run of the tile's blocks
        // (counts every block published in the run); the CTA that completes a row merges it.
        // The ticket thread's gpu-scope fence after the CTA barrier orders every warp's
        // partial stores before its ticket (cumulative release, as in a grid barrier).
        const bool seg_end = (n + 1 == n_items) || x.t != done.t || x.g != done.g;
        if (!seg_end || seg == 0) continue;
        if (MERGE && run0) {
            // the run covered blocks [0, done.b]: rows it completes are written now; the others
            // get the merged prefix in slot 0 and m = -inf markers in slots 1..done.b
            const int h = done.g * HG + hl;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int qc = 2 * t4 + c;
                if (qc >= nrows_of(done, qt)) continue;
                const int r = done.tl.row0 + kQT * qt + qc;
                const float Mx = c ? RM1 : RM0, Lx = c ? RL1 : RL0;
                if (done.b + 1 >= tv.row_blocks(r)) {
                    __nv_bfloat16* orow = out + static_cast<size_t>(r) * d + h * DH;
#pragma unroll
                    for (int mt = 0; mt < NK; ++mt) {
                        orow[16 * mt + g8] = __float2bfloat16(__fdiv_rn(RA[mt][c], Lx));
                        orow[16 * mt + g8 + 8] = __float2bfloat16(__fdiv_rn(RA[mt][2 + c], Lx));
                    }
                } else {
                    const size_t p0 = (static_cast<size_t>(r) * nb_max + 0) * H + h;
                    float* pa = part_acc + p0 * DH;
#pragma unroll
                    for (int mt = 0; mt < NK; ++mt) {
                        pa[16 * mt + g8] = RA[mt][c];
                        pa[16 * mt + g8 + 8] = RA[mt][2 + c];
                    }
                    if (g8 == 0) {
                        part_ml[2 * p0] = Mx;
                        part_ml[2 * p0 + 1] = Lx;
                        for (int b = 1; b <= done.b; ++b)
                            part_ml[2 * ((static_cast<size_t>(r) * nb_max + b) * H + h)] = -INFINITY;
                    }
                }
            }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(n_cons * 32) : "memory");
        if (threadIdx.x < done.tl.nrows) {
            const int r = done.tl.row0 + threadIdx.x;
            int last = 0;
            if (!(MERGE && run0 && done.b + 1 >= tv.row_blocks(r))) {  // not completed in registers
                __threadfence();
                int* c = row_ctr + static_cast<size_t>(r) * G + done.g;
                const int old = atomicAdd(c, seg);
                last = (old + seg == tv.row_blocks(r));
                if (last) {
                    *c = 0;  // re-armed for the next launch
                    __threadfence();  // acquire side: the other CTAs' partials are read after the barrier
                }
            }
            flag[threadIdx.x] = last;
        }
        seg = 0;
        asm volatile("bar.sync 1, %0;" ::"r"(n_cons * 32) : "memory");
        int any = 0;
        for (int j = 0; j < done.tl.nrows; ++j) any |= flag[j];
        if (any) {
            const int h = done.g * HG + hl;
            for (int j = qt; j < done.tl.nrows; j += QW) {
                if (!flag[j]) continue;
                const int r = done.tl.row0 + j;
                const int nbr = tv.row_blocks(r);
                // merge from the identity (-inf, 0, 0): the first merge reproduces partial 0
                float Mx = -INFINITY, Lx = 0.f, A[DPL];
#pragma unroll
                for (int e = 0; e < DPL; ++e) A[e] = 0.f;
                constexpr int kMB = 4;
                for (int b0 = 0; b0 < nbr; b0 += kMB) {
                    float mb[kMB], lb[kMB], ab[kMB][DPL];
#pragma unroll
                    for (int u = 0; u < kMB; ++u) {
                        const int b = min(b0 + u, nbr - 1);
                        const size_t pidx = (static_cast<size_t>(r) * nb_max + b) * H + h;
                        mb[u] = __ldcg(part_ml + 2 * pidx);
                        lb[u] = __ldcg(part_ml + 2 * pidx + 1);
#pragma unroll
                        for (int e = 0; e < DPL; ++e) ab[u][e] = __ldcg(part_acc + pidx * DH + lane * DPL + e);
                    }
#pragma unroll
                    for (int u = 0; u < kMB; ++u)
                        // mb = -inf: a marker inside a merged run (skipped: an exact no-op there)
                        if (b0 + u < nbr && mb[u] != -INFINITY) attn_merge<DPL>(Mx, Lx, A, mb[u], lb[u], ab[u]);
                }
#pragma unroll
                for (int e = 0; e < DPL; ++e)
                    out[static_cast<size_t>(r) * d + h * DH + lane * DPL + e] = __float2bfloat16(__fdiv_rn(A[e], Lx));
            }
        }
        // flags are rewritten by the next item's ticket
        asm volatile("bar.sync 1, %0;" ::"r"(n_cons * 32) : "memory");
    }
}

template <int DH, bool MERGE>
void launch_impl(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, int n_rows,
                 const AttnTileDev* tiles, int n_tiles, int QW, int H, int d, int nb_max, long long est_items,
                 const AttnScratch& sc, __nv_bfloat16* out, cudaStream_t st) {
    auto stage_of = [&](int G) { return 2 * static_cast<size_t>(kChunk) * ((H / G) * DH * 2 + 16); };
    auto fixed_of = [&](int G) {
        const size_t thr = 32 * (QW * H / G + 1);
        return static_cast<size_t>(8 * 8 + 4 * kMaxTileRows + 4 * (thr + 5) + 8 + 8 * (thr + 3)) + 128;
    };
    auto next_div = [&](int g) {
        int g2 = g + 1;
        while (H % g2) ++g2;
        return g2;
    };
    static const int regs = [] {
        cudaFuncAttributes fa{};
        return cudaFuncGetAttributes(&fa, attn_kernel<DH, MERGE>) == cudaSuccess && fa.numRegs > 0 ? fa.numRegs : 128;
    }();
    static const int env_sm = [] {
        const char* v = getenv("SGB_ATTN_PERSM");  // tuning experiments only
        return v ? atoi(v) : 0;
    }();
    static const int balance_env = [] {
        const char* v = getenv("SGB_ATTN_BALANCE");  // A/B: 0 = by item count, 1 = by weight
        return v ? atoi(v) : -1;
    }();
    // measured (scripts/bench_tree_attn.py, c3 rollouts): weighting pays when the shared tiles
    // hold > 8 verify rows (B <= 16 at C_peak 211); with 2-3 rows per sequence the item count
    // split is faster
    const int balance = balance_env >= 0 ? balance_env : (QW >= 2 ? 1 : 0);
    static const int g_force = [] {
        const char* v = getenv("SGB_ATTN_G");  // tuning experiments only
        return v ? atoi(v) : 0;
    }();
    static const int max_sm = [] {
        const char* v = getenv("SGB_ATTN_MAXSM");  // tuning experiments only
        return v ? std::max(1, std::min(16, atoi(v))) : 4;
    }();
    // CTAs per SM for a head grouping: shared memory for >= 2 stages each, and registers
    auto ctas_per_sm = [&](int G) {
        const int threads = 32 * (QW * (H / G) + 1);
        const int by_regs = std::max(1, 65536 / (threads * ((regs + 7) / 8 * 8)));
        int n = 0;
        while (n < std::min(by_regs, g_attn_sm_cap > 0 ? 1 : max_sm) && (n + 1) * (2 * stage_of(G) + fixed_of(G)) <= static_cast<size_t>(kSmemBudget) &&
               (n + 1) * threads <= 2048)
            ++n;
        return n;
    };
    // head groups: the grouping with the most consumer warps resident per SM (measured:
    // decode throughput follows it, scripts/bench_attn.py), ties to fewer groups; more
    // groups only when the launch has too few items to cover the SMs
    const int max_cons = MERGE ? kMaxConsMerge : kMaxCons;
    int G = 0, best = -1;
    for (int g = 1; g <= H; g = next_div(g)) {
        if (QW * (H / g) > max_cons) continue;
        const int n = ctas_per_sm(g);
        if (n == 0) continue;
        const int w = n * QW * (H / g);
        if (w > best) {
            best = w;
            G = g;
        }
        if (g == H) break;
    }
    if (G == 0) throw std::invalid_argument("attention: shared memory too small for the model width");
    while (G < H && est_items * G < 2 * 148 && ctas_per_sm(next_div(G)) > 0) G = next_div(G);
    if (g_force > 0 && H % g_force == 0 && QW * (H / g_force) <= max_cons && ctas_per_sm(g_force) > 0) G = g_force;
    const size_t stage = stage_of(G), fixed = fixed_of(G);
    const int threads = 32 * (QW * (H / G) + 1);
    int per_sm = ctas_per_sm(G);
    if (env_sm > 0 && env_sm <= per_sm) per_sm = env_sm;
    const int nst = static_cast<int>(std::min<size_t>(8, (kSmemBudget / per_sm - fixed) / stage));
    const size_t smem = nst * stage + fixed;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_kernel<DH, MERGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget);
        attr = true;
    }
    if (static_cast<long long>(n_rows) * G > sc.ctr_cap) throw std::invalid_argument("attention: row tickets too small");
    long long grid = std::max(1LL, std::min<long long>(est_items * G, 148LL * per_sm));
    if (g_attn_sm_cap > 0) grid = std::min<long long>(grid, g_attn_sm_cap);  // one CTA per SM on a subset of SMs
    launch_pdl(attn_kernel<DH, MERGE>, dim3(static_cast<unsigned>(grid)), dim3(threads), smem, st, q, K, V, rows, tiles,
               n_tiles, H, d, G, QW, nst, nb_max, balance, 1.0f / sqrtf(static_cast<float>(DH)), sc.part_acc, sc.part_ml,
               sc.row_ctr, out);
}

void launch_any(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, int n_rows,
                const AttnTileDev* tiles, int n_tiles, int QW, int H, int d, int max_virtual_len, long long est_items,
                const AttnScratch& sc, __nv_bfloat16* out, cudaStream_t st, bool merge_ok = false) {
    if (n_tiles <= 0) return;
    if (n_tiles > kMaxScanTiles) throw std::invalid_argument("attention: too many tiles in one launch");
    if (H > 64) throw std::invalid_argument("attention: at most 64 heads");
    const int dh = d / H;
    const int nb = attn_splits_for(max_virtual_len);
    static const int merge_env = [] {
        const char* v = getenv("SGB_ATTN_MERGE");  // A/B: 0 = publish every block partial
        return v ? atoi(v) : 1;
    }();
    // in-register block merge for shared tiles of <= 8 rows (QW = 1): measured (scripts/attn_merge_ab.sh)
    // 0.380 -> 0.333 ms at the c5 verify shape (48 x 4 rows, ctx 2200, 32 heads); with wider tiles
    // its 8-warp cap costs more occupancy than the partials it saves (16 x 13 rows: 0.15 -> 0.22 ms)
    const bool merge = tiles != nullptr && merge_ok && merge_env != 0 && (merge_env == 2 || QW == 1);
    if (dh == 128) {
        if (merge) launch_impl<128, true>(q, K, V, rows, n_rows, tiles, n_tiles, QW, H, d, nb, est_items, sc, out, st);
        else launch_impl<128, false>(q, K, V, rows, n_rows, tiles, n_tiles, QW, H, d, nb, est_items, sc, out, st);
    } else if (dh == 64) {
        if (merge) launch_impl<64, true>(q, K, V, rows, n_rows, tiles, n_tiles, QW, H, d, nb, est_items, sc, out, st);
        else launch_impl<64, false>(q, K, V, rows, n_rows, tiles, n_tiles, QW, H, d, nb, est_items, sc, out, st);
    } else {
        throw std::invalid_argument("attention: head dim must be 64 or 128");
    }
    SGB_KCHECK();
}

}  // namespace

int g_attn_sm_cap = 0;

int attn_splits_for(int max_virtual_len) { return (max_virtual_len + kBlock - 1) / kBlock; }

int attn_tile_qw(const std::vector<std::array<int, 4>>& groups) {
    int mx = 1;
    for (const auto& g : groups) mx = std::max(mx, g[1]);
    static const int cap = [] {
        const char* v = getenv("SGB_ATTN_QW");  // tuning experiments only
        return v ? std::max(1, std::min(kMaxCons / 2, atoi(v))) : 2;
    }();
    return std::min(cap, (mx + kQT - 1) / kQT);
}

long long build_attn_tiles(const std::vector<std::array<int, 4>>& groups, std::vector<AttnTileDev>& out, int qw,
                           bool boundary) {
    out.clear();
    long long n = 0;
    const int rows_per_tile = kQT * qw;
    static const int bnd_env = [] {
        const char* v = getenv("SGB_ATTN_BOUNDARY");  // A/B switch (0 = boundary blocks per row)
        return v ? atoi(v) : 1;
    }();
    boundary = boundary && bnd_env != 0;
    for (const auto& g : groups) {
        const int row0 = g[0], nr = g[1], ctx_len = g[2], vmax = g[3];
        const int nb = attn_splits_for(vmax);
        // blocks entirely inside the committed prefix are shared by the tile's rows; with
        // `boundary` so is the block holding the end of the prefix (its path chunks per row).
        // Measured (scripts/bench_tree_attn.py, profiles/r01_tree_boundary.txt): it pays when
        // that block starts with >= 1 whole prefix chunk, or with many rows per group; with
        // a few rows and no shared chunk the per-row items run in parallel instead (12 heads,
        // 16 x 13 rows, ctx 1100: 0.099 vs 0.123 ms)
        const bool bnd = boundary && nr > 1 && (ctx_len % kBlock >= kChunk || nr > 2 * kQT);
        const int nsb = nr > 1 ? std::min(nb, ctx_len / kBlock + (bnd ? 1 : 0)) : 0;
        const int bsh = bnd ? ctx_len : -1;
        // ... and the blocks that reach into each row's own tree path run per row, listed
        // right after the row's shared tile so every CTA's slice mixes heavy and light items
        for (int o = 0; o < nr; o += rows_per_tile) {
            const int nt = std::min(rows_per_tile, nr - o);
            if (nsb > 0) {
                out.push_back(AttnTileDev{row0 + o, nt, 0, nsb, bsh});
                n += nsb;
            }
            if (nb > nsb)
                for (int r = o; r < o + nt; ++r) {
                    out.push_back(AttnTileDev{row0 + r, 1, nsb, nb, -1});
                    n += nb - nsb;
                }
        }
    }
    return n;
}

void launch_attention(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, long long /*kv_slots*/,
                      const AttnRowsDev& rows, int M, int H, int d, int max_virtual_len, double total_keys,
                      const AttnScratch& sc, __nv_bfloat16* out, cudaStream_t st) {
    if (M <= 0) return;
    const long long est = static_cast<long long>(total_keys / kBlock) + M;
    launch_any(q, K, V, rows, M, nullptr, M, 1, H, d, max_virtual_len, est, sc, out, st);
}

void launch_attention_tiles(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, long long /*kv_slots*/,
                            const AttnRowsDev& rows, int M, const AttnTileDev* tiles, int n_tiles, long long n_items,
                            int qw, int H, int d, int max_virtual_len, const AttnScratch& sc, __nv_bfloat16* out,
                            cudaStream_t st, bool merge) {
    if (M <= 0) return;
    launch_any(q, K, V, rows, M, tiles, n_tiles, qw, H, d, max_virtual_len, n_items, sc, out, st, merge);
}

}  // namespace sgb
