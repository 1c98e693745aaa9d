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
// Kernel: one warp per (row, head, split of 256 virtual positions). Inside a split the
// warp walks 32-position chunks aligned to absolute virtual indices; each lane scores one
// key (bf16 K row, fp32 dot against the fp32 query), the warp does an online-softmax
// update per chunk, and the lane owning head dims [lane*DH/32, ...) accumulates P.V.
// Splits are merged by attn_combine_kernel in split order. Chunk and split boundaries
// depend only on the virtual index, so results are bit-identical between the AR path
// and the tree path (batch invariance, SURVEY.md §7 hard part 1).
//
// Roofline: HBM-bound on K/V reads (2*ctx*DH*2 bytes per (row,head)); see DESIGN.md.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kSplit = 256;
constexpr int kWarps = 4;

template <int DH>
__global__ void __launch_bounds__(32 * kWarps)
    attn_split_kernel(const float* __restrict__ q, const __nv_bfloat16* __restrict__ K,
                      const __nv_bfloat16* __restrict__ V, AttnRowsDev rows, int H, int d, int n_splits,
                      float scale, float* __restrict__ part_acc, float* __restrict__ part_ml) {
    constexpr int PL = DH / 32;  // dims per lane in P.V
    __shared__ __align__(16) float qs[kWarps][DH];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sp = blockIdx.x;
    const int h = blockIdx.y * kWarps + warp;
    const int r = blockIdx.z;
    if (h >= H) return;
    const int ctx_len = rows.ctx_len[r];
    const int chain_len = rows.chain_len[r];
    const int Lv = ctx_len + chain_len;
    const long long ctx_base = rows.ctx_base[r];
    const long long* chain = rows.chain_slots + static_cast<size_t>(r) * kMaxChain;
    const size_t pidx = (static_cast<size_t>(r) * H + h) * n_splits + sp;
    const int v0 = sp * kSplit;
    if (v0 >= Lv) {
        if (lane == 0) {
            part_ml[2 * pidx] = -INFINITY;
            part_ml[2 * pidx + 1] = 0.f;
        }
        return;
    }
    const int v1 = min(Lv, v0 + kSplit);
    const float* qrow = q + static_cast<size_t>(r) * d + h * DH;
    for (int e = lane; e < DH; e += 32) qs[warp][e] = qrow[e];
    __syncwarp();

    float m = -INFINITY, l = 0.f;
    float acc[PL];
#pragma unroll
    for (int i = 0; i < PL; ++i) acc[i] = 0.f;

    for (int c = v0; c < v1; c += 32) {
        const int v = c + lane;
        const bool valid = v < v1;
        long long slot = 0;
        if (valid) slot = v < ctx_len ? ctx_base + v : chain[v - ctx_len];
        float s = -INFINITY;
        if (valid) {
            // all 16-byte pieces of this lane's key row are issued before any math so the
            // whole row (DH*2 bytes) is in flight at once
            const uint4* kr = reinterpret_cast<const uint4*>(K + slot * d + h * DH);
            uint4 kreg[DH / 8];
#pragma unroll
            for (int e8 = 0; e8 < DH / 8; ++e8) kreg[e8] = __ldg(kr + e8);
            float dot = 0.f;
#pragma unroll
            for (int e8 = 0; e8 < DH / 8; ++e8) {
                const uint4 u = kreg[e8];
                const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 f = __bfloat1622float2(b2[t]);
                    dot = fmaf(qs[warp][e8 * 8 + 2 * t], f.x, dot);
                    dot = fmaf(qs[warp][e8 * 8 + 2 * t + 1], f.y, dot);
                }
            }
            s = dot * scale;
        }
        const float cm = warp_max(s);
        const float nm = fmaxf(m, cm);
        const float alpha = (m == -INFINITY) ? 0.f : expf(m - nm);
        const float p = valid ? expf(s - nm) : 0.f;
        l = l * alpha + warp_sum(p);
#pragma unroll
        for (int i = 0; i < PL; ++i) acc[i] *= alpha;
        const int nvalid = min(32, v1 - c);
        // P.V over the chunk: fully unrolled so the 32 value-row loads (one coalesced
        // DH*2-byte row per key across the warp) are all in flight before the FMAs; the
        // accumulation order stays j = 0..31.
        if constexpr (PL == 4) {
            uint2 vv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const long long sj = __shfl_sync(0xffffffffu, slot, j);
                if (j < nvalid) vv[j] = __ldg(reinterpret_cast<const uint2*>(V + sj * d + h * DH + lane * PL));
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float pj = __shfl_sync(0xffffffffu, p, j);
                if (j < nvalid) {
                    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[j].x));
                    const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[j].y));
                    acc[0] = fmaf(pj, a.x, acc[0]);
                    acc[1] = fmaf(pj, a.y, acc[1]);
                    acc[2] = fmaf(pj, b.x, acc[2]);
                    acc[3] = fmaf(pj, b.y, acc[3]);
                }
            }
        } else if constexpr (PL == 2) {
            unsigned vv[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const long long sj = __shfl_sync(0xffffffffu, slot, j);
                if (j < nvalid) vv[j] = __ldg(reinterpret_cast<const unsigned*>(V + sj * d + h * DH + lane * PL));
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float pj = __shfl_sync(0xffffffffu, p, j);
                if (j < nvalid) {
                    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&vv[j]));
                    acc[0] = fmaf(pj, a.x, acc[0]);
                    acc[1] = fmaf(pj, a.y, acc[1]);
                }
            }
        } else {
            for (int j = 0; j < nvalid; ++j) {
                const float pj = __shfl_sync(0xffffffffu, p, j);
                const long long sj = __shfl_sync(0xffffffffu, slot, j);
                const __nv_bfloat16* vr = V + sj * d + h * DH + lane * PL;
#pragma unroll
                for (int i = 0; i < PL; ++i) acc[i] = fmaf(pj, __bfloat162float(vr[i]), acc[i]);
            }
        }
        m = nm;
    }
    float* pa = part_acc + pidx * DH + lane * PL;
#pragma unroll
    for (int i = 0; i < PL; ++i) pa[i] = acc[i];
    if (lane == 0) {
        part_ml[2 * pidx] = m;
        part_ml[2 * pidx + 1] = l;
    }
}

// Merge the splits of one (row, head) in split order -> bf16 attention output.
template <int DH>
__global__ void attn_combine_kernel(const float* __restrict__ part_acc, const float* __restrict__ part_ml, int H,
                                    int n_splits, __nv_bfloat16* __restrict__ out, int d) {
    const int r = blockIdx.x, h = blockIdx.y;
    const size_t base = (static_cast<size_t>(r) * H + h) * n_splits;
    float M = -INFINITY;
    for (int s = 0; s < n_splits; ++s) M = fmaxf(M, part_ml[2 * (base + s)]);
    float L = 0.f;
    for (int s = 0; s < n_splits; ++s) {
        const float ms = part_ml[2 * (base + s)];
        if (ms != -INFINITY) L += part_ml[2 * (base + s) + 1] * expf(ms - M);
    }
    for (int e = threadIdx.x; e < DH; e += blockDim.x) {
        float o = 0.f;
        for (int s = 0; s < n_splits; ++s) {
            const float ms = part_ml[2 * (base + s)];
            if (ms != -INFINITY) o += part_acc[(base + s) * DH + e] * expf(ms - M);
        }
        out[static_cast<size_t>(r) * d + h * DH + e] = __float2bfloat16(o / L);
    }
}

}  // namespace

int attn_splits_for(int max_virtual_len) { return (max_virtual_len + kSplit - 1) / kSplit; }

void launch_attention(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows, int M,
                      int H, int d, int max_virtual_len, float* part_acc, float* part_ml, __nv_bfloat16* out,
                      cudaStream_t st) {
    if (M <= 0) return;
    const int dh = d / H;
    const int ns = attn_splits_for(max_virtual_len);
    const float scale = 1.0f / sqrtf(static_cast<float>(dh));
    dim3 grid(ns, (H + kWarps - 1) / kWarps, M);
    switch (dh) {
        case 64:
            attn_split_kernel<64><<<grid, 32 * kWarps, 0, st>>>(q, K, V, rows, H, d, ns, scale, part_acc, part_ml);
            SGB_KCHECK();
            attn_combine_kernel<64><<<dim3(M, H), 64, 0, st>>>(part_acc, part_ml, H, ns, out, d);
            break;
        case 128:
            attn_split_kernel<128><<<grid, 32 * kWarps, 0, st>>>(q, K, V, rows, H, d, ns, scale, part_acc, part_ml);
            SGB_KCHECK();
            attn_combine_kernel<128><<<dim3(M, H), 128, 0, st>>>(part_acc, part_ml, H, ns, out, d);
            break;
        case 256:
            attn_split_kernel<256><<<grid, 32 * kWarps, 0, st>>>(q, K, V, rows, H, d, ns, scale, part_acc, part_ml);
            SGB_KCHECK();
            attn_combine_kernel<256><<<dim3(M, H), 128, 0, st>>>(part_acc, part_ml, H, ns, out, d);
            break;
        default:
            throw std::invalid_argument("attention: head dim must be 64, 128 or 256");
    }
    SGB_KCHECK();
}

}  // namespace sgb
