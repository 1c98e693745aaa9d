// Causal self-attention of the draft-training forward/backward on tensor cores.
//
// Replaces the reference's per-row scalar attention of the training blocks
// (include/sgrpo/tinylm.hpp:653-718 forward, :720-800 backward; used by
// draft_train_forward/backward, tinylm.hpp:881-953). The training chunk holds whole
// sequences back to back; row i attends keys j with seq_first[i] <= j <= i.
//
// FlashAttention-2 formulation with mma.sync.m16n8k16 (bf16 in, fp32 accumulate):
//   fwd   CTA = (64 query rows, head): stream 64-key tiles, online softmax, O and lse.
//   dKV   CTA = (64 keys, head): stream query tiles, recompute P, dV += P^T dO,
//         dK += dS^T Q.
//   dQ    CTA = (64 query rows, head): stream key tiles, dQ += dS K.
// Tiles never straddle sequences: a CTA's 64 rows (queries or keys) and every tile it
// streams start at seq_first + 64m, so a row's arithmetic does not depend on where its
// sequence sits in the training chunk or which sequences share it (the data-parallel
// shards then sum to the full-batch gradient). Two passes instead of atomics keep the
// update deterministic run to run. Operands are
// staged fp32 -> bf16 in shared memory (row stride DH+8 / 72 halves: conflict-free u32
// fragment loads). The weights are updated from these gradients, so the bf16 rounding sits
// inside the fp32-tolerance contract of draft_update (tests/test_gpu_draft_update.py).
#include <cuda_bf16.h>

#include <cfloat>

#include "common.cuh"
#include "train.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kTile = 64;   // rows (queries or keys) per CTA and per streamed tile
constexpr int kWarps = 4;   // 16 rows each
constexpr int kThr = 32 * kWarps;
constexpr int kTS = kTile + 8;  // transposed-tile row stride (halves)

__device__ __forceinline__ void mma16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t lds32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }

// fp32 rows [row0, row0+64) x [col, col+DH) of a row-major matrix (leading dim ld) ->
// bf16 smem tile [64][DH+8] (rows beyond R are zero).
template <int DH>
__device__ void stage_rows(const float* __restrict__ src, int ld, int col, int row0, int R, __nv_bfloat16* dst) {
    constexpr int S = DH + 8;
    for (int idx = threadIdx.x; idx < kTile * DH / 2; idx += kThr) {
        const int r = idx / (DH / 2), e = 2 * (idx % (DH / 2));
        float2 v = make_float2(0.f, 0.f);
        if (row0 + r < R) v = *reinterpret_cast<const float2*>(src + static_cast<size_t>(row0 + r) * ld + col + e);
        *reinterpret_cast<uint32_t*>(dst + r * S + e) = pack2(v.x, v.y);
    }
}
// same rows, transposed: bf16 smem tile [DH][64+8]
template <int DH>
__device__ void stage_cols(const float* __restrict__ src, int ld, int col, int row0, int R, __nv_bfloat16* dst) {
    for (int idx = threadIdx.x; idx < kTile * DH / 2; idx += kThr) {
        const int r = idx / (DH / 2), e = 2 * (idx % (DH / 2));
        float2 v = make_float2(0.f, 0.f);
        if (row0 + r < R) v = *reinterpret_cast<const float2*>(src + static_cast<size_t>(row0 + r) * ld + col + e);
        dst[e * kTS + r] = __float2bfloat16(v.x);
        dst[(e + 1) * kTS + r] = __float2bfloat16(v.y);
    }
}
// A fragments of a warp's 16 rows x DH straight from fp32 global (row0 = first row of the warp)
template <int DH>
__device__ void load_afrag(const float* __restrict__ src, int ld, int col, int row0, int R, uint32_t (*a)[4]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ra = row0 + g, rb = row0 + g + 8;
#pragma unroll
    for (int ks = 0; ks < DH / 16; ++ks) {
        const int e0 = ks * 16 + 2 * t, e1 = e0 + 8;
        float2 x0 = make_float2(0.f, 0.f), x1 = x0, x2 = x0, x3 = x0;
        if (ra < R) {
            x0 = *reinterpret_cast<const float2*>(src + static_cast<size_t>(ra) * ld + col + e0);
            x2 = *reinterpret_cast<const float2*>(src + static_cast<size_t>(ra) * ld + col + e1);
        }
        if (rb < R) {
            x1 = *reinterpret_cast<const float2*>(src + static_cast<size_t>(rb) * ld + col + e0);
            x3 = *reinterpret_cast<const float2*>(src + static_cast<size_t>(rb) * ld + col + e1);
        }
        a[ks][0] = pack2(x0.x, x0.y);
        a[ks][1] = pack2(x1.x, x1.y);
        a[ks][2] = pack2(x2.x, x2.y);
        a[ks][3] = pack2(x3.x, x3.y);
    }
}

// A fragment (k-step ks) of rows r0..r0+15 of a staged [64][DH+8] tile
template <int DH>
__device__ __forceinline__ void afrag_smem(const __nv_bfloat16* tile, int r0, int ks, uint32_t* a) {
    constexpr int S = DH + 8;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const __nv_bfloat16* p = tile + (r0 + g) * S + ks * 16 + 2 * t;
    a[0] = lds32(p);
    a[1] = lds32(p + 8 * S);
    a[2] = lds32(p + 8);
    a[3] = lds32(p + 8 * S + 8);
}

// ---------------------------------------------------------------- forward
template <int DH>
__global__ void __launch_bounds__(kThr) tattn_fwd_kernel(const float* __restrict__ qkv, const int* __restrict__ seq_first,
                                                         const int* __restrict__ seq_last, const int* __restrict__ tiles,
                                                         int d, int H, float scale, float* __restrict__ ctx,
                                                         __nv_bfloat16* __restrict__ ctx_b, float* __restrict__ lse) {
    constexpr int S = DH + 8;
    extern __shared__ __align__(16) __nv_bfloat16 sm[];
    __nv_bfloat16* Ks = sm;              // [64][DH+8]
    __nv_bfloat16* Vt = sm + kTile * S;  // [DH][72]
    const int h = blockIdx.y, i0 = tiles[blockIdx.x];
    const int sf = seq_first[i0], R = min(i0 + kTile, seq_last[i0] + 1);  // rows [i0, R) of one sequence
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ld = 3 * d, cq = h * DH, ck = d + h * DH, cv = 2 * d + h * DH;
    const int wr = i0 + warp * 16;
    uint32_t qa[DH / 16][4];
    load_afrag<DH>(qkv, ld, cq, wr, R, qa);
    const int rowa = wr + g, rowb = wr + g + 8;
    const int fa = rowa < R ? sf : 0x7fffffff, fb = rowb < R ? sf : 0x7fffffff;
    float o[DH / 8][4];
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float ma = -INFINITY, mb = -INFINITY, la = 0.f, lb = 0.f;
    for (int k0 = sf; k0 < R; k0 += kTile) {
        __syncthreads();
        stage_rows<DH>(qkv, ld, ck, k0, R, Ks);
        stage_cols<DH>(qkv, ld, cv, k0, R, Vt);
        __syncthreads();
        float s[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
#pragma unroll
            for (int ks = 0; ks < DH / 16; ++ks) {
                const __nv_bfloat16* kp = Ks + (nt * 8 + g) * S + ks * 16 + 2 * t;
                mma16816(s[nt], qa[ks], lds32(kp), lds32(kp + 8));
            }
        }
        // mask + scale, row maxima over the quad
        float xa = -INFINITY, xb = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int j = k0 + nt * 8 + 2 * t + u;
                s[nt][u] = (j >= fa && j <= rowa) ? s[nt][u] * scale : -INFINITY;
                s[nt][2 + u] = (j >= fb && j <= rowb) ? s[nt][2 + u] * scale : -INFINITY;
                xa = fmaxf(xa, s[nt][u]);
                xb = fmaxf(xb, s[nt][2 + u]);
            }
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 1));
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 2));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 1));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 2));
        const float na = fmaxf(ma, xa), nb = fmaxf(mb, xb);
        const float aa = (na == -INFINITY) ? 1.f : expf(ma - na), ab = (nb == -INFINITY) ? 1.f : expf(mb - nb);
        float sa = 0.f, sb = 0.f;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                s[nt][u] = (s[nt][u] == -INFINITY) ? 0.f : expf(s[nt][u] - na);
                s[nt][2 + u] = (s[nt][2 + u] == -INFINITY) ? 0.f : expf(s[nt][2 + u] - nb);
                sa += s[nt][u];
                sb += s[nt][2 + u];
            }
        sa += __shfl_xor_sync(0xffffffffu, sa, 1);
        sa += __shfl_xor_sync(0xffffffffu, sa, 2);
        sb += __shfl_xor_sync(0xffffffffu, sb, 1);
        sb += __shfl_xor_sync(0xffffffffu, sb, 2);
        la = la * aa + sa;
        lb = lb * ab + sb;
        ma = na;
        mb = nb;
#pragma unroll
        for (int n = 0; n < DH / 8; ++n) {
            o[n][0] *= aa;
            o[n][1] *= aa;
            o[n][2] *= ab;
            o[n][3] *= ab;
        }
        // O += P V
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t pa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                              pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
            for (int n = 0; n < DH / 8; ++n) {
                const __nv_bfloat16* vp = Vt + (n * 8 + g) * kTS + kk * 16 + 2 * t;
                mma16816(o[n], pa, lds32(vp), lds32(vp + 8));
            }
        }
    }
    const float ia = la > 0.f ? 1.f / la : 0.f, ib = lb > 0.f ? 1.f / lb : 0.f;
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) {
        const int e = h * DH + n * 8 + 2 * t;
        if (rowa < R) {
            const float x = o[n][0] * ia, y = o[n][1] * ia;
            *reinterpret_cast<float2*>(ctx + static_cast<size_t>(rowa) * d + e) = make_float2(x, y);
            *reinterpret_cast<uint32_t*>(ctx_b + static_cast<size_t>(rowa) * d + e) = pack2(x, y);
        }
        if (rowb < R) {
            const float x = o[n][2] * ib, y = o[n][3] * ib;
            *reinterpret_cast<float2*>(ctx + static_cast<size_t>(rowb) * d + e) = make_float2(x, y);
            *reinterpret_cast<uint32_t*>(ctx_b + static_cast<size_t>(rowb) * d + e) = pack2(x, y);
        }
    }
    if (t == 0) {
        if (rowa < R) lse[static_cast<size_t>(rowa) * H + h] = ma + logf(la);
        if (rowb < R) lse[static_cast<size_t>(rowb) * H + h] = mb + logf(lb);
    }
}

// D_i = dO_i . O_i per (row, head)
__global__ void tattn_rowdot_kernel(const float* __restrict__ ctx, const float* __restrict__ dctx, int R, int d, int H,
                                    float* __restrict__ Drow) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= R * H) return;
    const int i = w / H, h = w - i * H, dh = d / H;
    float s = 0.f;
    for (int e = lane; e < dh; e += 32) s += ctx[static_cast<size_t>(i) * d + h * dh + e] * dctx[static_cast<size_t>(i) * d + h * dh + e];
    s = warp_sum(s);
    if (lane == 0) Drow[w] = s;
}

// ---------------------------------------------------------------- dK, dV
template <int DH>
__global__ void __launch_bounds__(kThr) tattn_dkv_kernel(const float* __restrict__ qkv, const float* __restrict__ dctx,
                                                         const float* __restrict__ lse, const float* __restrict__ Drow,
                                                         const int* __restrict__ seq_first, const int* __restrict__ seq_last,
                                                         const int* __restrict__ tiles, int d, int H, float scale,
                                                         float* __restrict__ dqkv) {
    constexpr int S = DH + 8;
    extern __shared__ __align__(16) __nv_bfloat16 sm[];
    __nv_bfloat16* Qs = sm;                    // [64][DH+8]  rows x dims
    __nv_bfloat16* dOs = Qs + kTile * S;       // [64][DH+8]
    __nv_bfloat16* QT = dOs + kTile * S;       // [DH][72]    dims x rows
    __nv_bfloat16* dOT = QT + DH * kTS;        // [DH][72]
    __nv_bfloat16* Kc = dOT + DH * kTS;        // [64][DH+8]  this CTA's keys
    __nv_bfloat16* Vc = Kc + kTile * S;        // [64][DH+8]
    float* Ls = reinterpret_cast<float*>(Vc + kTile * S);  // [64] lse
    float* Ds = Ls + kTile;                                // [64] D
    int* Fs = reinterpret_cast<int*>(Ds + kTile);          // [64] seq_first
    const int h = blockIdx.y, j0 = tiles[blockIdx.x];
    const int R = seq_last[j0] + 1;                 // rows of this sequence end here
    const int KR = min(j0 + kTile, R);              // keys [j0, KR)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ld = 3 * d, cq = h * DH, ck = d + h * DH, cv = 2 * d + h * DH;
    const int wk = j0 + warp * 16;  // this warp's 16 keys
    stage_rows<DH>(qkv, ld, ck, j0, KR, Kc);
    stage_rows<DH>(qkv, ld, cv, j0, KR, Vc);
    const int keya = wk + g, keyb = wk + g + 8;
    float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
    for (int n = 0; n < DH / 8; ++n)
#pragma unroll
        for (int u = 0; u < 4; ++u) dk[n][u] = dv[n][u] = 0.f;
    for (int q0 = j0; q0 < R; q0 += kTile) {
        __syncthreads();
        stage_rows<DH>(qkv, ld, cq, q0, R, Qs);
        stage_rows<DH>(dctx, d, h * DH, q0, R, dOs);
        stage_cols<DH>(qkv, ld, cq, q0, R, QT);
        stage_cols<DH>(dctx, d, h * DH, q0, R, dOT);
        for (int r = threadIdx.x; r < kTile; r += kThr) {
            const bool ok = q0 + r < R;
            Ls[r] = ok ? lse[static_cast<size_t>(q0 + r) * H + h] : 0.f;
            Ds[r] = ok ? Drow[static_cast<size_t>(q0 + r) * H + h] : 0.f;
            Fs[r] = ok ? seq_first[q0 + r] : 0x7fffffff;
        }
        __syncthreads();
        // S^T (16 keys x 64 rows) = K Q^T ; dP^T = V dO^T
        float st[8][4], dpt[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
            for (int u = 0; u < 4; ++u) st[nt][u] = dpt[nt][u] = 0.f;
#pragma unroll
            for (int ks = 0; ks < DH / 16; ++ks) {
                uint32_t ka[4], va[4];
                afrag_smem<DH>(Kc, warp * 16, ks, ka);
                afrag_smem<DH>(Vc, warp * 16, ks, va);
                const __nv_bfloat16* qp = Qs + (nt * 8 + g) * S + ks * 16 + 2 * t;
                mma16816(st[nt], ka, lds32(qp), lds32(qp + 8));
                const __nv_bfloat16* op = dOs + (nt * 8 + g) * S + ks * 16 + 2 * t;
                mma16816(dpt[nt], va, lds32(op), lds32(op + 8));
            }
        }
        // P^T, dS^T (rows i = q0 + nt*8 + 2t + u, keys keya / keyb)
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int ri = nt * 8 + 2 * t + u, i = q0 + ri;
                const bool va_ = i < R && keya <= i && keya < KR;
                const bool vb_ = i < R && keyb <= i && keyb < KR;
                const float pa = va_ ? expf(st[nt][u] * scale - Ls[ri]) : 0.f;
                const float pb = vb_ ? expf(st[nt][2 + u] * scale - Ls[ri]) : 0.f;
                st[nt][u] = pa;
                st[nt][2 + u] = pb;
                dpt[nt][u] = pa * (dpt[nt][u] - Ds[ri]);
                dpt[nt][2 + u] = pb * (dpt[nt][2 + u] - Ds[ri]);
            }
        // dV += P^T dO ; dK += dS^T Q
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t pa[4] = {pack2(st[2 * kk][0], st[2 * kk][1]), pack2(st[2 * kk][2], st[2 * kk][3]),
                              pack2(st[2 * kk + 1][0], st[2 * kk + 1][1]), pack2(st[2 * kk + 1][2], st[2 * kk + 1][3])};
            uint32_t sa[4] = {pack2(dpt[2 * kk][0], dpt[2 * kk][1]), pack2(dpt[2 * kk][2], dpt[2 * kk][3]),
                              pack2(dpt[2 * kk + 1][0], dpt[2 * kk + 1][1]),
                              pack2(dpt[2 * kk + 1][2], dpt[2 * kk + 1][3])};
#pragma unroll
            for (int n = 0; n < DH / 8; ++n) {
                const __nv_bfloat16* op = dOT + (n * 8 + g) * kTS + kk * 16 + 2 * t;
                mma16816(dv[n], pa, lds32(op), lds32(op + 8));
                const __nv_bfloat16* qp = QT + (n * 8 + g) * kTS + kk * 16 + 2 * t;
                mma16816(dk[n], sa, lds32(qp), lds32(qp + 8));
            }
        }
    }
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) {
        const int e = n * 8 + 2 * t;
        if (keya < KR) {
            *reinterpret_cast<float2*>(dqkv + static_cast<size_t>(keya) * ld + ck + e) =
                make_float2(dk[n][0] * scale, dk[n][1] * scale);
            *reinterpret_cast<float2*>(dqkv + static_cast<size_t>(keya) * ld + cv + e) = make_float2(dv[n][0], dv[n][1]);
        }
        if (keyb < KR) {
            *reinterpret_cast<float2*>(dqkv + static_cast<size_t>(keyb) * ld + ck + e) =
                make_float2(dk[n][2] * scale, dk[n][3] * scale);
            *reinterpret_cast<float2*>(dqkv + static_cast<size_t>(keyb) * ld + cv + e) = make_float2(dv[n][2], dv[n][3]);
        }
    }
}

// ---------------------------------------------------------------- dQ
template <int DH>
__global__ void __launch_bounds__(kThr) tattn_dq_kernel(const float* __restrict__ qkv, const float* __restrict__ dctx,
                                                        const float* __restrict__ lse, const float* __restrict__ Drow,
                                                        const int* __restrict__ seq_first, const int* __restrict__ seq_last,
                                                        const int* __restrict__ tiles, int d, int H, float scale,
                                                        float* __restrict__ dqkv) {
    constexpr int S = DH + 8;
    extern __shared__ __align__(16) __nv_bfloat16 sm[];
    __nv_bfloat16* Ks = sm;               // [64][DH+8]
    __nv_bfloat16* Vs = Ks + kTile * S;   // [64][DH+8]
    __nv_bfloat16* KT = Vs + kTile * S;   // [DH][72]
    __nv_bfloat16* Qc = KT + DH * kTS;    // [64][DH+8]  this CTA's query rows
    __nv_bfloat16* Oc = Qc + kTile * S;   // [64][DH+8]  their dO
    const int h = blockIdx.y, i0 = tiles[blockIdx.x];
    const int sf = seq_first[i0], R = min(i0 + kTile, seq_last[i0] + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int ld = 3 * d, cq = h * DH, ck = d + h * DH, cv = 2 * d + h * DH;
    const int wr = i0 + warp * 16;
    stage_rows<DH>(qkv, ld, cq, i0, R, Qc);
    stage_rows<DH>(dctx, d, h * DH, i0, R, Oc);
    const int rowa = wr + g, rowb = wr + g + 8;
    const int fa = rowa < R ? sf : 0x7fffffff, fb = rowb < R ? sf : 0x7fffffff;
    const float La = rowa < R ? lse[static_cast<size_t>(rowa) * H + h] : 0.f;
    const float Lb = rowb < R ? lse[static_cast<size_t>(rowb) * H + h] : 0.f;
    const float Da = rowa < R ? Drow[static_cast<size_t>(rowa) * H + h] : 0.f;
    const float Db = rowb < R ? Drow[static_cast<size_t>(rowb) * H + h] : 0.f;
    float dq[DH / 8][4];
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) dq[n][0] = dq[n][1] = dq[n][2] = dq[n][3] = 0.f;
    for (int k0 = sf; k0 < R; k0 += kTile) {
        __syncthreads();
        stage_rows<DH>(qkv, ld, ck, k0, R, Ks);
        stage_rows<DH>(qkv, ld, cv, k0, R, Vs);
        stage_cols<DH>(qkv, ld, ck, k0, R, KT);
        __syncthreads();
        float s[8][4], dp[8][4];
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
            for (int u = 0; u < 4; ++u) s[nt][u] = dp[nt][u] = 0.f;
#pragma unroll
            for (int ks = 0; ks < DH / 16; ++ks) {
                uint32_t qa[4], oa[4];
                afrag_smem<DH>(Qc, warp * 16, ks, qa);
                afrag_smem<DH>(Oc, warp * 16, ks, oa);
                const __nv_bfloat16* kp = Ks + (nt * 8 + g) * S + ks * 16 + 2 * t;
                mma16816(s[nt], qa, lds32(kp), lds32(kp + 8));
                const __nv_bfloat16* vp = Vs + (nt * 8 + g) * S + ks * 16 + 2 * t;
                mma16816(dp[nt], oa, lds32(vp), lds32(vp + 8));
            }
        }
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int j = k0 + nt * 8 + 2 * t + u;
                const float pa = (j >= fa && j <= rowa) ? expf(s[nt][u] * scale - La) : 0.f;
                const float pb = (j >= fb && j <= rowb) ? expf(s[nt][2 + u] * scale - Lb) : 0.f;
                s[nt][u] = pa * (dp[nt][u] - Da);
                s[nt][2 + u] = pb * (dp[nt][2 + u] - Db);
            }
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            uint32_t sa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                              pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
            for (int n = 0; n < DH / 8; ++n) {
                const __nv_bfloat16* kp = KT + (n * 8 + g) * kTS + kk * 16 + 2 * t;
                mma16816(dq[n], sa, lds32(kp), lds32(kp + 8));
            }
        }
    }
#pragma unroll
    for (int n = 0; n < DH / 8; ++n) {
        const int e = n * 8 + 2 * t;
        if (rowa < R)
            *reinterpret_cast<float2*>(dqkv + static_cast<size_t>(rowa) * ld + cq + e) =
                make_float2(dq[n][0] * scale, dq[n][1] * scale);
        if (rowb < R)
            *reinterpret_cast<float2*>(dqkv + static_cast<size_t>(rowb) * ld + cq + e) =
                make_float2(dq[n][2] * scale, dq[n][3] * scale);
    }
}

template <int DH>
void fwd_impl(const float* qkv, const int* seq_first, const int* seq_last, const int* tiles, int n_tiles, int d, int H,
              float* ctx, __nv_bfloat16* ctx_b, float* lse, cudaStream_t st) {
    const size_t smem = (static_cast<size_t>(kTile) * (DH + 8) + static_cast<size_t>(DH) * kTS) * 2;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tattn_fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        attr = true;
    }
    const float scale = 1.0f / sqrtf(static_cast<float>(DH));
    tattn_fwd_kernel<DH><<<dim3(n_tiles, H), kThr, smem, st>>>(qkv, seq_first, seq_last, tiles, d, H, scale, ctx, ctx_b,
                                                              lse);
    SGB_KCHECK();
}

template <int DH>
void bwd_impl(const float* qkv, const float* ctx, const float* dctx, const float* lse, const int* seq_first,
              const int* seq_last, const int* tiles, int n_tiles, int R, int d, int H, float* Drow, float* dqkv,
              cudaStream_t st) {
    const float scale = 1.0f / sqrtf(static_cast<float>(DH));
    const int warps = R * H;
    tattn_rowdot_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(ctx, dctx, R, d, H, Drow);
    SGB_KCHECK();
    const size_t smem_kv = (4 * static_cast<size_t>(kTile) * (DH + 8) + 2 * static_cast<size_t>(DH) * kTS) * 2 +
                           3 * kTile * 4;
    const size_t smem_q = (4 * static_cast<size_t>(kTile) * (DH + 8) + static_cast<size_t>(DH) * kTS) * 2;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tattn_dkv_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_kv));
        cudaFuncSetAttribute(tattn_dq_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_q));
        attr = true;
    }
    const dim3 grid(n_tiles, H);
    tattn_dkv_kernel<DH><<<grid, kThr, smem_kv, st>>>(qkv, dctx, lse, Drow, seq_first, seq_last, tiles, d, H, scale,
                                                      dqkv);
    SGB_KCHECK();
    tattn_dq_kernel<DH><<<grid, kThr, smem_q, st>>>(qkv, dctx, lse, Drow, seq_first, seq_last, tiles, d, H, scale, dqkv);
    SGB_KCHECK();
}

}  // namespace

void launch_train_attn_fwd(const float* qkv, const int* seq_first, const int* seq_last, const int* tiles, int n_tiles,
                           int d, int H, float* ctx, __nv_bfloat16* ctx_b, float* lse, cudaStream_t st) {
    if (n_tiles <= 0) return;
    const int dh = d / H;
    if (dh == 128) fwd_impl<128>(qkv, seq_first, seq_last, tiles, n_tiles, d, H, ctx, ctx_b, lse, st);
    else if (dh == 64) fwd_impl<64>(qkv, seq_first, seq_last, tiles, n_tiles, d, H, ctx, ctx_b, lse, st);
    else throw std::invalid_argument("train attention: head dim must be 64 or 128");
}

void launch_train_attn_bwd(const float* qkv, const float* ctx, const float* dctx, const float* lse,
                           const int* seq_first, const int* seq_last, const int* tiles, int n_tiles, int R, int d,
                           int H, float* Drow, float* dqkv, cudaStream_t st) {
    if (n_tiles <= 0) return;
    const int dh = d / H;
    if (dh == 128) bwd_impl<128>(qkv, ctx, dctx, lse, seq_first, seq_last, tiles, n_tiles, R, d, H, Drow, dqkv, st);
    else if (dh == 64) bwd_impl<64>(qkv, ctx, dctx, lse, seq_first, seq_last, tiles, n_tiles, R, d, H, Drow, dqkv, st);
    else throw std::invalid_argument("train attention: head dim must be 64 or 128");
}

}  // namespace sgb
