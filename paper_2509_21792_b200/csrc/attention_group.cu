// Prefix-shared tree attention: the verify rows of one sequence (and the frontier rows of
// one draft level) read the sequence's committed K/V once per tile instead of once per row.
//
// Reference semantics: the same decode_blocks attention (include/sgrpo/tinylm.hpp:335-395)
// under build_tree_mask (src/drafttree.cpp:145-168): row i of a sequence's tree attends to
// the committed cache [0, p) plus its own ancestors-or-self chain. The reference evaluates
// each row separately; on the B200 the per-row kernel (attention.cu) does the same and so
// streams the prefix N_verify times per step -- at c3's B=1 tail that is 211 x 257 MB per
// step, the largest single cost of a speculative step.
//
// Tile = up to 64 consecutive rows with one (ctx_base, ctx_len, shared prompt) -- one
// sequence's rows. Work item = (tile, 64-key block, head). The block's committed keys
// ([kb, min(kb+64, ctx_len))) are staged once into shared memory (cp.async, padded rows)
// and used by every row of the tile; chain (tree-path) keys past ctx_len are row-specific
// and are read per row from the scratch slots (L2-resident, at most kMaxChain per row).
// Scores run as a register-tiled CUDA-core product (2 rows x 4 keys per thread), softmax
// per row per KPC-key chunk, then P.V (4 rows x DH/16 dims per thread). The last item of a
// (tile, head) merges each row's block partials in block order (atomic ticket).
//
// Bit-identity with the per-row kernel: every (row, key) score, chunk softmax step, P.V
// accumulation and the merge use the helpers of attn_numerics.cuh in the same order, with
// chunk/block boundaries fixed in virtual key index. So a tree row computed here equals the
// AR row of the same token computed by attention.cu bit for bit (spec == AR rollouts).
//
// Roofline: per item 2*64*DH*2 bytes of K/V (HBM, once per tile instead of once per row)
// and 4*DH flops per (row, key); at N_verify >= 13 rows per sequence the tile is bound by
// the CUDA-core FMA rate rather than by HBM.
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "attn_numerics.cuh"
#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kGT = 256;    // threads per CTA
constexpr int kGR = kAttnTileRows;  // rows per tile
constexpr int kGB = kAttnBlock;     // keys per block

SGB_DEV void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
SGB_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int NP>
SGB_DEV constexpr int piece_at(int i) {
    // butterfly order of the per-row kernel: pieces combined as ((0+4)+(2+6))+((1+5)+(3+7))
    if constexpr (NP == 8) {
        constexpr int o[8] = {0, 4, 2, 6, 1, 5, 3, 7};
        return o[i];
    } else {
        constexpr int o[4] = {0, 2, 1, 3};
        return o[i];
    }
}

// Fold piece partial `a` (the i-th in piece_at order) into the running tree state.
template <int NP>
SGB_DEV void tree_fold(int i, float a, float& T, float& S, float& X, float& dot) {
    if constexpr (NP == 8) {
        switch (i) {
            case 0: T = a; break;
            case 1: S = __fadd_rn(T, a); break;
            case 2: T = a; break;
            case 3: X = __fadd_rn(S, __fadd_rn(T, a)); break;
            case 4: T = a; break;
            case 5: S = __fadd_rn(T, a); break;
            case 6: T = a; break;
            default: dot = __fadd_rn(X, __fadd_rn(S, __fadd_rn(T, a))); break;
        }
    } else {
        switch (i) {
            case 0: T = a; break;
            case 1: X = __fadd_rn(T, a); break;
            case 2: T = a; break;
            default: dot = __fadd_rn(X, __fadd_rn(T, a)); break;
        }
    }
}

SGB_DEV void bf16x16_to_f32(const uint4& u0, const uint4& u1, float* k) {
    const __nv_bfloat162* b0 = reinterpret_cast<const __nv_bfloat162*>(&u0);
    const __nv_bfloat162* b1 = reinterpret_cast<const __nv_bfloat162*>(&u1);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(b0[e]);
        k[2 * e] = f.x;
        k[2 * e + 1] = f.y;
        const float2 g = __bfloat1622float2(b1[e]);
        k[8 + 2 * e] = g.x;
        k[8 + 2 * e + 1] = g.y;
    }
}

// 16-dim fmaf chain from 0 in dim order (the per-row kernel's lane slice)
SGB_DEV float chain16(const float* q, const float* k) {
    float a = 0.f;
#pragma unroll
    for (int e = 0; e < 16; ++e) a = fmaf(q[e], k[e], a);
    return a;
}

template <int DH, int KPC>
struct GLayout {
    static constexpr int KS = DH + 8;   // bf16 elements per staged key row (16 B pad: conflict-free)
    static constexpr int QS = DH + 4;   // floats per staged query row
    static constexpr int PS = kGB + 1;  // floats per score / probability row
    static constexpr int NC = kGB / KPC;
    static constexpr size_t k_off = 0;
    static constexpr size_t v_off = k_off + sizeof(__nv_bfloat16) * kGB * KS;
    static constexpr size_t q_off = v_off + sizeof(__nv_bfloat16) * kGB * KS;
    static constexpr size_t p_off = q_off + sizeof(float) * kGR * QS;
    static constexpr size_t a_off = p_off + sizeof(float) * (kGR * PS + 8 * NC);
    static constexpr size_t lv_off = a_off + sizeof(float) * kGR * NC;
    static constexpr size_t misc_off = lv_off + sizeof(int) * kGR;
    static constexpr size_t bytes = misc_off + 16;
};

template <int DH, int KPC, int RI>
SGB_DEV void scores_shared(const float* Qs, const __nv_bfloat16* Ks, float* Ps, int R, int nsh, float scale) {
    using Lay = GLayout<DH, KPC>;
    constexpr int NP = DH / 16;
    const int rq = threadIdx.x >> 4, kq = threadIdx.x & 15;
    if (kq >= nsh) return;
    for (int pass = 0; pass * 16 * RI < R; ++pass) {
        const int rbase = pass * 16 * RI + rq;
        if (rbase >= R) return;
        int rr[RI], kk[4];
#pragma unroll
        for (int i = 0; i < RI; ++i) rr[i] = min(rbase + 16 * i, R - 1);
#pragma unroll
        for (int j = 0; j < 4; ++j) kk[j] = min(kq + 16 * j, nsh - 1);
        float T[RI][4], S[RI][4], X[RI][4], D[RI][4];
#pragma unroll
        for (int pi = 0; pi < NP; ++pi) {
            const int p = piece_at<NP>(pi);
            float qv[RI][16];
#pragma unroll
            for (int i = 0; i < RI; ++i) {
                const float4* qp = reinterpret_cast<const float4*>(Qs + rr[i] * Lay::QS + 16 * p);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float4 a = qp[t];
                    qv[i][4 * t] = a.x;
                    qv[i][4 * t + 1] = a.y;
                    qv[i][4 * t + 2] = a.z;
                    qv[i][4 * t + 3] = a.w;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4* kp = reinterpret_cast<const uint4*>(Ks + kk[j] * Lay::KS + 16 * p);
                float kf[16];
                bf16x16_to_f32(kp[0], kp[1], kf);
#pragma unroll
                for (int i = 0; i < RI; ++i) tree_fold<NP>(pi, chain16(qv[i], kf), T[i][j], S[i][j], X[i][j], D[i][j]);
            }
        }
#pragma unroll
        for (int i = 0; i < RI; ++i) {
            const int r = rbase + 16 * i;
            if (r >= R) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = kq + 16 * j;
                if (k < nsh) Ps[r * Lay::PS + k] = attn_scale(D[i][j], scale);
            }
        }
    }
}

template <int DH, int KPC>
__global__ void __launch_bounds__(kGT, 2)
    attn_group_kernel(const float* __restrict__ q, const __nv_bfloat16* __restrict__ K,
                      const __nv_bfloat16* __restrict__ V, AttnRowsDev rows, const AttnTileDev* __restrict__ tiles,
                      int n_tiles, int H, int d, int nb_max, float scale, float* __restrict__ part_acc,
                      float* __restrict__ part_ml, int* __restrict__ tile_ctr, __nv_bfloat16* __restrict__ out) {
    using Lay = GLayout<DH, KPC>;
    constexpr int NP = DH / 16;
    constexpr int DPT = DH / 16;  // P.V dims per thread
    extern __shared__ __align__(128) uint8_t smem[];
    __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smem + Lay::k_off);
    __nv_bfloat16* Vs = reinterpret_cast<__nv_bfloat16*>(smem + Lay::v_off);
    float* Qs = reinterpret_cast<float*>(smem + Lay::q_off);
    float* Ps = reinterpret_cast<float*>(smem + Lay::p_off);
    float* Al = reinterpret_cast<float*>(smem + Lay::a_off);
    int* lv = reinterpret_cast<int*>(smem + Lay::lv_off);
    int* misc = reinterpret_cast<int*>(smem + Lay::misc_off);
    const int tid = threadIdx.x;

    pdl_wait();
    pdl_trigger();
    // ---- which tile: the one whose item range holds blockIdx.x (tiles sorted by item0)
    const int item = blockIdx.x;
    for (int t = tid; t < n_tiles; t += kGT) {
        const int lo = tiles[t].item0;
        const int hi = t + 1 < n_tiles ? tiles[t + 1].item0 : 0x7fffffff;
        if (lo <= item && item < hi) misc[0] = t;
    }
    __syncthreads();
    const int t = misc[0];
    const AttnTileDev tile = tiles[t];
    const int local = item - tile.item0;
    const int h = local % H, b = local / H;
    const int R = tile.nrows, r0 = tile.row0;
    const int ctx_len = rows.ctx_len[r0];
    const long long ctx_base = rows.ctx_base[r0];
    const int pre_len = rows.pre_len ? rows.pre_len[r0] : 0;
    const long long pre_base = rows.pre_len ? rows.pre_base[r0] : 0;
    const int kb = b * kGB;
    const int nsh = max(0, min(kGB, ctx_len - kb));
    const size_t col = static_cast<size_t>(h) * DH;

    // ---- stage the block's committed K/V (shared by the tile) and the tile's queries
    constexpr int CPR = DH / 8;  // 16-byte pieces per key row
    for (int u = tid; u < nsh * CPR; u += kGT) {
        const int key = u / CPR, c = u % CPR;
        const int v = kb + key;
        const long long slot = v < pre_len ? pre_base + v : ctx_base + v;
        const size_t src = static_cast<size_t>(slot) * d + col + 8 * c;
        cp_async16(Ks + key * Lay::KS + 8 * c, K + src);
        cp_async16(Vs + key * Lay::KS + 8 * c, V + src);
    }
    constexpr int QPR = DH / 4;
    for (int u = tid; u < R * QPR; u += kGT) {
        const int r = u / QPR, c = u % QPR;
        cp_async16(Qs + r * Lay::QS + 4 * c, q + static_cast<size_t>(r0 + r) * d + col + 4 * c);
    }
    if (tid < R) lv[tid] = ctx_len + rows.chain_len[r0 + tid];
    cp_async_wait_all();
    __syncthreads();

    // ---- scores over the shared keys
    if (nsh > 0) {
        if (R <= 16) scores_shared<DH, KPC, 1>(Qs, Ks, Ps, R, nsh, scale);
        else scores_shared<DH, KPC, 2>(Qs, Ks, Ps, R, nsh, scale);
    }
    // ---- scores over each row's own chain keys in this block (global / L2)
    if (kb + kGB > ctx_len) {
        for (int u = tid; u < R * kMaxChain; u += kGT) {
            const int r = u / kMaxChain, c = u % kMaxChain;
            const int v = ctx_len + c;
            if (v < kb || v >= kb + kGB || v >= lv[r]) continue;
            const long long slot = rows.chain_slots[static_cast<size_t>(r0 + r) * kMaxChain + c];
            const __nv_bfloat16* kr = K + static_cast<size_t>(slot) * d + col;
            const float* qr = Qs + r * Lay::QS;
            float T = 0.f, S = 0.f, X = 0.f, D = 0.f;
#pragma unroll
            for (int pi = 0; pi < NP; ++pi) {
                const int p = piece_at<NP>(pi);
                const uint4* kp = reinterpret_cast<const uint4*>(kr + 16 * p);
                float kf[16];
                bf16x16_to_f32(__ldg(kp), __ldg(kp + 1), kf);
                tree_fold<NP>(pi, chain16(qr + 16 * p, kf), T, S, X, D);
            }
            Ps[r * Lay::PS + (v - kb)] = attn_scale(D, scale);
        }
    }
    __syncthreads();

    // ---- chunked online softmax, one warp per row. The running max after chunk c is the
    // prefix max over chunks <= c (max is exact, so a lane scan gives the per-row kernel's
    // value); exps are independent given it; each chunk's sum is the same xor tree over its
    // KPC lanes; only l's fma chain over chunks is sequential.
    {
        const int warp = tid >> 5, lane = tid & 31;
        float* Lsum = Ps + kGR * Lay::PS;  // scratch after the score rows: [8 warps][NC]
        for (int r = warp; r < R; r += kGT / 32) {
            const int nk = min(lv[r], kb + kGB) - kb;
            if (nk <= 0) continue;  // warp-uniform
            float* pr = Ps + r * Lay::PS;
            float sv[2], pm[2], pv[2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int j = lane + 32 * hf;
                sv[hf] = j < nk ? pr[j] : -INFINITY;
                float cm = sv[hf];
#pragma unroll
                for (int o = 1; o < KPC; o <<= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
                pm[hf] = cm;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float y = __shfl_up_sync(0xffffffffu, pm[hf], o);
                    if (lane >= o) pm[hf] = fmaxf(pm[hf], y);
                }
            }
            const float half_max = __shfl_sync(0xffffffffu, pm[0], 31);
            pm[1] = fmaxf(pm[1], half_max);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int j = lane + 32 * hf;
                const int c = j / KPC;
                // running max before this chunk: the prefix max at the previous chunk's last key
                const int src = (c * KPC - 1) & 31;
                const float prev0 = __shfl_sync(0xffffffffu, pm[0], src);
                const float prev1 = __shfl_sync(0xffffffffu, pm[1], src);
                const float mprev = c == 0 ? -INFINITY : (c * KPC - 1 < 32 ? prev0 : prev1);
                pv[hf] = j < nk ? attn_p(sv[hf], pm[hf]) : 0.f;
                float ps = pv[hf];
#pragma unroll
                for (int o = KPC / 2; o > 0; o >>= 1) ps = __fadd_rn(ps, __shfl_xor_sync(0xffffffffu, ps, o));
                if (j < nk) pr[j] = pv[hf];
                if ((j % KPC) == 0 && j < nk) {
                    Al[r * Lay::NC + c] = attn_alpha(mprev, pm[hf]);
                    Lsum[warp * Lay::NC + c] = ps;
                }
            }
            __syncwarp();
            if (lane == 0) {
                float l = 0.f;
                const int nc = (nk + KPC - 1) / KPC;
                for (int c = 0; c < nc; ++c) l = attn_l(l, Al[r * Lay::NC + c], Lsum[warp * Lay::NC + c]);
                const size_t pidx = (static_cast<size_t>(r0 + r) * nb_max + b) * H + h;
                part_ml[2 * pidx + 1] = l;
            }
            // final running max = prefix max at the last valid key
            const int lastj = nk - 1;
            const float mfin = __shfl_sync(0xffffffffu, lastj < 32 ? pm[0] : pm[1], lastj & 31);
            if (lane == 0) {
                const size_t pidx = (static_cast<size_t>(r0 + r) * nb_max + b) * H + h;
                part_ml[2 * pidx] = mfin;
            }
            __syncwarp();
        }
    }
    __syncthreads();

    // ---- P.V: rows rg + 16 i, dims ds*DPT .. +DPT
    {
        const int rg = tid >> 4, ds = tid & 15;
        for (int pass = 0; pass * 64 < R; ++pass) {
            int rr[4], nk[4];
            int nkmax = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                rr[i] = pass * 64 + rg + 16 * i;
                nk[i] = rr[i] < R ? max(0, min(lv[rr[i]], kb + kGB) - kb) : 0;
                nkmax = max(nkmax, nk[i]);
            }
            if (nkmax == 0) break;
            float acc[4][DPT];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int e = 0; e < DPT; ++e) acc[i][e] = 0.f;
            for (int c = 0; c * KPC < nkmax; ++c) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (c * KPC < nk[i]) {
                        const float al = Al[rr[i] * Lay::NC + c];
#pragma unroll
                        for (int e = 0; e < DPT; ++e) acc[i][e] = __fmul_rn(acc[i][e], al);
                    }
#pragma unroll
                for (int j = 0; j < KPC; ++j) {
                    const int v = c * KPC + j;
                    if (v >= nkmax) break;
                    if (v < nsh) {
                        float vf[DPT];
                        const __nv_bfloat16* vp = Vs + v * Lay::KS + ds * DPT;
                        if constexpr (DPT == 8) {
                            const uint4 u = *reinterpret_cast<const uint4*>(vp);
                            const __nv_bfloat162* bb = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const float2 f = __bfloat1622float2(bb[e]);
                                vf[2 * e] = f.x;
                                vf[2 * e + 1] = f.y;
                            }
                        } else {
                            const uint2 u = *reinterpret_cast<const uint2*>(vp);
                            const __nv_bfloat162* bb = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                            for (int e = 0; e < DPT / 2; ++e) {
                                const float2 f = __bfloat1622float2(bb[e]);
                                vf[2 * e] = f.x;
                                vf[2 * e + 1] = f.y;
                            }
                        }
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (v < nk[i]) {
                                const float pj = Ps[rr[i] * Lay::PS + v];
#pragma unroll
                                for (int e = 0; e < DPT; ++e) acc[i][e] = fmaf(pj, vf[e], acc[i][e]);
                            }
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (v < nk[i]) {
                                const long long slot =
                                    rows.chain_slots[static_cast<size_t>(r0 + rr[i]) * kMaxChain + (kb + v - ctx_len)];
                                const __nv_bfloat16* vp = V + static_cast<size_t>(slot) * d + col + ds * DPT;
                                float vf[DPT];
#pragma unroll
                                for (int e = 0; e < DPT; e += 2) {
                                    const float2 f =
                                        __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vp + e));
                                    vf[e] = f.x;
                                    vf[e + 1] = f.y;
                                }
                                const float pj = Ps[rr[i] * Lay::PS + v];
#pragma unroll
                                for (int e = 0; e < DPT; ++e) acc[i][e] = fmaf(pj, vf[e], acc[i][e]);
                            }
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (nk[i] > 0) {
                    const size_t pidx = (static_cast<size_t>(r0 + rr[i]) * nb_max + b) * H + h;
                    float* pa = part_acc + pidx * DH + ds * DPT;
#pragma unroll
                    for (int e = 0; e < DPT; ++e) pa[e] = acc[i][e];
                }
        }
    }

    // ---- ticket on (tile, head): the last block merges every row of the tile in block order
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        int* c = tile_ctr + static_cast<size_t>(t) * H + h;
        const int old = atomicAdd(c, 1);
        const int last = old + 1 == tile.nb;
        if (last) *c = 0;  // re-armed for the next launch
        misc[1] = last;
    }
    __syncthreads();
    if (!misc[1]) return;
    __threadfence();
    {
        const int rg = tid >> 4, ds = tid & 15;
        for (int r = rg; r < R; r += 16) {
            const int nbr = (lv[r] + kGB - 1) / kGB;
            float Mx = -INFINITY, Lx = 0.f, A[DPT];
#pragma unroll
            for (int e = 0; e < DPT; ++e) A[e] = 0.f;
            for (int bb = 0; bb < nbr; ++bb) {
                const size_t pidx = (static_cast<size_t>(r0 + r) * nb_max + bb) * H + h;
                const float mb = __ldcg(part_ml + 2 * pidx), lb = __ldcg(part_ml + 2 * pidx + 1);
                float ab[DPT];
#pragma unroll
                for (int e = 0; e < DPT; ++e) ab[e] = __ldcg(part_acc + pidx * DH + ds * DPT + e);
                attn_merge<DPT>(Mx, Lx, A, mb, lb, ab);
            }
            __nv_bfloat16* o = out + static_cast<size_t>(r0 + r) * d + col + ds * DPT;
#pragma unroll
            for (int e = 0; e < DPT; ++e) o[e] = __float2bfloat16(__fdiv_rn(A[e], Lx));
        }
    }
}

template <int DH, int KPC>
void launch_group_impl(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows,
                       const AttnTileDev* tiles, int n_tiles, int n_items, int H, int d, int nb_max,
                       const AttnScratch& sc, __nv_bfloat16* out, cudaStream_t st) {
    using Lay = GLayout<DH, KPC>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_group_kernel<DH, KPC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(Lay::bytes));
        attr = true;
    }
    launch_pdl(attn_group_kernel<DH, KPC>, dim3(static_cast<unsigned>(n_items)), dim3(kGT), Lay::bytes, st, q, K, V,
               rows, tiles, n_tiles, H, d, nb_max, 1.0f / sqrtf(static_cast<float>(DH)), sc.part_acc, sc.part_ml,
               sc.row_ctr, out);
}

}  // namespace

void launch_attention_group(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows,
                            const AttnTileDev* tiles, int n_tiles, int n_items, int H, int d, int max_virtual_len,
                            const AttnScratch& sc, __nv_bfloat16* out, cudaStream_t st) {
    if (n_tiles <= 0 || n_items <= 0) return;
    const int dh = d / H;
    const int nb = attn_splits_for(max_virtual_len);
    if (static_cast<long long>(n_tiles) * H > sc.ctr_cap) throw std::invalid_argument("attention: tile tickets too small");
    const int kpc = d <= 3328 ? 8 : 4;  // same chunking as the per-row kernel (numerics)
    if (dh == 128 && kpc == 8) launch_group_impl<128, 8>(q, K, V, rows, tiles, n_tiles, n_items, H, d, nb, sc, out, st);
    else if (dh == 128 && kpc == 4) launch_group_impl<128, 4>(q, K, V, rows, tiles, n_tiles, n_items, H, d, nb, sc, out, st);
    else if (dh == 64 && kpc == 8) launch_group_impl<64, 8>(q, K, V, rows, tiles, n_tiles, n_items, H, d, nb, sc, out, st);
    else throw std::invalid_argument("attention: head dim must be 64 or 128");
    SGB_KCHECK();
}

}  // namespace sgb
