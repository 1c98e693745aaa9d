// Attention numerics shared by the per-row kernel (attention.cu) and the prefix-shared
// group kernel (attention_group.cu).
//
// Batch invariance requires a verify row and the later AR row of the same
// token to produce identical bits even when they run in different kernels. Both kernels
// therefore spell every rounding step out with explicit intrinsics (no contraction choices
// left to the compiler) and follow the same order:
//   score   = fl(fl(q . k) * scale), q . k summed as 16-dim fmaf chains per piece, pieces
//             combined in the butterfly tree ((a0+a4)+(a2+a6))+((a1+a5)+(a3+a7)) (dh=128)
//             or (a0+a2)+(a1+a3) (dh=64);
//   chunk   = KPC keys: m' = max(m, max s), alpha = m==-inf ? 0 : exp(m-m'),
//             p_j = exp(s_j - m'), l = fma(l, alpha, tree-sum(p)), acc = acc*alpha then
//             acc = fma(p_j, v_j, acc) for j in key order;
//   merge   = 64-key block partials in block order from the identity (-inf, 0, 0).
// Reference semantics: softmax_row (include/sgrpo/nn.hpp:157-169) over the keys of
// decode_blocks (include/sgrpo/tinylm.hpp:335-395).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace sgb {

constexpr int kAttnBlock = 64;  // keys per softmax partial (part of the numerics)

SGB_DEV float attn_scale(float dot, float scale) { return __fmul_rn(dot, scale); }

// The per-chunk exponentials use the SFU (__expf: ex2.approx of x * log2 e, ~2 ulp): six per chunk
// sit on every consumer warp's dependent chain, and the latency-bound small-B kernels run that
// chain ~50 times per launch. Every inference attention kernel takes them from here, so their
// bits stay identical to each other (batch invariance); the block merges keep expf.
// exp(m_old - m_new), 0 for the fresh state
SGB_DEV float attn_alpha(float m_old, float m_new) { return m_old == -INFINITY ? 0.f : __expf(__fsub_rn(m_old, m_new)); }

SGB_DEV float attn_p(float s, float m_new) { return __expf(__fsub_rn(s, m_new)); }

SGB_DEV float attn_l(float l, float alpha, float psum) { return fmaf(l, alpha, psum); }

// fixed tree sum of one chunk's probabilities (what warp_sum yields with zeros beyond KPC)
template <int KPC>
SGB_DEV float attn_psum(const float* p) {
    if constexpr (KPC == 8) {
        return __fadd_rn(__fadd_rn(__fadd_rn(p[0], p[4]), __fadd_rn(p[2], p[6])),
                         __fadd_rn(__fadd_rn(p[1], p[5]), __fadd_rn(p[3], p[7])));
    } else {
        static_assert(KPC == 4, "KPC must be 4 or 8");
        return __fadd_rn(__fadd_rn(p[0], p[2]), __fadd_rn(p[1], p[3]));
    }
}

// one ordered merge step of a block partial (mb, lb, ab[]) into the running (Mx, Lx, A[])
template <int N>
SGB_DEV void attn_merge(float& Mx, float& Lx, float* A, float mb, float lb, const float* ab) {
    const float Mn = fmaxf(Mx, mb);
    const float ca = Mx == -INFINITY ? 0.f : expf(__fsub_rn(Mx, Mn));
    const float cb = expf(__fsub_rn(mb, Mn));
    Lx = fmaf(Lx, ca, __fmul_rn(lb, cb));
#pragma unroll
    for (int e = 0; e < N; ++e) A[e] = fmaf(A[e], ca, __fmul_rn(ab[e], cb));
    Mx = Mn;
}

}  // namespace sgb
