// Online draft learning on the device: teacher-forced draft forward with saved
// activations, SmoothL1 + chunked LM-head cross-entropy, hand-written backward, AdamW.
//
// Reference (include/sgrpo/...):
//   grpo.hpp:278-344     draft_loss_grad (rows = pairs (t_j, f_{j-1}), j = 1..n-2)
//   tinylm.hpp:881-953   draft_train_forward / draft_train_backward
//   tinylm.hpp:653-800   train_blocks_fwd / train_blocks_bwd (causal attention, LN, GELU)
//   nn.hpp:100-125       layernorm_bwd;  nn.hpp:135-144 gelu_grad
//   grpo.cpp:142-161     AdamW::step (m, v fp32; math in fp64; decoupled weight decay)
// The projection GEMMs (forward, dgrad, wgrad) run on the tcgen05 GEMM (gemm.cu); the
// kernels here are the row-wise and attention pieces. Every reduction has a fixed order
// (per-row sequential / fixed block partials), so an update is deterministic.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "train.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kT = 256;

__device__ float block_sum_f(float v, float* red) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float s = 0.f;
    for (int i = 0; i < kT / 32; ++i) s += red[i];
    return s;
}

__device__ double block_sum_dd(double v, double* red) {
    v = warp_sum_d(v);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < kT / 32; ++i) s += red[i];
    return s;
}

// LayerNorm forward saving (mu, rstd) (nn.hpp:70-98 with LnCache).
__global__ void __launch_bounds__(kT) ln_fwd_stats_kernel(const float* __restrict__ x, int d, const float* __restrict__ g,
                                                          const float* __restrict__ b, __nv_bfloat16* __restrict__ a,
                                                          float* __restrict__ y, float* __restrict__ mu_out,
                                                          float* __restrict__ rs_out) {
    __shared__ float red[kT / 32];
    const int r = blockIdx.x;
    const float* xr = x + static_cast<size_t>(r) * d;
    float s = 0.f;
    for (int e = threadIdx.x; e < d; e += kT) s += xr[e];
    const float mu = block_sum_f(s, red) / d;
    float v = 0.f;
    for (int e = threadIdx.x; e < d; e += kT) {
        const float t = xr[e] - mu;
        v += t * t;
    }
    const float rs = 1.0f / sqrtf(block_sum_f(v, red) / d + 1e-5f);
    for (int e = threadIdx.x; e < d; e += kT) {
        const float o = g[e] * (xr[e] - mu) * rs + b[e];
        if (a) a[static_cast<size_t>(r) * d + e] = __float2bfloat16(o);
        if (y) y[static_cast<size_t>(r) * d + e] = o;
    }
    if (threadIdx.x == 0) {
        mu_out[r] = mu;
        rs_out[r] = rs;
    }
}

// LayerNorm backward (nn.hpp:100-125): dx = (dn - mean(dn) - xhat*mean(dn*xhat)) * rstd (+ resid);
// per-row contributions to dgamma/dbeta go to a [rows][2d] scratch reduced later in order.
__global__ void __launch_bounds__(kT) ln_bwd_kernel(const float* __restrict__ x, const float* __restrict__ g,
                                                    const float* __restrict__ mu, const float* __restrict__ rs,
                                                    const float* __restrict__ dy, const float* __restrict__ resid,
                                                    int d, float* __restrict__ dx, float* __restrict__ dgb_rows) {
    __shared__ float red[kT / 32];
    const int r = blockIdx.x;
    const size_t o = static_cast<size_t>(r) * d;
    const float m = mu[r], s = rs[r];
    float s1 = 0.f, s2 = 0.f;
    for (int e = threadIdx.x; e < d; e += kT) {
        const float xh = (x[o + e] - m) * s;
        const float dn = dy[o + e] * g[e];
        s1 += dn;
        s2 += dn * xh;
    }
    s1 = block_sum_f(s1, red);
    s2 = block_sum_f(s2, red);
    for (int e = threadIdx.x; e < d; e += kT) {
        const float xh = (x[o + e] - m) * s;
        const float dn = dy[o + e] * g[e];
        float v = (dn - s1 / d - xh * s2 / d) * s;
        if (resid) v += resid[o + e];
        dx[o + e] = v;
        dgb_rows[2 * o + e] = dy[o + e] * xh;
        dgb_rows[2 * o + d + e] = dy[o + e];
    }
}

// Column sums of a [rows][cols] fp32 matrix in fixed row order, added into out[cols].
__global__ void colsum_add_kernel(const float* __restrict__ m, int rows, int cols, float* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= cols) return;
    float s = 0.f;
    for (int r = 0; r < rows; ++r) s += m[static_cast<size_t>(r) * cols + c];
    out[c] += s;
}

__device__ __forceinline__ float gelu_f(float x) {
    const float c = 0.7978845608028654f;
    return 0.5f * x * (1.0f + tanhf(c * (x + 0.044715f * x * x * x)));
}
__device__ __forceinline__ float gelu_grad_f(float x) {  // nn.hpp:135-144
    const float c = 0.7978845608028654f;
    const float x3 = x * x * x;
    const float th = tanhf(c * (x + 0.044715f * x3));
    return 0.5f * (1.0f + th) + 0.5f * x * (1.0f - th * th) * c * (1.0f + 3.0f * 0.044715f * x * x);
}

__global__ void gelu_fwd_kernel(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ y) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        y[i] = __float2bfloat16(gelu_f(x[i]));
}

__global__ void gelu_bwd_kernel(const float* __restrict__ x, const float* __restrict__ dy, size_t n,
                                __nv_bfloat16* __restrict__ dx) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dx[i] = __float2bfloat16(dy[i] * gelu_grad_f(x[i]));
}

// Causal attention over each sequence's own rows (tinylm.hpp:673-700), fp32, one CTA per

// SmoothL1(beta=1) vs the target feature (grpo.hpp:311-322): dfeat and the per-row loss.
__global__ void __launch_bounds__(kT) smoothl1_kernel(const float* __restrict__ fhat, const float* __restrict__ feat_base,
                                                      const long long* __restrict__ tgt_off, int d, double scale,
                                                      float* __restrict__ dfeat, double* __restrict__ loss_row) {
    __shared__ double red[kT / 32];
    const int r = blockIdx.x;
    const float* f = feat_base + tgt_off[r];
    double acc = 0.0;
    for (int e = threadIdx.x; e < d; e += kT) {
        const double err = static_cast<double>(fhat[static_cast<size_t>(r) * d + e]) - static_cast<double>(f[e]);
        const double ae = fabs(err);
        double g;
        if (ae <= 1.0) {
            acc += scale * 0.5 * err * err;
            g = scale * err;
        } else {
            acc += scale * (ae - 0.5);
            g = err > 0 ? scale : -scale;
        }
        dfeat[static_cast<size_t>(r) * d + e] = static_cast<float>(g);
    }
    acc = block_sum_dd(acc, red);
    if (threadIdx.x == 0) loss_row[r] = acc;
}

// Cross entropy vs the next token through the frozen LM head (grpo.hpp:323-338):
// loss row and dlogits = scale * (softmax - onehot) in bf16.
__global__ void __launch_bounds__(kT) ce_kernel(const float* __restrict__ logits, int V, const int* __restrict__ tgt,
                                                double scale, const double* __restrict__ row_scale,
                                                __nv_bfloat16* __restrict__ dlog, double* __restrict__ loss_row) {
    // Two passes over the 608 KB row: (1) online max + sum of exp with per-thread rescaling
    // (fp32 exps, fp64 sums), (2) the bf16 gradient scale * (softmax - onehot). The gradient
    // is stored in bf16, so its exps are fp32; the loss keeps an fp64 log-sum-exp.
    __shared__ double redd[kT / 32];
    __shared__ float redf[kT / 32];
    const int r = blockIdx.x;
    const float* L = logits + static_cast<size_t>(r) * V;
    float mt = -INFINITY;
    double st = 0.0;
    const bool vec = (V & 3) == 0;
    auto see = [&](float x) {
        if (x > mt) {
            st = st * static_cast<double>(expf(mt - x)) + 1.0;
            mt = x;
        } else {
            st += static_cast<double>(expf(x - mt));
        }
    };
    if (vec) {
        const float4* L4 = reinterpret_cast<const float4*>(L);
        for (int c = threadIdx.x; c < V / 4; c += kT) {
            const float4 x = L4[c];
            see(x.x);
            see(x.y);
            see(x.z);
            see(x.w);
        }
    } else {
        for (int c = threadIdx.x; c < V; c += kT) see(L[c]);
    }
    // block max, then rescale every thread's sum to it
    float mx = warp_max(mt);
    if ((threadIdx.x & 31) == 0) redf[threadIdx.x >> 5] = mx;
    __syncthreads();
    float m2 = redf[0];
    for (int i = 1; i < kT / 32; ++i) m2 = fmaxf(m2, redf[i]);
    const double s = block_sum_dd(mt == -INFINITY ? 0.0 : st * static_cast<double>(expf(mt - m2)), redd);
    const double lse = static_cast<double>(m2) + log(s);
    const float lse_f = static_cast<float>(lse);
    if (row_scale) scale = row_scale[r];  // policy loss: advantage / N on response rows, 0 on prompt rows
    const float sc = static_cast<float>(scale);
    const int t = tgt[r];
    __nv_bfloat16* D = dlog + static_cast<size_t>(r) * V;
    if (vec) {
        const float4* L4 = reinterpret_cast<const float4*>(L);
        for (int c = threadIdx.x; c < V / 4; c += kT) {
            const float4 x = L4[c];
            float g0 = sc * expf(x.x - lse_f), g1 = sc * expf(x.y - lse_f), g2 = sc * expf(x.z - lse_f),
                  g3 = sc * expf(x.w - lse_f);
            const int c0 = 4 * c;
            if (t == c0) g0 -= sc;
            if (t == c0 + 1) g1 -= sc;
            if (t == c0 + 2) g2 -= sc;
            if (t == c0 + 3) g3 -= sc;
            __nv_bfloat162 a = __floats2bfloat162_rn(g0, g1), b = __floats2bfloat162_rn(g2, g3);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t*>(&a);
            u.y = *reinterpret_cast<uint32_t*>(&b);
            *reinterpret_cast<uint2*>(D + c0) = u;
        }
    } else {
        for (int c = threadIdx.x; c < V; c += kT) {
            float g = sc * expf(L[c] - lse_f);
            if (c == t) g -= sc;
            D[c] = __float2bfloat16(g);
        }
    }
    if (threadIdx.x == 0) loss_row[r] = -scale * (static_cast<double>(L[t]) - lse);
}

// [rows][cols] (fp32 or bf16) -> [cols][ld] bf16 transposed (zero-padded columns).
template <class Tin>
__global__ void transpose_bf16_kernel(const Tin* __restrict__ src, int rows, int cols, int src_ld,
                                      __nv_bfloat16* __restrict__ dst, int ld) {
    __shared__ float tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int r = r0 + k, c = c0 + threadIdx.x;
        float v = 0.f;
        if (r < rows && c < cols) {
            if constexpr (sizeof(Tin) == 4) v = src[static_cast<size_t>(r) * src_ld + c];
            else v = __bfloat162float(src[static_cast<size_t>(r) * src_ld + c]);
        }
        tile[k][threadIdx.x] = v;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int c = c0 + k, r = r0 + threadIdx.x;
        if (c < cols && r < ld) dst[static_cast<size_t>(c) * ld + r] = __float2bfloat16(r < rows ? tile[threadIdx.x][k] : 0.f);
    }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ x, size_t n, __nv_bfloat16* __restrict__ y) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        y[i] = __float2bfloat16(x[i]);
}

// AdamW (grpo.cpp:142-161): m, v stored fp32, arithmetic in fp64.
__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, size_t n, double lr, double b1, double b2, double eps, double wd,
                             double bc1, double bc2) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const double gi = g[i];
        const float mi = static_cast<float>(b1 * m[i] + (1.0 - b1) * gi);
        const float vi = static_cast<float>(b2 * v[i] + (1.0 - b2) * gi * gi);
        m[i] = mi;
        v[i] = vi;
        const double mh = mi / bc1, vh = vi / bc2;
        const double pi = p[i];
        p[i] = static_cast<float>(pi - lr * (mh / (sqrt(vh) + eps) + wd * pi));
    }
}

// x0[r] = tok_emb[tok[r]] + pos_emb[pos[r]] (target_train_forward, tinylm.hpp:813-819)
__global__ void embed_sum_kernel(const int* __restrict__ tok, const int* __restrict__ pos, int d,
                                 const float* __restrict__ te, const float* __restrict__ pe, float* __restrict__ x) {
    const int r = blockIdx.x;
    const float* a = te + static_cast<size_t>(tok[r]) * d;
    const float* b = pe + static_cast<size_t>(pos[r]) * d;
    float* o = x + static_cast<size_t>(r) * d;
    for (int e = threadIdx.x; e < d; e += blockDim.x) o[e] = a[e] + b[e];
}

// embedding gradients (tinylm.hpp:857-865), deterministic: one CTA per distinct embedding row,
// which adds the dx rows that hit it (CSR, ascending row order) -- grad[key[k]] += sum dx[rows]
__global__ void embed_grad_kernel(const int* __restrict__ key, const int* __restrict__ ptr,
                                  const int* __restrict__ rows, int d, const float* __restrict__ dx,
                                  float* __restrict__ grad) {
    const int k = blockIdx.x;
    float* o = grad + static_cast<size_t>(key[k]) * d;
    const int j0 = ptr[k], j1 = ptr[k + 1];
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
        float acc = o[e];
        for (int j = j0; j < j1; ++j) acc += dx[static_cast<size_t>(rows[j]) * d + e];
        o[e] = acc;
    }
}

int grid_n(size_t n) {
    size_t b = (n + 255) / 256;
    if (b > 148 * 32) b = 148 * 32;
    return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

void launch_ln_fwd_stats(const float* x, int R, int d, const float* g, const float* b, __nv_bfloat16* a, float* y,
                         float* mu, float* rs, cudaStream_t st) {
    if (R <= 0) return;
    ln_fwd_stats_kernel<<<R, kT, 0, st>>>(x, d, g, b, a, y, mu, rs);
    SGB_KCHECK();
}
void launch_ln_bwd(const float* x, const float* g, const float* mu, const float* rs, const float* dy,
                   const float* resid, int R, int d, float* dx, float* dgb_rows, cudaStream_t st) {
    if (R <= 0) return;
    ln_bwd_kernel<<<R, kT, 0, st>>>(x, g, mu, rs, dy, resid, d, dx, dgb_rows);
    SGB_KCHECK();
}
void launch_colsum_add(const float* m, int rows, int cols, float* out, cudaStream_t st) {
    if (rows <= 0) return;
    colsum_add_kernel<<<(cols + 127) / 128, 128, 0, st>>>(m, rows, cols, out);
    SGB_KCHECK();
}
void launch_gelu_fwd(const float* x, size_t n, __nv_bfloat16* y, cudaStream_t st) {
    gelu_fwd_kernel<<<grid_n(n), 256, 0, st>>>(x, n, y);
    SGB_KCHECK();
}
void launch_gelu_bwd(const float* x, const float* dy, size_t n, __nv_bfloat16* dx, cudaStream_t st) {
    gelu_bwd_kernel<<<grid_n(n), 256, 0, st>>>(x, dy, n, dx);
    SGB_KCHECK();
}
void launch_smoothl1(const float* fhat, const float* feat_base, const long long* tgt_off, int R, int d, double scale,
                     float* dfeat, double* loss_row, cudaStream_t st) {
    if (R <= 0) return;
    smoothl1_kernel<<<R, kT, 0, st>>>(fhat, feat_base, tgt_off, d, scale, dfeat, loss_row);
    SGB_KCHECK();
}
void launch_ce(const float* logits, int R, int V, const int* tgt, double scale, __nv_bfloat16* dlog, double* loss_row,
               cudaStream_t st, const double* row_scale) {
    if (R <= 0) return;
    ce_kernel<<<R, kT, 0, st>>>(logits, V, tgt, scale, row_scale, dlog, loss_row);
    SGB_KCHECK();
}
void launch_transpose_bf16(const float* src, int rows, int cols, int src_ld, __nv_bfloat16* dst, int ld,
                           cudaStream_t st) {
    dim3 grid((cols + 31) / 32, (ld + 31) / 32);
    transpose_bf16_kernel<float><<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, src_ld, dst, ld);
    SGB_KCHECK();
}
void launch_transpose_bf16(const __nv_bfloat16* src, int rows, int cols, int src_ld, __nv_bfloat16* dst, int ld,
                           cudaStream_t st) {
    dim3 grid((cols + 31) / 32, (ld + 31) / 32);
    transpose_bf16_kernel<__nv_bfloat16><<<grid, dim3(32, 8), 0, st>>>(src, rows, cols, src_ld, dst, ld);
    SGB_KCHECK();
}
void launch_f32_to_bf16(const float* x, size_t n, __nv_bfloat16* y, cudaStream_t st) {
    f32_to_bf16_kernel<<<grid_n(n), 256, 0, st>>>(x, n, y);
    SGB_KCHECK();
}
void launch_adamw(float* p, const float* g, float* m, float* v, size_t n, double lr, double b1, double b2, double eps,
                  double wd, long long t, cudaStream_t st) {
    const double bc1 = 1.0 - pow(b1, static_cast<double>(t));
    const double bc2 = 1.0 - pow(b2, static_cast<double>(t));
    adamw_kernel<<<grid_n(n), 256, 0, st>>>(p, g, m, v, n, lr, b1, b2, eps, wd, bc1, bc2);
    SGB_KCHECK();
}

void launch_embed_sum(const int* tok, const int* pos, int R, int d, const float* te, const float* pe, float* x,
                      cudaStream_t st) {
    if (R <= 0) return;
    embed_sum_kernel<<<R, 256, 0, st>>>(tok, pos, d, te, pe, x);
    SGB_KCHECK();
}
void launch_embed_grad(const int* key, const int* ptr, const int* rows, int n_keys, int d, const float* dx,
                       float* grad, cudaStream_t st) {
    if (n_keys <= 0) return;
    embed_grad_kernel<<<n_keys, 256, 0, st>>>(key, ptr, rows, d, dx, grad);
    SGB_KCHECK();
}

}  // namespace sgb
