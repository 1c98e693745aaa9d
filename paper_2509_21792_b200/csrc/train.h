// Launchers of the online draft-learning kernels (train.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>

namespace sgb {

void launch_ln_fwd_stats(const float* x, int R, int d, const float* g, const float* b, __nv_bfloat16* a, float* y,
                         float* mu, float* rs, cudaStream_t st);
void launch_ln_bwd(const float* x, const float* g, const float* mu, const float* rs, const float* dy,
                   const float* resid, int R, int d, float* dx, float* dgb_rows, cudaStream_t st);
void launch_colsum_add(const float* m, int rows, int cols, float* out, cudaStream_t st);
void launch_gelu_fwd(const float* x, size_t n, __nv_bfloat16* y, cudaStream_t st);
void launch_gelu_bwd(const float* x, const float* dy, size_t n, __nv_bfloat16* dx, cudaStream_t st);
// Causal training attention on tensor cores (train_attn.cu): row i attends keys
// seq_first[i] .. i. Forward writes ctx (fp32 + bf16) and lse [R][H]; backward writes
// dq/dk/dv into dqkv [R][3d] and uses Drow [R][H] as scratch.
// tiles[n_tiles]: first row of every 64-row tile, tiles starting at seq_first + 64m.
void launch_train_attn_fwd(const float* qkv, const int* seq_first, const int* seq_last, const int* tiles, int n_tiles,
                           int d, int H, float* ctx, __nv_bfloat16* ctx_b, float* lse, cudaStream_t st);
void launch_train_attn_bwd(const float* qkv, const float* ctx, const float* dctx, const float* lse,
                           const int* seq_first, const int* seq_last, const int* tiles, int n_tiles, int R, int d,
                           int H, float* Drow, float* dqkv, cudaStream_t st);
void launch_smoothl1(const float* fhat, const float* feat_base, const long long* tgt_off, int R, int d, double scale,
                     float* dfeat, double* loss_row, cudaStream_t st);
// row_scale (optional, [R]) replaces scale per row
void launch_ce(const float* logits, int R, int V, const int* tgt, double scale, __nv_bfloat16* dlog, double* loss_row,
               cudaStream_t st, const double* row_scale = nullptr);
void launch_embed_sum(const int* tok, const int* pos, int R, int d, const float* te, const float* pe, float* x,
                      cudaStream_t st);
// grad[key[k]][:] += sum over rows[ptr[k] .. ptr[k+1]) of dx[row][:] (fixed order: deterministic)
void launch_embed_grad(const int* key, const int* ptr, const int* rows, int n_keys, int d, const float* dx,
                       float* grad, cudaStream_t st);
void launch_transpose_bf16(const float* src, int rows, int cols, int src_ld, __nv_bfloat16* dst, int ld,
                           cudaStream_t st);
void launch_transpose_bf16(const __nv_bfloat16* src, int rows, int cols, int src_ld, __nv_bfloat16* dst, int ld,
                           cudaStream_t st);
void launch_f32_to_bf16(const float* x, size_t n, __nv_bfloat16* y, cudaStream_t st);
void launch_adamw(float* p, const float* g, float* m, float* v, size_t n, double lr, double b1, double b2, double eps,
                  double wd, long long t, cudaStream_t st);

}  // namespace sgb
