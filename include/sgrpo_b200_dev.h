/*
 * sgrpo_b200_dev.h -- test-only entry points of libsgrpo_b200_dev.so: kernel self-tests on
 * host-supplied operands and microbenchmarks. Not part of the drop-in boundary
 * (include/sgrpo_b200.h); the tests and scripts/ load this library beside the product one.
 * Same status codes as sgrpo_b200.h; sgb_dev_last_error() returns this library's message.
 */
#ifndef SGRPO_B200_DEV_H
#define SGRPO_B200_DEV_H

#ifdef __cplusplus
extern "C" {
#endif

const char* sgb_dev_last_error(void);

/* GEMM microbenchmark (device-resident operands): average device ms per launch. */
int sgb_bench_gemm(int M, int N, int K, int splits, int iters, double* ms_out);

/* Decode-attention microbenchmark: B rows x (ctx + 1) keys, H heads of dh. */
int sgb_bench_attention(int B, int ctx, int H, int dh, int iters, double* ms_out);
/* Attention self-test: row r attends to n_keys[r] keys (rows concatenated in k/v
 * [sum n_keys][H*dh] fp32, converted to bf16); the last key of each row goes through the
 * tree-path slot list. out [B][H*dh] (bf16 values). */
int sgb_debug_attention(int B, const int* n_keys, int H, int dh, const float* q, const float* k, const float* v,
                        float* out);

/* sgb_group_advantages (sgrpo_b200.h) on host token tables ([n_groups*g][stride], lens / prompt_lens
 * per sequence). */
int sgb_debug_group_advantages(const int* tokens, const int* lens, const int* prompt_lens, int n_groups, int g,
                               int stride, const long long* answers, double eps_var, double* rewards,
                               double* advantages, int* valid);

/* Prefix-shared tree attention self-test. n_groups sequences; group g has ctx_len[g]
 * committed keys (kctx/vctx rows, concatenated over groups) and n_rows[g] tree rows in
 * level order with parent[r] (index within the group, -1 = root); row r attends to the
 * group's committed keys then its ancestors-or-self node keys (knode/vnode, one per row),
 * exactly the verify rows of a speculative step (build_tree_mask, drafttree.cpp:145-168;
 * decode_blocks, tinylm.hpp:335-395). The rows run through BOTH the per-row kernel
 * (out_row) and the prefix-shared group kernel (out_group); [rows][H*dh], bf16 values. */
int sgb_debug_tree_attention(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H, int dh,
                             const float* q, const float* kctx, const float* vctx, const float* knode,
                             const float* vnode, float* out_row, float* out_group);

/* The same self-test through attention_tree.cu (the engine's tree-verify / draft-level kernel:
 * one CTA per row tile and head over the whole key range); out_tree [rows][H*dh]. */
int sgb_debug_tree_attention_tree(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H, int dh,
                                  const float* q, const float* kctx, const float* vctx, const float* knode,
                                  const float* vnode, float* out_tree);
/* Tree-verify microbenchmark of attention_tree.cu (same shapes as sgb_bench_tree_attention). */
int sgb_bench_tree_attention_tree(int B, int N, int ctx, int H, int dh, int iters, double* ms_tree);
/* Cluster decode attention (AR steps, one row per group) next to attention.cu on the same
 * inputs (debug), and an AR attention microbenchmark: ms per launch of the three kernels. */
int sgb_debug_attention_decode(int n_groups, const int* ctx_len, int H, int dh, const float* q, const float* kctx,
                               const float* vctx, const float* knode, const float* vnode, float* out_row,
                               float* out_decode);
int sgb_bench_attention_decode(int B, int ctx, int H, int dh, int iters, double* ms_row, double* ms_tree,
                               double* ms_decode);

/* Two-lane concurrency microbenchmark: one layer's attention (B rows x (ctx + 1) keys) on
 * one stream and its four GEMMs (M rows, width H*dh, d_ff) on another, on persistent grids
 * capped at attn_cap / gemm_cap SMs (0 = all). out[3] = ms per iteration: attention alone,
 * GEMMs alone, both concurrently. */
int sgb_bench_overlap(int B, int ctx, int H, int dh, int dff, int M, int attn_cap, int gemm_cap, int iters,
                      double* out);

/* Tree-verify attention microbenchmark: B sequences x (ctx committed keys + an EAGLE-shaped
 * tree of N rows); ms per launch of the per-row and of the prefix-shared group kernel. */
int sgb_bench_tree_attention(int B, int N, int ctx, int H, int dh, int iters, double* ms_row, double* ms_group);

/* tcgen05 GEMM self-test: out[M][N] = bf16(x)[M][K] . bf16(w)[N][K]^T (K-major). */
int sgb_debug_gemm(const float* w, const float* x, int M, int N, int K, float* out, int* splits_out);

#ifdef __cplusplus
}
#endif

#endif /* SGRPO_B200_DEV_H */
