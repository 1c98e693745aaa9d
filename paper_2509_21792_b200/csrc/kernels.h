// Launchers of the sm_100a kernels (rowops.cu, attention.cu, sample.cu, tree.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <array>
#include <cstddef>
#include <vector>

namespace sgb {

constexpr int kMaxChain = 8;  // l_max + 1 (root + tree depth) per attention row

// Per-row attention metadata (see attention.cu).
struct AttnRowsDev {
    const long long* ctx_base;     // [M] global KV slot of virtual index 0
    const int* ctx_len;            // [M] contiguous prefix length
    const int* chain_len;          // [M] number of chain (tree-path) slots
    const long long* chain_slots;  // [M][kMaxChain] global KV slots, root-first
    // optional shared prompt: virtual index v < pre_len[r] reads slot pre_base[r] + v instead
    // of ctx_base[r] + v (the G members of a group read their prompt's K/V from one copy)
    const long long* pre_base = nullptr;
    const int* pre_len = nullptr;
};

// ---- rowops.cu
void launch_embed_ln(const int* tokens, const int* positions, int M, int d, const float* tok_emb, const float* pos_emb,
                     const float* g, const float* b, float* x, __nv_bfloat16* a, cudaStream_t st);
void launch_reduce_residual_ln(const float* P, int S, int M, int d, float* x, bool accumulate, const float* pos_emb,
                               const int* positions, const float* g, const float* b, __nv_bfloat16* a, float* y,
                               cudaStream_t st);
void launch_reduce_gelu(const float* P, int S, int M, int N, __nv_bfloat16* out, cudaStream_t st);
void launch_reduce_plain(const float* P, int S, int M, int N, float* out, cudaStream_t st);
void launch_reduce_qkv(const float* P, int S, int M, int d, float* q, __nv_bfloat16* kc, __nv_bfloat16* vc,
                       const long long* kv_dst, cudaStream_t st);
void launch_gather_fuse(const int* tokens, const long long* feat_off, const float* feat_base, const float* tok_emb,
                        int R, int d, __nv_bfloat16* out, cudaStream_t st);
void launch_transpose_to_bf16(const float* src, int in, int out_dim, __nv_bfloat16* dst, int dst_ld, cudaStream_t st);
void launch_gather_rows_bf16(const __nv_bfloat16* src, const int* idx, int R, int d, __nv_bfloat16* dst,
                             cudaStream_t st);
void launch_init_normal(float* out, size_t n, unsigned long long seed, float std_, cudaStream_t st);
void launch_fill(float* out, size_t n, float v, cudaStream_t st);

// ---- attention.cu
// Block partials + per-(row, head group) tickets of the persistent attention kernel.
struct AttnScratch {
    float* part_acc;  // [rows][nb_max][H][dh]
    float* part_ml;   // [rows][nb_max][H][2]
    int* row_ctr;     // [ctr_cap], zero between launches
    long long ctr_cap;
};
extern int g_attn_sm_cap;  // attention.cu persistent grid cap (0 = every SM, several CTAs each)
int attn_splits_for(int max_virtual_len);
// Tiles of rows sharing keys (attention.cu): rows [row0, row0+nrows) read the same keys in
// 64-key blocks [blo, bhi) -- one row, or up to 8*qw verify rows of one sequence over the
// blocks inside its committed prefix (kAttnTileRows queries per mma tile).
constexpr int kAttnTileRows = 8;
// bsh >= 0 marks a boundary tile: its last block bhi-1 holds the end of the common prefix
// (bsh keys) and then each row's own tree path; 16-key chunks inside [0, bsh) are staged
// once for all rows, the chunks past it once per row (the row's own keys), so the tile's
// rows no longer re-stream the prefix tail of that block one by one.
struct AttnTileDev {
    int row0, nrows, blo, bhi, bsh;
};
// groups: (row0, nrows, ctx_len, max virtual length) of rows sharing one committed prefix.
// attn_tile_qw: 8-query tiles per CTA item for these groups; build_attn_tiles returns the
// number of (tile, block) items of tiles of up to 8*qw rows
int attn_tile_qw(const std::vector<std::array<int, 4>>& groups);
// boundary: the rows of a group share their first ctx_len keys exactly (tree verify, draft
// levels), so shared tiles also take the block holding the end of the prefix (bsh)
long long build_attn_tiles(const std::vector<std::array<int, 4>>& groups, std::vector<AttnTileDev>& out, int qw,
                           bool boundary = false);
// merge: allow the in-register block merge (few-row tiles over long prefixes: tree verify,
// draft levels, catch-up rows); the AR prompt tiles keep the 16-warp kernel
void launch_attention_tiles(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, long long kv_slots,
                            const AttnRowsDev& rows, int M, const AttnTileDev* tiles, int n_tiles, long long n_items,
                            int qw, int H, int d, int max_virtual_len, const AttnScratch& sc, __nv_bfloat16* out,
                            cudaStream_t st, bool merge = true);
// total_keys: sum over rows of keys attended (host estimate; only sizes the launch)
// K/V: one layer of a [kv_slots][d] bf16 store
void launch_attention(const float* q, const __nv_bfloat16* K, const __nv_bfloat16* V, long long kv_slots,
                      const AttnRowsDev& rows, int M, int H, int d, int max_virtual_len, double total_keys,
                      const AttnScratch& sc, __nv_bfloat16* out, cudaStream_t st);

// ---- attention_tree.cu: tree-verify / draft-level attention, one CTA per (tile of <= 64 rows
// of one sequence, head) over the whole key range (prefix through a TMA ring, path keys from a
// node table in shared memory), bit-identical to launch_attention / launch_attention_tiles
struct TreeGroupDev {
    int row0, nrows, ctx_len, n_nodes;  // rows share keys [0, ctx_len); paths = node slots
    long long node_base;                // first KV slot of the group's node rows
    long long ctx_base, pre_base;       // committed prefix slots (pre_base for v < pre_len)
    int pre_len, pad;
};
struct TreeTileDev {
    int group, r0, nr;
};
int tree_attn_warps(int max_rows_per_group, int n_groups, int H, int dh, int max_nodes);
void build_tree_tiles(const std::vector<TreeGroupDev>& groups, int W, std::vector<TreeTileDev>& out);
// kmap / vmap: 2-D TMA maps over the store viewed as [layers * n_slots][d] (16 x 64 boxes,
// SWIZZLE_128B); layer_row0 = layer * n_slots; K / V: this layer's [n_slots][d] base
// AR steps (one row per group): a (row, head)'s 64-key blocks over a cluster of CTAs and their
// warps, block partials merged in order through distributed shared memory
void launch_attention_decode(const float* q, const CUtensorMap& kmap, const CUtensorMap& vmap, long long layer_row0,
                             const __nv_bfloat16* K, const __nv_bfloat16* V, const TreeGroupDev* groups, int n_groups,
                             int max_ctx, int H, int d, __nv_bfloat16* out, cudaStream_t st);
void launch_attention_tree(const float* q, const CUtensorMap& kmap, const CUtensorMap& vmap, long long layer_row0,
                           const __nv_bfloat16* K, const __nv_bfloat16* V, const AttnRowsDev& rows,
                           const TreeGroupDev* groups, const TreeTileDev* tiles, int n_tiles, int W, int H, int d,
                           int max_nodes, __nv_bfloat16* out, cudaStream_t st);

// ---- rewards.cu: per-sequence task reward and per-group standardized advantages
void launch_group_advantages(int n_groups, int g, const int* tok, long long stride, const int* len, const int* plen,
                             const long long* answer, double eps_var, double* rewards, double* adv, int* valid,
                             cudaStream_t st);

// ---- sample.cu
// Per-(row, chunk) records + per-row tickets of the multi-CTA row reductions.
struct RowScratch {
    void* buf;
    size_t bytes;
    int* ctr;       // [rows], zero between launches
    float* rowmax;  // [rows]
    int* exact;     // [rows] T > 0: 1 = the row's draw was resolved by the exact sequential pass
    unsigned long long* n_exact;  // running count of such rows (diagnostics)
    int rows;
};
size_t row_scratch_bytes(int rows, int V);
// uniforms (optional, [R]): the draw's Rng(key).uniform() supplied by the caller instead of
// derived from (seeds, key_pos) -- the "identical logits and supplied uniforms" parity mode
void launch_emit(const float* logits, int V, const int* row_idx, const unsigned long long* seeds, const int* key_pos,
                 int R, double temperature, int* out, int* err, const RowScratch& sc, cudaStream_t st,
                 const double* uniforms = nullptr);
// device evaluation of the glibc exp restatement (glibc_exp.cuh), for the parity tests
void launch_debug_exp(const double* x, size_t n, double* out, cudaStream_t st);
int emit_launches(double temperature);
void launch_topk_lsm(const float* logits, int V, int R, int k, int* out_tok, double* out_lp, const RowScratch& sc,
                     cudaStream_t st);

// ---- tree.cu
// Per-step descriptor of the live sequences (index i = live order), uploaded once a step.
struct StepSeqDev {
    int seq;        // global sequence slot
    int p;          // root position (= tokens.size()-1)
    int k, l;       // k_eff, l_eff (scheduler.cpp:127-133)
    int nsel;       // rows this sequence verifies
    int vrow_off;   // first verify row
    int root_row;   // row of this sequence's root logits in the draft top-k output (-1: no draft)
    int len_cap;
    int pre_len;         // prompt length (prefix shared by the group's members)
    long long pre_base;  // KV slot of the group leader's position 0
};

struct TreeDev {
    int tmax;                 // node capacity per sequence
    int ds;                   // draft feature / scratch slots per sequence
    int* tok;                 // [S][tmax]
    int* par;                 // [S][tmax]
    int* dep;                 // [S][tmax]
    double* lp;               // [S][tmax]
    double* conf;             // [S][tmax]
    int* fslot;               // [S][tmax] draft feature slot of expanded nodes
    int* n_nodes;             // [S]
    int* lvl_start;           // [S]
    int* lvl_cnt;             // [S]
    int* frontier;            // [S][16]
    int* sel;                 // [S][tmax] selected node ids (ascending)
    // rejection-sampling mode (reject.cu): children are SAMPLED from the draft distribution and
    // the tree shape must not depend on their values -- confidences are the static weights
    // conf(child j) = conf(parent) * 2^-(j+1) (exact dyadics), ties by node index only
    int static_rank = 0;
    int* qrow = nullptr;      // [S][tmax] expanded node -> row of its draft logits (q) buffer
};

struct SeqStateDev {
    int* tokens;                  // [S][max_seq]
    int* len;                     // [S]
    int* finished;                // [S]
    int* hit_eos;                 // [S]
    unsigned long long* seed;     // [S]
    int max_seq;
};

// Rows of a forward pass (inputs the forward consumes + attention metadata).
struct RowsDev {
    int* tok;              // [M]
    int* pos;              // [M]
    long long* kv_dst;     // [M]
    long long* ctx_base;   // [M]
    int* ctx_len;          // [M]
    int* chain_len;        // [M]
    long long* chain;      // [M][kMaxChain]
    long long* feat_off;   // [M] draft: offset of the previous feature (fuse input)
    long long* out_off;    // [M] draft: destination offset of the output feature
    int* key_pos;          // [M] verify: sampling key position
    unsigned long long* seed;  // [M] verify: sequence seed
    int* par_row;          // [M] verify: parent row within the sequence (-1 root)
    long long* pre_base;   // [M] verify: shared prompt K/V base (group leader)
    int* pre_len;          // [M] verify: shared prompt length
};

void launch_tree_root(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const int* topk_tok,
                      const double* topk_lp, int kmax_row, cudaStream_t st);
// qoff >= 0 (rejection mode): frontier node j of sequence i gets qrow = qoff + drow_off[i] + j
void launch_tree_frontier(int B, int level, const StepSeqDev* steps, const int* drow_off, const SeqStateDev& ss,
                          const TreeDev& tr, const RowsDev& rows, long long dcache_stride, long long dscratch_base,
                          int d, cudaStream_t st, int qoff = -1);
void launch_tree_expand(int B, int level, const StepSeqDev* steps, const int* drow_off, const TreeDev& tr,
                        const int* topk_tok, const double* topk_lp, cudaStream_t st);
void launch_tree_select(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const RowsDev& rows,
                        long long tcache_stride, long long tscratch_base, unsigned char* mask_dbg, int* err,
                        cudaStream_t st);
void launch_walk_commit(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const RowsDev& rows,
                        const int* emitted, int* acc_rows, int* result, cudaStream_t st);
// ---- reject.cu: speculative rejection sampling (the rollout's `acceptance = 1` mode)
// K i.i.d. children per row from q = softmax(draft logits / T): key of child c of row r is
// mix_key(keys[r], c); qstat[r] = (max, sum exp((l - max) / T)) of the row
void launch_sample_children(const float* q, int R, int V, int k, double temperature,
                            const unsigned long long* keys, int* out_tok, double* out_lp, double* qstat,
                            cudaStream_t st);
// multi-round speculative sampling walk (accept child x with prob min(1, r(x) / q(x)), residual
// r <- norm(max(r - q, 0)) after each rejection, bonus drawn from the final residual) + the
// same token commit as walk_commit. A node without selected children emits emitted[row] (the
// keyed sample_token draw), so AR steps equal the strict-match mode bit for bit.
void launch_walk_reject(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const RowsDev& rows,
                        const int* emitted, const float* logits, const float* rowmax, const float* qbuf,
                        const double* qstat, int V, double temperature, float* resid, int* acc_rows, int* result,
                        cudaStream_t st);
// test entry: n_trials independent rounds of ONE node: k candidates sampled from q, the
// multi-round rejection against p, out_tok = emitted token, out_acc = candidate accepted (1) or
// residual / bonus draw (0). Same device code as the rollout kernels.
void launch_debug_spec_sample(const float* p, const float* q, int V, int k, double temperature, int n_trials,
                              unsigned long long seed, float* resid, int* out_tok, int* out_acc, cudaStream_t st);

void launch_commit_kv(int B, const StepSeqDev* steps, const int* acc_rows, const int* result, int layers, int d,
                      __nv_bfloat16* K, __nv_bfloat16* V, long long layer_stride, long long tcache_stride,
                      long long tscratch_base, const float* hidden, float* feats, int max_seq, cudaStream_t st);
void launch_copy_rows_f32(const float* src, const int* src_row, const long long* dst_off, int R, int d, float* dst,
                          cudaStream_t st);
void launch_copy_kv_prefix(const int* src_seq, const int* dst_seq, const int* plen, int n, int max_plen, int layers,
                           int d, __nv_bfloat16* K, __nv_bfloat16* V, long long layer_stride, long long seq_stride,
                           cudaStream_t st);
void launch_prefill_commit(int n, const int* seqs, const int* qlen, const int* len_cap, const int* emitted,
                           const SeqStateDev& ss, cudaStream_t st);
void launch_gather_tokens(const int* seq, const int* pos, int R, const SeqStateDev& ss, int* out, cudaStream_t st);

}  // namespace sgb
