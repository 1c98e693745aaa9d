// Host engine of the B200 rollout: device-resident weights, paged-by-sequence KV stores,
// and the step loop of generate_dynamic_batch (scheduler.cpp:236-354) expressed as
// batched sm_100a kernels. One Engine per GPU; the C-ABI (capi.cpp) owns it.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <array>
#include <vector>

#include "gemm.h"
#include "kernels.h"

namespace sgb {

struct ModelDims {
    int vocab = 0, d = 0, layers = 0, heads = 0, dff = 0, max_seq = 0;
};

struct LayerDev {
    GemmWeight qkv, wo, w1, w2;
    const float *ln1_g = nullptr, *ln1_b = nullptr, *ln2_g = nullptr, *ln2_b = nullptr;
};

// Offsets of the reference's flat parameter layout (tinylm.hpp:58-81, 133-189).
struct FlatLayout {
    size_t tok_emb = 0, pos_emb = 0, lnf_g = 0, lnf_b = 0, lm_head = 0, w_fuse = 0, total = 0;
    struct L {
        size_t ln1_g, ln1_b, wq, wk, wv, wo, ln2_g, ln2_b, w1, w2;
    };
    std::vector<L> layers;
    static FlatLayout target(const ModelDims& m);
    static FlatLayout draft(const ModelDims& m, int n_layers);
};

struct KvStore {
    __nv_bfloat16* K = nullptr;
    __nv_bfloat16* V = nullptr;
    int layers = 0;
    long long n_slots = 0;       // per layer
    long long seq_stride = 0;    // slots per sequence region
    long long scratch_base = 0;  // first scratch slot
    long long layer_stride() const { return n_slots; }
};

struct SpecCfg {
    int n_verify = 1, k_draft = 0, l_draft = 0;
};

struct RolloutArgs {
    std::vector<std::vector<int>> prompts;
    int g = 1;
    double alpha = 2.0;
    int k_max = 10, l_max = 6, c_peak = 1;
    int mode = 0;  // 0 vanilla, 1 fixed_spec, 2 adaptive_spec (scheduler.hpp:46)
    bool early_term = true;
    double temperature = 0.0;
    uint64_t seed = 0;
    int max_new_tokens = 0;
    SpecCfg fixed;
    std::vector<int> seq_max_new;  // optional per-sequence caps (c3 extension)
    bool want_features = true;
    int sid_offset = 0;  // global sid of local sequence 0 (seed parity under sharding)
    // 0: keyed strict match (verify, drafttree.cpp:170-222; the parity mode), 1: speculative
    // rejection sampling (reject.cu; T > 0 only -- at T = 0 it is the strict-match mode)
    int acceptance = 0;
    // optional caller buffer [n_seqs][max_seq-1][d] for the features (skips RolloutResult.features):
    // one pinned-staging DMA of the feature store, then a multi-threaded host scatter
    float* features_out = nullptr;
};

struct StepStat {
    int b_cur = 0, n_verify = 0, k_draft = 0, l_draft = 0, accepted = 0, rows = 0, draft_rows = 0;
};

// Per kernel-class device time (CUDA events on the launching stream) and algorithmic work.
enum KernelClass { kClsGemm = 0, kClsAttn, kClsRow, kClsLmHead, kClsSample, kClsTree, kClsCommit, kNumCls };
struct KernelProfile {
    double ms = 0, bytes = 0, flops = 0;
    long long launches = 0;
};

struct RolloutResult {
    std::vector<std::vector<int>> tokens;
    std::vector<int> prompt_len, hit_eos;
    std::vector<std::vector<float>> features;
    std::vector<StepStat> steps;
    std::vector<int> events;  // (step, seq, accepted) triples
    long long total_accepted = 0, total_verify_slots = 0;
    long long target_forwards = 0, draft_forwards = 0, kernel_launches = 0;
    double seconds = 0;  // device time of the step loop incl. prefill (CUDA events)
    double prefill_seconds = 0;
    std::vector<double> step_seconds;  // device time of every decode step (CUDA events)
    std::vector<double> step_bytes, step_flops;  // SURVEY §8(d) algorithmic bytes / flops per step
    long long h2d_bytes = 0, d2h_bytes = 0;
    // host side of the step loop: device idle between a step's end and its successor's first
    // operation (host planning + launch latency; CUDA events) and host time spent issuing the
    // steps (wall clock, up to the per-step sync) -- what a device-resident / graph loop could save
    double host_gap_seconds = 0, host_enqueue_seconds = 0;
    bool waves = false;  // more sequences than KV regions: groups were admitted as regions freed
};

class Engine {
   public:
    Engine(const ModelDims& dims, int draft_layers, int device, int max_seqs, int max_rows, int k_max, int l_max);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    const ModelDims& dims() const { return dims_; }
    int draft_layers() const { return dlayers_; }
    size_t target_param_count() const { return tlay_.total; }
    size_t draft_param_count() const { return dlay_.total; }

    void upload_target(const float* flat, size_t n);  // host fp32, reference layout
    void upload_draft(const float* flat, size_t n);
    void init_random(uint64_t seed);                  // benchmark weights (device RNG)
    void download_draft(float* flat, size_t n);

    // ---- per-op parity entry points (host in / host out)
    void cache_reset(int slot, bool draft);
    int cache_len(int slot, bool draft) const;
    void cache_read(int slot, bool draft, float* k, float* v);  // [layers][len][d]
    void cache_gather_tail(int slot, int base, const int* keep, int n);
    void forward_target(int slot, const int* tokens, const int* positions, int rows, const unsigned char* mask,
                        float* logits, float* hidden);
    void forward_draft(int slot, const int* tokens, const float* prev_feat, const int* positions, int rows, bool extend,
                       float* feats, float* logits);
    // sample_token per row; uniforms (optional) replace the keyed Rng(key).uniform() draws;
    // exact_rows (optional) receives 1 for rows resolved by the exact sequential pass
    void emit(const float* logits, int rows, int vocab, double temperature, const unsigned long long* seeds,
              const int* key_pos, int* out, const double* uniforms = nullptr, int* exact_rows = nullptr);
    void debug_exp(const double* x, size_t n, double* y);
    unsigned long long exact_draws();  // T > 0 draws resolved by the exact sequential pass so far
    void topk_logsoftmax(const float* logits, int rows, int vocab, int k, int* tok, double* lp);

    // ---- the rollout (generate_dynamic_batch drop-in)
    RolloutResult rollout(const RolloutArgs& args);

    // device-resident state of the last rollout (for the draft update)
    const float* d_feats() const { return feats_; }
    const int* d_tokens() const { return ss_.tokens; }
    cudaStream_t stream() const { return st_; }
    long long launches() const { return launches_; }
    void set_profiling(bool on);
    void set_force_splits(int s) { force_splits_ = s; }
    void read_profile(KernelProfile* out, int n, bool reset);

    // ---- online draft learning (draft_update, grpo.cpp:177-186)
    struct DraftUpdateArgs {
        // sequences: either host data (tokens/lens/features) or the last rollout (device-resident)
        bool use_last_rollout = false;
        int n_seqs = 0;
        const int* tokens = nullptr;      // concatenated
        const int* lens = nullptr;        // [n_seqs]
        const float* features = nullptr;  // concatenated (len-1)*d per sequence
        double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8, weight_decay = 0.0;
        double w_feat = 1.0, w_tok = 0.1;
        long long rows_total = 0;  // > 0: global row normaliser (data-parallel shard)
        bool apply_step = true;    // false: only compute loss + gradient (grad_out)
        float* grad_out = nullptr; // optional host copy of the gradient (reference flat layout)
        // optional hook run on the device gradient before the AdamW step (NCCL all-reduce)
        void (*grad_hook)(float* dgrad, size_t n, cudaStream_t st, void* ctx) = nullptr;
        void* hook_ctx = nullptr;
    };
    struct DraftLossTerms {
        double feature_loss = 0, token_loss = 0, total = 0;
        long long rows = 0;
        double seconds = 0;
    };
    DraftLossTerms draft_update(const DraftUpdateArgs& a);

    // ---- GRPO policy update on the device (policy_update, grpo.cpp:163-175)
    struct PolicyArgs {
        int n_seqs = 0;
        const int* tokens = nullptr;       // concatenated
        const int* lens = nullptr;         // [n_seqs]
        const int* prompt_lens = nullptr;  // [n_seqs]
        const double* weights = nullptr;   // [n_seqs] TrainSeq::weight (the advantage)
        double lr = 2e-4, beta1 = 0.9, beta2 = 0.999, eps = 1e-8, weight_decay = 0.0;
        long long tokens_total = 0;  // > 0: global response-token normaliser (data-parallel shard)
        bool apply_step = true;
        float* grad_out = nullptr;  // optional host copy of the gradient (reference flat layout)
        void (*grad_hook)(float* dgrad, size_t n, cudaStream_t st, void* ctx) = nullptr;
        void* hook_ctx = nullptr;
    };
    struct PolicyTerms {
        double loss = 0;
        long long tokens = 0, rows = 0;
        double seconds = 0;
        bool skipped = false;
    };
    // keep the fp32 target master on the device from the next upload (needed by policy_update)
    void policy_enable();
    PolicyTerms policy_update(const PolicyArgs& a);
    void download_target(float* flat, size_t n);
    void policy_adamw_state(float* m, float* v, long long* t, bool upload);
    void adamw_reset();
    void adamw_state(float* m, float* v, long long* t, bool upload);
    // measure_c_peak's latency_fn on the device (roofline.cpp:78-108 / tools/sgrpo.cpp:38-49):
    // one batched target forward of b rows (EOS token, position 0, self-only attention),
    // median device seconds over `reps` after `warmup` untimed launches.
    double latency_probe(int b, int warmup, int reps);

    // debug tree driver (tests): expands one tree on device with host-supplied logits
    struct DebugTree {
        std::vector<int> tok, par, dep, sel;
        std::vector<double> lp, conf;
        std::vector<unsigned char> mask;
    };
    DebugTree debug_tree_cb(int root_token, int k, int l, int n_verify,
                            void (*fn)(void* ctx, int n_front, const int* node_ids, const int* tok, const int* par,
                                       int n_nodes, float* logits_out),
                            void* ctx);

   private:
    struct Fwd {
        int M = 0;
        bool draft = false;
        const float* feat_base = nullptr;  // draft fuse features
        float* y_out = nullptr;            // final LN fp32 [M][d]
        bool logits = false;
        int lm_rows = 0;
        const int* lm_idx = nullptr;  // subset of rows for the LM head (nullptr = all)
        float* logits_out = nullptr;
        int max_vlen = 0;
        double attn_kv_unique = 0;  // distinct KV tokens read per layer (roofline bytes)
        double attn_row_keys = 0;   // sum over rows of keys attended (roofline flops)
        bool prefix_share = false;  // verify rows read their prompt K/V from the group leader
        // rows sharing one committed prefix: (row0, nrows, ctx_len, max virtual length); the
        // prefix blocks then run as shared tiles of up to 8 rows (attention.cu)
        const std::vector<std::array<int, 4>>* groups = nullptr;
        // the groups' rows share exactly ctx_len keys (tree verify, draft levels; not the
        // AR prompt groups): shared tiles also cover the prefix-end block (attention.cu)
        bool groups_exact = false;
        // tree-verify / draft-level groups for attention_tree.cu (nullptr: attention.cu)
        const std::vector<TreeGroupDev>* tree = nullptr;
        // attention.cu shared tiles may merge block partials in registers (not the AR prompt tiles)
        bool merge_tiles = false;
        // AR step of few rows: `tree` holds one group per row, run by the cluster decode kernel
        bool decode = false;
        int decode_max_ctx = 0;
    };
    void forward(const Fwd& f);
    bool boundary_tiles() const;

  public:
    // rewards (grpo.cpp:99-116) and standardized advantages (grpo.cpp:121-136) of the last
    // rollout's groups, computed from its token table in HBM; valid[b] = 0 for filtered groups
    void group_advantages(const long long* answers, int n_groups, int g, double eps_var, double* rewards, double* adv,
                          int* valid);
    // cumulative count of target forward launches (the reference's target_forward_calls())
    long long target_forward_calls() const { return target_forward_calls_; }

  private:
    void convert_target(const float* staging);
    void convert_draft();
    void alloc_rows();
    void upload_rows_host(int M, const std::vector<int>& tok, const std::vector<int>& pos,
                          const std::vector<long long>& kv_dst, const std::vector<long long>& ctx_base,
                          const std::vector<int>& ctx_len, const std::vector<int>& chain_len,
                          const std::vector<long long>& chain, const std::vector<long long>* feat_off);
    void lm_head(const __nv_bfloat16* a_rows, const GemmAct& act, int R, float* logits);
    void count(int n = 1) { launches_ += n; }
    void gemm(const GemmWeight& w, const GemmAct& a, int M, const GemmEpi& epi, int cls, double out_bytes);
    void ln(int M, const float* g, const float* b, float* y);
    // x (+)= a.W^T [+ pos_emb], then LayerNorm(x) -> a_ (and y): the residual GEMMs (wo, w2)
    // and the draft fuse. Token tiles >= 64 run the GEMM in kEpiPartials mode (one unit per
    // (tile, chunk)) and add the chunks in order inside the LayerNorm kernel; smaller ones
    // use the GEMM's own split-K finisher. Both give the same bits.
    void gemm_resid_ln(const GemmWeight& w, const GemmAct& a, int M, bool accumulate, bool add_pos, const float* g,
                       const float* b, float* y);
    int pbeg();
    void pend(int cls, int e0, double bytes, double flops);
    void pflush();
    struct PRec {
        int cls, e0, e1;
        double bytes, flops;
    };
    bool prof_ = false;
    std::vector<cudaEvent_t> evs_;
    int ev_used_ = 0;
    std::vector<PRec> precs_;
    KernelProfile prof_cls_[kNumCls];

    ModelDims dims_;
    int dlayers_, device_, max_seqs_, max_rows_, k_max_, l_max_;
    cudaStream_t st_ = nullptr;
    FlatLayout tlay_, dlay_;

    // weights
    std::vector<LayerDev> tL_, dL_;
    __nv_bfloat16 *tw_ = nullptr, *dw_ = nullptr;  // bf16 weight arenas
    float* tsmall_ = nullptr;                      // target fp32: tok_emb | pos_emb | LN params
    float* dmaster_ = nullptr;                     // draft fp32 flat (master weights)
    const float *tok_emb_ = nullptr, *pos_emb_ = nullptr, *lnf_g_ = nullptr, *lnf_b_ = nullptr;
    const float *dlnf_g_ = nullptr, *dlnf_b_ = nullptr;
    GemmWeight lm_head_, w_fuse_;
    bool target_ready_ = false, draft_ready_ = false;

    // kv + sequence state
    KvStore tkv_, dkv_;
    SeqStateDev ss_{};
    float* feats_ = nullptr;  // [S][max_seq][d]
    float* dfeat_ = nullptr;  // [S][ds][d]
    TreeDev tr_{};
    std::vector<int> cache_len_t_, cache_len_d_;

    // activations
    float *x_ = nullptr, *q_ = nullptr, *y_ = nullptr, *logits_ = nullptr, *featin_ = nullptr;
    RowScratch rsc_{};  // multi-CTA sampling / top-k records
    float* gpart_ = nullptr;  // kEpiPartials chunk sums [chunks][max_rows][d]
    float* feats_host_ = nullptr;  // pinned staging of the feature store (lazy)
    size_t feats_host_cap_ = 0;
    size_t gpart_cap_ = 0;
    float *pacc_ = nullptr, *pml_ = nullptr;
    AttnScratch asc_{};
    __nv_bfloat16 *a_ = nullptr, *att_ = nullptr, *h_ = nullptr, *fuse_ = nullptr, *a2_ = nullptr;
    GemmAct act_a_, act_att_, act_h_, act_fuse_, act_a2_;
    GemmWorkspace ws_;
    int force_splits_ = 0;
    int max_vlen_cap_ = 0;
    // row descriptors
    RowsDev rows_{};
    int* lm_idx_ = nullptr;
    int *topk_tok_ = nullptr, *emitted_ = nullptr, *acc_rows_ = nullptr, *result_ = nullptr, *err_ = nullptr;
    double* topk_lp_ = nullptr;
    StepSeqDev* steps_ = nullptr;
    AttnTileDev* tiles_ = nullptr;  // [2 * max_rows] attention tiles of the current forward
    std::vector<AttnTileDev> htiles_;
    std::vector<std::array<int, 4>> groups_;
    std::vector<TreeGroupDev> tgroups_;
    std::vector<TreeTileDev> ttiles_;
    TreeGroupDev* d_tgroups_ = nullptr;
    TreeTileDev* d_ttiles_ = nullptr;
    CUtensorMap tkmap_, tvmap_, dkmap_, dvmap_;  // [layers * n_slots][d] views of the KV stores
    bool tree_attn_ok(int max_nodes) const;
    int* drow_ = nullptr;
    int* misc_i_ = nullptr;
    long long* misc_l_ = nullptr;
    unsigned char* mask_dbg_ = nullptr;
    int *h_result_ = nullptr;  // pinned
    long long launches_ = 0;

    // ---- training state (allocated on the first draft_update)
    struct Train {
        bool ready = false;
        int rmax = 0, lc = 0, smax = 0;
        float *x0, *xmid, *xfin, *fhat, *dlnf, *dx, *dxmid, *dx0, *ctx, *dctx, *da, *qkv, *dqkv, *fch, *dhg, *dgb;
        float *lse, *Drow, *mu1, *rs1, *mu2, *rs2, *muf, *rsf, *logits, *sc, *grad, *m, *v, *feat_in;
        __nv_bfloat16 *fuse, *a1, *a2, *ctx_b, *fhat_b, *dx_b, *dxmid_b, *hg, *dfch_b, *dqkv_b, *dlog, *tA, *tB;
        __nv_bfloat16 *dflat_b, *wqkv_ref, *lm_ref;
        int *tok, *pos, *next, *seq_first, *seq_last, *tiles;
        long long *prev_off, *tgt_off;
        double* loss_row;
        long long adam_t = 0;
        size_t feat_cap = 0;
        GemmAct act_fuse, act_a1, act_a2, act_ctx, act_hg, act_dx, act_dxmid, act_dfch, act_dqkv, act_dlog;
        GemmWeight w2_ref, w1_ref, wo_ref, wqkv_ref_w, lm_ref_w;
    } tr2_;
    std::vector<int> last_lens_;   // token counts of the last rollout's sequences
    std::vector<int> last_plens_;  // and their prompt lengths
    bool last_waves_ = false;      // the last rollout recycled KV regions (its data left HBM)
    long long target_forward_calls_ = 0;
    double* adv_buf_ = nullptr;    // [2 * max_rows] rewards + advantages of group_advantages
    // rejection-sampling mode buffers (allocated on first use): draft logits of every expanded
    // node of a step [max_rows][V], their (max, sum) stats, per-sequence residuals, child keys
    float* qbuf_ = nullptr;
    double* qstat_ = nullptr;
    unsigned long long* rkeys_ = nullptr;
    void reject_alloc();
    void train_alloc();
    void train_refresh_ref_weights();
    // ---- policy update state (engine_policy.cu)
    bool keep_master_ = false;
    float* tmaster_ = nullptr;  // fp32 target master (reference flat layout)
    bool draft_lm_stale_ = false;
    std::vector<void*> pol_ptrs_;
    struct Pol {
        bool ready = false;
        int rmax = 0, lc = 0;
        long long adam_t = 0;
        float *grad = nullptr, *m = nullptr, *v = nullptr;
        __nv_bfloat16 *flat_b = nullptr, *wqkv_ref = nullptr;
        struct Layer {
            float *x_in, *mu1, *rs1, *qkv, *ctx, *lse, *xmid, *mu2, *rs2, *fch;
            __nv_bfloat16 *a1, *ctxb, *a2, *hg;
            GemmAct act_a1, act_ctx, act_a2, act_hg;
        };
        std::vector<Layer> L;
        struct Refs {
            GemmWeight wqkv, wo, w1, w2;
        };
        std::vector<Refs> refs;
        GemmWeight lm_ref;
        float *xfin, *fhat, *muf, *rsf, *dlnf, *dx, *dxmid, *da, *dctx, *dqkv, *dhg, *dgb, *Drow, *logits;
        __nv_bfloat16 *fhat_b, *dfch_b, *dx_b, *dxmid_b, *dqkv_b, *dlog, *tA, *tB;
        int *tok, *pos, *next, *seq_first, *seq_last, *tiles, *csr;
        double *rscale, *loss_row;
        GemmAct act_fhat, act_dx, act_dxmid, act_dfch, act_dqkv, act_dlog;
    } pol_;
    void policy_alloc();
    void policy_refresh_ref_weights();
    void wgrad(const __nv_bfloat16* dyT, int N, const __nv_bfloat16* xT, int Kfeat, int Rp, float* grad_dst, int ld);
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr, evs_a_ = nullptr, evs_b_ = nullptr, evs_c_ = nullptr;  // rollout / per-step
};

}  // namespace sgb
