/*
 * sgrpo_b200.h -- C-ABI of the B200-native GRPO-rollout hot path (libsgrpo_b200.so).
 *
 * This is the drop-in boundary for the reference's C++ operator API (namespace sgrpo,
 * /root/reference/proj). Every entry point below names the reference interface it
 * replaces (file:line, relative to proj/). Arguments are plain pointers and sizes; host
 * buffers in, host buffers out; no C++ or torch types cross the boundary.
 *
 * Errors: every function returns an int status (SGB_OK == 0). Non-zero codes map onto the
 * exception types the reference throws:
 *   SGB_EINVAL  1  std::invalid_argument   (empty input, bad token id, bad config, ...)
 *   SGB_ERANGE  2  std::out_of_range       (position >= max_seq_len, cache capacity)
 *   SGB_ERUNTIME 3 std::runtime_error      (non-finite logits, weights not uploaded)
 *   SGB_EDOMAIN 4  std::domain_error       (NaN / all -inf logits in sampling)
 *   SGB_ECUDA   5  CUDA failure -- there is NO CPU fallback
 * sgb_last_error() returns the thread-local message of the last failure.
 */
#ifndef SGRPO_B200_H
#define SGRPO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGB_ABI_VERSION 1

/* ModelConfig (include/sgrpo/tinylm.hpp:16-37). */
typedef struct sgb_model_config {
    int vocab_size, d_model, n_layers, n_heads, d_ff, max_seq_len;
    unsigned long long seed;
} sgb_model_config;

/* SchedParams + GenOptions (include/sgrpo/scheduler.hpp:34-58). */
typedef struct sgb_gen_options {
    double alpha;              /* Eq. 3 alpha (SchedParams.alpha)               */
    int k_max, l_max, c_peak;  /* SchedParams                                    */
    int mode;                  /* DecodeMode: 0 vanilla, 1 fixed_spec, 2 adaptive */
    int early_term;            /* GenOptions.early_term                          */
    double temperature;        /* GenOptions.temperature                         */
    unsigned long long seed;   /* GenOptions.seed                                */
    int max_new_tokens;        /* GenOptions.max_new_tokens (0: max_seq_len)     */
    int fixed_n_verify, fixed_k_draft, fixed_l_draft; /* GenOptions.fixed        */
    const int* seq_max_new;    /* optional per-sequence caps (c3 extension) or NULL */
    int want_features;         /* copy SeqResult.features back                   */
    int sid_offset;            /* global sid of this shard's first sequence (data-parallel ranks) */
    double* step_seconds;      /* optional [step_cap]: measured device seconds of every step (GenStats
                                  StepRecord.sim_latency_s, scheduler.cpp:356-368), or NULL */
    int acceptance;            /* 0: keyed strict match, the reference's verify (drafttree.cpp:170-222);
                                  1: speculative rejection sampling (draft children sampled from q,
                                  accept min(1, p/q), residual resample; T > 0; lossless in
                                  distribution, not token-identical to the reference) */
} sgb_gen_options;

/* GenStats summary (scheduler.hpp:68-89) plus device measurements. */
typedef struct sgb_rollout_stats {
    long long total_accepted, total_verify_slots; /* tau = accepted / slots (scheduler.cpp:72-75) */
    int n_steps;
    long long target_forwards, draft_forwards, kernel_launches;
    double seconds; /* device time of prefill + step loop, CUDA events (inputs resident) */
    long long h2d_bytes, d2h_bytes; /* host<->device bytes moved by the call */
    /* host side of the step loop: device idle from a step's end to the next step's first
     * operation (CUDA events), and host wall time issuing the steps (up to each step's sync) */
    double host_gap_seconds, host_enqueue_seconds;
} sgb_rollout_stats;

typedef struct sgb_engine sgb_engine;

const char* sgb_last_error(void);
int sgb_version(void);
int sgb_device_count(int* out);

/* Engine: one per GPU. Owns bf16 weights, KV stores for max_seqs sequences of
 * max_seq_len tokens, and activation buffers for max_rows rows per forward.
 * k_max/l_max bound the speculation tree (SchedParams.k_max/l_max). */
int sgb_engine_create(const sgb_model_config* cfg, int draft_layers, int device, int max_seqs, int max_rows,
                      int k_max, int l_max, sgb_engine** out);
int sgb_engine_destroy(sgb_engine* e);
int sgb_param_counts(sgb_engine* e, size_t* target, size_t* draft);

/* Weights in the reference's flat fp32 layout: init_model (tinylm.hpp:133-150) and
 * init_draft (tinylm.hpp:172-189); also the SGRPOCK1 payload (src/tinylm.cpp:14-105). */
int sgb_upload_target(sgb_engine* e, const float* flat, size_t n);
int sgb_upload_draft(sgb_engine* e, const float* flat, size_t n);
int sgb_download_draft(sgb_engine* e, float* flat, size_t n);
/* Benchmark weights drawn on the device with init_flat's distributions (not bit-identical). */
int sgb_init_random(sgb_engine* e, unsigned long long seed);

/* SGRPOCK1 checkpoints (src/tinylm.cpp:14-105): header query (host only, no GPU), load into
 * the engine (target or draft, config must match; payload mmapped and converted on the
 * device), and save the engine's fp32 draft master in the reference's byte layout. */
int sgb_checkpoint_info(const char* path, int* kind /* 0 target, 1 draft */, sgb_model_config* cfg,
                        int* draft_layers, size_t* param_count);
int sgb_load_checkpoint(sgb_engine* e, const char* path, int* kind);
int sgb_save_draft_checkpoint(sgb_engine* e, const char* path);

/* ---- per-op parity entry points -------------------------------------------------- */
/* KvCacheT reset / len / gather_tail (tinylm.hpp:232-269). slot = engine sequence slot. */
int sgb_cache_reset(sgb_engine* e, int slot, int draft);
int sgb_cache_len(sgb_engine* e, int slot, int draft, int* out);
int sgb_cache_read(sgb_engine* e, int slot, int draft, float* k, float* v); /* [layers][len][d] */
int sgb_cache_gather_tail(sgb_engine* e, int slot, int base, const int* keep, int n);

/* forward_target<T> (tinylm.hpp:422-463): mask NULL = causal; rows are appended to the
 * slot's cache. logits [rows][vocab], hidden [rows][d]. */
int sgb_forward_target(sgb_engine* e, int slot, const int* tokens, const int* positions, int rows,
                       const unsigned char* mask, float* logits, float* hidden);
/* forward_draft_rows<T> (tinylm.hpp:502-563) with cache = the slot's draft cache. */
int sgb_forward_draft_rows(sgb_engine* e, int slot, const int* tokens, const float* prev_features,
                           const int* positions, int rows, int extend_cache, float* features, float* logits);
/* sample_token<T> (tinylm.hpp:591-628) per row with key mix_key(seeds[i], key_pos[i])
 * (the key verify derives, drafttree.cpp:184-190). */
int sgb_sample_rows(sgb_engine* e, const float* logits, int rows, int vocab, double temperature,
                    const unsigned long long* seeds, const int* key_pos, int* out);
/* sample_token<T> (tinylm.hpp:591-628) with the draw's uniform SUPPLIED per row (u = uniforms[i]
 * * sum instead of Rng(key).uniform() * sum): the "identical logits and supplied uniforms" parity
 * mode. Every CDF term is glibc's exp bit for bit; rows whose u lies within the fast path's
 * summation-order error bound of a CDF boundary are redone in the reference's sequential order
 * (exact_rows[i] = 1, optional). */
int sgb_sample_rows_u(sgb_engine* e, const float* logits, int rows, int vocab, double temperature,
                      const double* uniforms, int* out, int* exact_rows);
/* Test entry for the rejection-sampling acceptance (reject.cu): n_trials independent rounds of one
 * node -- k candidates drawn from softmax(q_logits / T), multi-round rejection against
 * softmax(p_logits / T). out_tok = emitted token, out_acc = 1 if a candidate was accepted. */
int sgb_debug_spec_sample(sgb_engine* e, const float* p_logits, const float* q_logits, int vocab, int k,
                          double temperature, int n_trials, unsigned long long seed, int* out_tok, int* out_acc);
/* Count of T > 0 draws (rollouts and sample calls) the engine resolved by the exact pass. */
int sgb_exact_draws(sgb_engine* e, unsigned long long* out);
/* The device's exp(): the restatement of glibc's exp (csrc/glibc_exp.cuh), for parity tests. */
int sgb_debug_exp(sgb_engine* e, const double* x, size_t n, double* out);

/* log_softmax_row<double> + topk_tokens (nn.hpp:172-180, drafttree.cpp:20-30). */
int sgb_topk_logsoftmax(sgb_engine* e, const float* logits, int rows, int vocab, int k, int* tokens,
                        double* log_probs);

/* expand_tree_with + rerank_candidates + build_tree_mask (drafttree.cpp:34-168) on the
 * device, with the draft logits of each expanded node supplied by a callback (the
 * reference's ExpandFn, drafttree.hpp:33). Outputs: nodes (tok/par/dep/lp/conf, capacity
 * cap), selected node ids [n_sel] and mask [n_sel][n_sel]. */
typedef void (*sgb_logits_fn)(void* ctx, int n_front, const int* node_ids, const int* node_tok,
                              const int* node_par, int n_nodes, float* logits_out);
int sgb_build_tree(sgb_engine* e, int root_token, int k_draft, int l_draft, int n_verify, sgb_logits_fn fn,
                   void* ctx, int cap, int* tok, int* par, int* dep, double* lp, double* conf, int* n_nodes,
                   int* sel, int* n_sel, unsigned char* mask);

/* ---- the hot path ------------------------------------------------------------------ */
/* generate_dynamic_batch (include/sgrpo/scheduler.hpp:99-102, src/scheduler.cpp:236-354).
 * prompts: concatenated token ids, prompt_lens[n_prompts]; g = group size.
 * Outputs (sequence order = global sid = prompt_idx*g + r):
 *   tokens [n_prompts*g][max_seq_len] (row i holds lens[i] tokens), lens, prompt_len, hit_eos,
 *   features [n_prompts*g][max_seq_len-1][d] (optional, NULL to skip).
 * Per-step GenStats records (b_cur, n_verify, k_draft, l_draft, accepted) go to
 * step_rec[5*i..] for i < min(n_steps, step_cap). */
int sgb_rollout(sgb_engine* e, const int* prompts, const int* prompt_lens, int n_prompts, int g,
                const sgb_gen_options* opt, int* tokens, int* lens, int* prompt_len, int* hit_eos, float* features,
                int* step_rec, int step_cap, sgb_rollout_stats* stats);

/* Kernel-class profiler: CUDA events around every launch on the engine's stream.
 * Classes: 0 GEMM (tcgen05), 1 attention, 2 row ops (LN/reduce/GELU/scatter), 3 LM head,
 * 4 sampling, 5 tree/walk, 6 KV commit. Per class: device ms, algorithmic bytes/flops, launches. */
int sgb_profile_enable(sgb_engine* e, int on);
int sgb_profile_read(sgb_engine* e, int n_cls, double* ms, double* bytes, double* flops, long long* launches,
                     int reset);

/* ---- online draft learning ------------------------------------------------------------ */
/* AdamW hyper-parameters (grpo.hpp:97-103) and loss weights (draft_update, grpo.hpp:115-116). */
typedef struct sgb_adamw {
    double lr, beta1, beta2, eps, weight_decay;
    double w_feat, w_tok;
    long long rows_total; /* > 0: global row normaliser for a data-parallel shard (grpo.hpp:286-290) */
    int apply_step;       /* 0: loss + gradient only */
    int allreduce_grad;   /* 1: NCCL all-reduce (sum) of the gradient over the engine's DP group */
} sgb_adamw;

/* ---- data parallelism over NVLink: one engine per GPU / process ------------- */
/* NCCL unique id (128 bytes) created on rank 0 and shared by the caller's launcher. */
int sgb_nccl_unique_id(unsigned char* id128);
/* Join the data-parallel group (ncclCommInitRank) on the engine's device. */
int sgb_nccl_init(sgb_engine* e, int rank, int world, const unsigned char* id128);
/* C2: in-place sum over ranks of small host vectors (rollout statistics, row counts). */
int sgb_allreduce_sum_f64(sgb_engine* e, double* vals, int n);
int sgb_allreduce_sum_i64(sgb_engine* e, long long* vals, int n);

/* DraftLossTerms (grpo.hpp:79-84) + device seconds. */
typedef struct sgb_draft_terms {
    double feature_loss, token_loss, total;
    long long rows;
    double seconds;
} sgb_draft_terms;

/* draft_update (grpo.cpp:177-186 -> draft_loss_grad grpo.hpp:278-344 -> AdamW::step
 * grpo.cpp:142-161) on sequences given by the host: tokens concatenated, lens[n_seqs],
 * features concatenated ((len-1)*d per sequence). grad_out (optional) receives the fp32
 * gradient in the reference flat draft layout. The AdamW moments live in the engine. */
int sgb_draft_update(sgb_engine* e, int n_seqs, const int* tokens, const int* lens, const float* features,
                     const sgb_adamw* opt, float* grad_out, sgb_draft_terms* terms);
/* Same, on the sequences of the engine's last sgb_rollout, read straight from HBM. */
int sgb_draft_update_last(sgb_engine* e, const sgb_adamw* opt, float* grad_out, sgb_draft_terms* terms);
/* Reset the AdamW moments and step counter (a fresh AdamW object). */
int sgb_adamw_reset(sgb_engine* e);
/* AdamW::m, AdamW::v, AdamW::t (grpo.hpp:97-103) of the device draft optimizer: upload = 1
 * installs a caller's optimizer state (m / v NULL = zeros), 0 reads it back (NULL = skip). */
int sgb_adamw_state(sgb_engine* e, float* m, float* v, long long* t, int upload);
/* GenStats.events (scheduler.hpp:73-86, scheduler.cpp:326) of the engine's last sgb_rollout:
 * (step, seq, accepted) triples, min(n, cap) written; the measured prefill seconds
 * (GenStats.prefill_sim_s). */
int sgb_rollout_events(sgb_engine* e, int* triples, long long cap, long long* n, double* prefill_seconds);
/* Per-step algorithmic work of the last rollout (bf16 weight + K/V bytes, GEMM +
 * attention flops, target and draft passes) and the measured device seconds of each step:
 * roofline time = sum_t max(bytes_t / BW, flops_t / F). min(n, cap) entries written. */
int sgb_rollout_roofline(sgb_engine* e, double* bytes, double* flops, double* seconds, long long cap, long long* n);

/* ---- GRPO policy update on the device (policy_update, grpo.cpp:163-175) -------------------- */
/* Keep the fp32 target master on the device from the next sgb_upload_target / sgb_init_random
 * (the policy update trains it; 4 bytes per parameter). */
int sgb_policy_enable(sgb_engine* e);
/* The fp32 target master (reference flat layout), e.g. to mirror Model::flat after an update. */
int sgb_download_target(sgb_engine* e, float* flat, size_t n);
typedef struct sgb_policy_terms {
    double loss;      /* policy_loss_grad's return value (grpo.hpp:235-276) */
    long long tokens; /* response tokens of these sequences (the loss normaliser unless rows_total) */
    long long rows;   /* training rows (n - 1 per sequence with a response) */
    double seconds;
    int skipped;      /* no response tokens: nothing to do (policy_update returns false) */
} sgb_policy_terms;
/* policy_loss_grad (grpo.hpp:235-276: target_train_forward / backward, tinylm.hpp:804-866) over
 * TrainSeq{tokens, prompt_len, weight = advantage} and one AdamW::step (grpo.cpp:142-161) on the
 * device master, then the bf16 inference weights are rebuilt. opt->rows_total > 0: global
 * response-token count of a data-parallel shard; opt->allreduce_grad: NCCL sum of the gradient.
 * opt->w_feat / w_tok are unused. */
int sgb_policy_update(sgb_engine* e, int n_seqs, const int* tokens, const int* lens, const int* prompt_lens,
                      const double* weights, const sgb_adamw* opt, float* grad_out, sgb_policy_terms* terms);
/* AdamW::m / v / t of the device policy optimizer (upload = 1 installs, 0 reads back). */
int sgb_policy_adamw_state(sgb_engine* e, float* m, float* v, long long* t, int upload);

/* ---- hardware profile: C_peak calibration (Alg. 2, src/roofline.cpp:39-108) ------------- */
/* detect_knee (roofline.cpp:39-76): farthest point from the chord of the unit-normalised
 * curve; confidence in [0, 1]. n >= 4 (else SGB_EINVAL). */
int sgb_detect_knee(const int* b, const double* s, int n, int* index, double* confidence);
/* measure_c_peak (roofline.cpp:78-108) with the reference CLI's latency_fn
 * (tools/sgrpo.cpp:38-49): a batched b-row target forward (EOS token, position 0, self-only
 * mask) on the engine's device, median of `reps` CUDA-event timings for b = 1..b_max.
 * curve_s (optional) receives the b_max median latencies in seconds. */
int sgb_measure_c_peak(sgb_engine* e, int b_max, int warmup, int reps, int* c_peak, double* confidence,
                       int* low_confidence, double* curve_s);

/* target_forward_calls() (include/sgrpo/tinylm.hpp:288-291): cumulative target forward
 * LAUNCHES of this engine (one per prefill chunk / decode step / forward_target call, not one
 * per sequence); the draft update never runs the target (SPEC acceptance criterion 10). */
int sgb_target_forward_calls(sgb_engine* e, long long* out);

/* GRPO rewards and advantages of the LAST rollout's groups, from its token table in HBM:
 * rewards[s] = compute_reward (src/grpo.cpp:99-116) of sequence s's response (tokens after
 * its prompt, scored against answers[s / g] = a + b of query s / g, call site grpo.cpp:352-363);
 * advantages = standardize_advantages (grpo.cpp:121-136) per group, valid[b] = 0 where the
 * reference returns nullopt (sd < eps_var; advantages 0). n_groups * g must equal the last
 * rollout's sequence count. */
int sgb_group_advantages(sgb_engine* e, const long long* answers, int n_groups, int g, double eps_var,
                         double* rewards, double* advantages, int* valid);

/* Data-parallel group-reward/advantage gather (north star: NCCL where the path shards):
 * recv[r * n + i] = rank r's send[i] (ncclAllGather over the engine's communicator). */
int sgb_allgather_f64(sgb_engine* e, const double* send, int n, double* recv);

#ifdef __cplusplus
}
#endif

#endif /* SGRPO_B200_H */
