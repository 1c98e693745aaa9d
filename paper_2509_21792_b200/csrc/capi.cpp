// The drop-in boundary: extern "C" entry points declared in include/sgrpo_b200.h.
// Each translates exceptions to the status codes of util.h and records a thread-local
// message (sgb_last_error), mirroring the reference's exception types
// (SURVEY.md §8b). There is no CPU fallback: every compute entry point runs CUDA.
#include <cuda_bf16.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <cstdio>
#include <fcntl.h>
#include <sys/stat.h>
#include <sys/mman.h>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include <nccl.h>

#include "sgrpo_b200.h"
#include "engine.h"
#include "gemm.h"
#include "kernels.h"
#include "util.h"

struct sgb_engine {
    std::unique_ptr<sgb::Engine> eng;
    sgb_model_config cfg{};  // as created (checkpoint headers carry it)
    int draft_layers = 1;
    std::vector<int> last_events;  // (step, seq, accepted) of the last rollout
    double last_prefill_s = 0;
    std::vector<double> last_bytes, last_flops, last_secs;  // per-step algorithmic work + device time
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return sgb::SGB_OK;
    } catch (const sgb::CudaError& e) {
        g_err = e.what();
        return sgb::SGB_ECUDA;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return sgb::SGB_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return sgb::SGB_ERANGE;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return sgb::SGB_EDOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return sgb::SGB_ERUNTIME;
    }
}

sgb::Engine& E(sgb_engine* e) {
    if (!e || !e->eng) throw std::invalid_argument("null engine");
    return *e->eng;
}
}  // namespace

// ---------------------------------------------------------------- data parallel (NCCL)
namespace {
struct DpGroup {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    double* dbuf = nullptr;
};
std::unordered_map<const sgb_engine*, DpGroup>& groups() {
    static std::unordered_map<const sgb_engine*, DpGroup> g;
    return g;
}
void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}
// NCCL prints a version banner on stdout at its first call (also at NCCL_DEBUG=WARN); callers
// (bench.py) keep stdout for their own output, so NCCL's setup calls run with fd 1 pointed at
// stderr.
struct StdoutToStderr {
    int saved = -1;
    StdoutToStderr() {
        fflush(stdout);
        saved = dup(1);
        if (saved >= 0) dup2(2, 1);
    }
    ~StdoutToStderr() {
        fflush(stdout);
        if (saved >= 0) {
            dup2(saved, 1);
            close(saved);
        }
    }
};

DpGroup& group_of(sgb_engine* e) {
    auto it = groups().find(e);
    if (it == groups().end() || !it->second.comm) throw std::invalid_argument("engine has no NCCL group (sgb_nccl_init)");
    return it->second;
}
// gradient all-reduce hook run by draft_update before the AdamW step (C1)
void grad_allreduce_hook(float* g, size_t n, cudaStream_t st, void* ctx) {
    DpGroup* dg = static_cast<DpGroup*>(ctx);
    nccl_check(ncclAllReduce(g, g, n, ncclFloat, ncclSum, dg->comm, st), "ncclAllReduce(grad)");
}
}  // namespace

template <class T>
void allreduce_host(sgb_engine* e, T* vals, int n, ncclDataType_t type) {
    DpGroup& g = group_of(e);
    if (n < 0 || static_cast<size_t>(n) * sizeof(T) > 4096 * sizeof(double)) throw std::invalid_argument("allreduce size");
    cudaStream_t st = E(e).stream();
    SGB_CUDA(cudaMemcpyAsync(g.dbuf, vals, n * sizeof(T), cudaMemcpyHostToDevice, st));
    nccl_check(ncclAllReduce(g.dbuf, g.dbuf, n, type, ncclSum, g.comm, st), "ncclAllReduce");
    SGB_CUDA(cudaMemcpyAsync(vals, g.dbuf, n * sizeof(T), cudaMemcpyDeviceToHost, st));
    SGB_CUDA(cudaStreamSynchronize(st));
}

extern "C" {

const char* sgb_last_error(void) { return g_err.c_str(); }

int sgb_version(void) { return SGB_ABI_VERSION; }

int sgb_device_count(int* out) {
    return guarded([&] { SGB_CUDA(cudaGetDeviceCount(out)); });
}

int sgb_engine_create(const sgb_model_config* c, int draft_layers, int device, int max_seqs, int max_rows, int k_max,
                      int l_max, sgb_engine** out) {
    return guarded([&] {
        if (!c || !out) throw std::invalid_argument("null argument");
        sgb::ModelDims d;
        d.vocab = c->vocab_size;
        d.d = c->d_model;
        d.layers = c->n_layers;
        d.heads = c->n_heads;
        d.dff = c->d_ff;
        d.max_seq = c->max_seq_len;
        auto* h = new sgb_engine;
        try {
            h->eng = std::make_unique<sgb::Engine>(d, draft_layers, device, max_seqs, max_rows, k_max, l_max);
            h->cfg = *c;
            h->draft_layers = draft_layers;
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int sgb_engine_destroy(sgb_engine* e) {
    return guarded([&] {
        auto it = groups().find(e);
        if (it != groups().end()) {
            if (it->second.comm) ncclCommDestroy(it->second.comm);
            if (it->second.dbuf) cudaFree(it->second.dbuf);
            groups().erase(it);
        }
        delete e;
    });
}

int sgb_param_counts(sgb_engine* e, size_t* target, size_t* draft) {
    return guarded([&] {
        *target = E(e).target_param_count();
        *draft = E(e).draft_param_count();
    });
}

int sgb_upload_target(sgb_engine* e, const float* flat, size_t n) {
    return guarded([&] { E(e).upload_target(flat, n); });
}
int sgb_upload_draft(sgb_engine* e, const float* flat, size_t n) {
    return guarded([&] { E(e).upload_draft(flat, n); });
}
int sgb_download_draft(sgb_engine* e, float* flat, size_t n) {
    return guarded([&] { E(e).download_draft(flat, n); });
}
int sgb_init_random(sgb_engine* e, unsigned long long seed) {
    return guarded([&] { E(e).init_random(seed); });
}

int sgb_cache_reset(sgb_engine* e, int slot, int draft) {
    return guarded([&] { E(e).cache_reset(slot, draft != 0); });
}
int sgb_cache_len(sgb_engine* e, int slot, int draft, int* out) {
    return guarded([&] { *out = E(e).cache_len(slot, draft != 0); });
}
int sgb_cache_read(sgb_engine* e, int slot, int draft, float* k, float* v) {
    return guarded([&] { E(e).cache_read(slot, draft != 0, k, v); });
}
int sgb_cache_gather_tail(sgb_engine* e, int slot, int base, const int* keep, int n) {
    return guarded([&] { E(e).cache_gather_tail(slot, base, keep, n); });
}

int sgb_forward_target(sgb_engine* e, int slot, const int* tokens, const int* positions, int rows,
                       const unsigned char* mask, float* logits, float* hidden) {
    return guarded([&] { E(e).forward_target(slot, tokens, positions, rows, mask, logits, hidden); });
}

int sgb_forward_draft_rows(sgb_engine* e, int slot, const int* tokens, const float* prev_features,
                           const int* positions, int rows, int extend_cache, float* features, float* logits) {
    return guarded(
        [&] { E(e).forward_draft(slot, tokens, prev_features, positions, rows, extend_cache != 0, features, logits); });
}

int sgb_sample_rows(sgb_engine* e, const float* logits, int rows, int vocab, double temperature,
                    const unsigned long long* seeds, const int* key_pos, int* out) {
    return guarded([&] { E(e).emit(logits, rows, vocab, temperature, seeds, key_pos, out); });
}

int sgb_sample_rows_u(sgb_engine* e, const float* logits, int rows, int vocab, double temperature,
                      const double* uniforms, int* out, int* exact_rows) {
    return guarded([&] {
        if (!uniforms) throw std::invalid_argument("sample_rows_u: uniforms required");
        E(e).emit(logits, rows, vocab, temperature, nullptr, nullptr, out, uniforms, exact_rows);
    });
}

int sgb_debug_spec_sample(sgb_engine* e, const float* p_logits, const float* q_logits, int vocab, int k,
                          double temperature, int n_trials, unsigned long long seed, int* out_tok, int* out_acc) {
    return guarded([&] {
        E(e);
        if (vocab <= 0 || n_trials <= 0) throw std::invalid_argument("debug_spec_sample: empty input");
        if (!(temperature > 0)) throw std::invalid_argument("rejection sampling needs temperature > 0");
        const size_t V = vocab;
        float *dp = nullptr, *dq = nullptr, *dr = nullptr;
        int *dt = nullptr, *da = nullptr;
        SGB_CUDA(cudaMalloc(&dp, V * 4));
        SGB_CUDA(cudaMalloc(&dq, V * 4));
        SGB_CUDA(cudaMalloc(&dr, V * 4 * static_cast<size_t>(n_trials)));
        SGB_CUDA(cudaMalloc(&dt, 4 * static_cast<size_t>(n_trials)));
        SGB_CUDA(cudaMalloc(&da, 4 * static_cast<size_t>(n_trials)));
        SGB_CUDA(cudaMemcpy(dp, p_logits, V * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dq, q_logits, V * 4, cudaMemcpyHostToDevice));
        sgb::launch_debug_spec_sample(dp, dq, vocab, k, temperature, n_trials, seed, dr, dt, da, nullptr);
        SGB_CUDA(cudaMemcpy(out_tok, dt, 4 * static_cast<size_t>(n_trials), cudaMemcpyDeviceToHost));
        SGB_CUDA(cudaMemcpy(out_acc, da, 4 * static_cast<size_t>(n_trials), cudaMemcpyDeviceToHost));
        for (void* x : {static_cast<void*>(dp), static_cast<void*>(dq), static_cast<void*>(dr), static_cast<void*>(dt),
                        static_cast<void*>(da)})
            cudaFree(x);
    });
}

int sgb_exact_draws(sgb_engine* e, unsigned long long* out) {
    return guarded([&] { *out = E(e).exact_draws(); });
}

int sgb_debug_exp(sgb_engine* e, const double* x, size_t n, double* out) {
    return guarded([&] { E(e).debug_exp(x, n, out); });
}

int sgb_topk_logsoftmax(sgb_engine* e, const float* logits, int rows, int vocab, int k, int* tokens,
                        double* log_probs) {
    return guarded([&] { E(e).topk_logsoftmax(logits, rows, vocab, k, tokens, log_probs); });
}

int sgb_build_tree(sgb_engine* e, int root_token, int k_draft, int l_draft, int n_verify, sgb_logits_fn fn,
                   void* ctx, int cap, int* tok, int* par, int* dep, double* lp, double* conf, int* n_nodes, int* sel,
                   int* n_sel, unsigned char* mask) {
    return guarded([&] {
        auto t = E(e).debug_tree_cb(root_token, k_draft, l_draft, n_verify, fn, ctx);
        const int n = static_cast<int>(t.tok.size());
        if (n > cap) throw std::invalid_argument("build_tree: capacity");
        std::copy(t.tok.begin(), t.tok.end(), tok);
        std::copy(t.par.begin(), t.par.end(), par);
        std::copy(t.dep.begin(), t.dep.end(), dep);
        std::copy(t.lp.begin(), t.lp.end(), lp);
        std::copy(t.conf.begin(), t.conf.end(), conf);
        std::copy(t.sel.begin(), t.sel.end(), sel);
        if (mask) std::copy(t.mask.begin(), t.mask.end(), mask);
        *n_nodes = n;
        *n_sel = static_cast<int>(t.sel.size());
    });
}

int sgb_rollout(sgb_engine* e, const int* prompts, const int* prompt_lens, int n_prompts, int g,
                const sgb_gen_options* opt, int* tokens, int* lens, int* prompt_len, int* hit_eos, float* features,
                int* step_rec, int step_cap, sgb_rollout_stats* stats) {
    return guarded([&] {
        sgb::Engine& en = E(e);
        if (!opt) throw std::invalid_argument("null options");
        if (n_prompts < 0) throw std::invalid_argument("generate: negative prompt count");
        sgb::RolloutArgs a;
        size_t off = 0;
        for (int i = 0; i < n_prompts; ++i) {
            if (prompt_lens[i] < 0) throw std::invalid_argument("generate: negative prompt length");
            a.prompts.emplace_back(prompts + off, prompts + off + prompt_lens[i]);
            off += prompt_lens[i];
        }
        a.g = g;
        a.alpha = opt->alpha;
        a.k_max = opt->k_max;
        a.l_max = opt->l_max;
        a.c_peak = opt->c_peak;
        a.mode = opt->mode;
        if (a.mode < 0 || a.mode > 2) throw std::invalid_argument("unknown decode mode");
        a.early_term = opt->early_term != 0;
        a.temperature = opt->temperature;
        a.seed = opt->seed;
        a.max_new_tokens = opt->max_new_tokens;
        a.fixed = sgb::SpecCfg{opt->fixed_n_verify, opt->fixed_k_draft, opt->fixed_l_draft};
        if (opt->seq_max_new) a.seq_max_new.assign(opt->seq_max_new, opt->seq_max_new + n_prompts * g);
        a.want_features = features != nullptr && opt->want_features;
        a.sid_offset = opt->sid_offset;
        a.acceptance = opt->acceptance;
        if (a.want_features) a.features_out = features;
        sgb::RolloutResult r = en.rollout(a);
        e->last_events = r.events;
        e->last_prefill_s = r.prefill_seconds;
        e->last_bytes = r.step_bytes;
        e->last_flops = r.step_flops;
        e->last_secs = r.step_seconds;
        const int T = en.dims().max_seq;
        const int ns = static_cast<int>(r.tokens.size());
        for (int s = 0; s < ns; ++s) {
            if (tokens) std::copy(r.tokens[s].begin(), r.tokens[s].end(), tokens + static_cast<size_t>(s) * T);
            if (lens) lens[s] = static_cast<int>(r.tokens[s].size());
            if (prompt_len) prompt_len[s] = r.prompt_len[s];
            if (hit_eos) hit_eos[s] = r.hit_eos[s];
        }
        if (step_rec) {
            const int n = std::min(step_cap, static_cast<int>(r.steps.size()));
            for (int i = 0; i < n; ++i) {
                step_rec[5 * i] = r.steps[i].b_cur;
                step_rec[5 * i + 1] = r.steps[i].n_verify;
                step_rec[5 * i + 2] = r.steps[i].k_draft;
                step_rec[5 * i + 3] = r.steps[i].l_draft;
                step_rec[5 * i + 4] = r.steps[i].accepted;
                if (opt->step_seconds) opt->step_seconds[i] = r.step_seconds[i];
            }
        }
        if (stats) {
            stats->total_accepted = r.total_accepted;
            stats->total_verify_slots = r.total_verify_slots;
            stats->n_steps = static_cast<int>(r.steps.size());
            stats->target_forwards = r.target_forwards;
            stats->draft_forwards = r.draft_forwards;
            stats->kernel_launches = r.kernel_launches;
            stats->seconds = r.seconds;
            stats->h2d_bytes = r.h2d_bytes;
            stats->d2h_bytes = r.d2h_bytes;
            stats->host_gap_seconds = r.host_gap_seconds;
            stats->host_enqueue_seconds = r.host_enqueue_seconds;
        }
    });
}


int sgb_nccl_unique_id(unsigned char* id128) {
    return guarded([&] {
        ncclUniqueId id;
        {
            StdoutToStderr guard;
            nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
        }
        static_assert(sizeof(id) == 128, "NCCL unique id size");
        std::memcpy(id128, &id, 128);
    });
}

int sgb_nccl_init(sgb_engine* e, int rank, int world, const unsigned char* id128) {
    return guarded([&] {
        E(e);
        ncclUniqueId id;
        std::memcpy(&id, id128, 128);
        DpGroup g;
        g.rank = rank;
        g.world = world;
        {
            StdoutToStderr guard;
            nccl_check(ncclCommInitRank(&g.comm, world, id, rank), "ncclCommInitRank");
        }
        SGB_CUDA(cudaMalloc(&g.dbuf, 4096 * sizeof(double)));
        groups()[e] = g;
    });
}


int sgb_target_forward_calls(sgb_engine* e, long long* out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("target_forward_calls: null output");
        *out = E(e).target_forward_calls();
    });
}

int sgb_group_advantages(sgb_engine* e, const long long* answers, int n_groups, int g, double eps_var,
                         double* rewards, double* advantages, int* valid) {
    return guarded([&] {
        if (!answers || !rewards || !advantages || !valid) throw std::invalid_argument("group_advantages: null output");
        E(e).group_advantages(answers, n_groups, g, eps_var, rewards, advantages, valid);
    });
}

int sgb_debug_group_advantages(const int* tokens, const int* lens, const int* prompt_lens, int n_groups, int g,
                               int stride, const long long* answers, double eps_var, double* rewards,
                               double* advantages, int* valid) {
    return guarded([&] {
        if (n_groups <= 0 || g < 2) throw std::invalid_argument("standardize_advantages: need G >= 2");
        const int n = n_groups * g;
        for (int s = 0; s < n; ++s)
            if (lens[s] < prompt_lens[s] || lens[s] > stride || prompt_lens[s] < 0)
                throw std::invalid_argument("group_advantages: bad sequence lengths");
        int *dt = nullptr, *dl = nullptr, *dp = nullptr, *dv = nullptr;
        long long* da = nullptr;
        double* db = nullptr;
        SGB_CUDA(cudaMalloc(&dt, sizeof(int) * static_cast<size_t>(n) * stride));
        SGB_CUDA(cudaMalloc(&dl, sizeof(int) * n));
        SGB_CUDA(cudaMalloc(&dp, sizeof(int) * n));
        SGB_CUDA(cudaMalloc(&dv, sizeof(int) * n_groups));
        SGB_CUDA(cudaMalloc(&da, sizeof(long long) * n_groups));
        SGB_CUDA(cudaMalloc(&db, sizeof(double) * 2 * n));
        SGB_CUDA(cudaMemcpy(dt, tokens, sizeof(int) * static_cast<size_t>(n) * stride, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dl, lens, sizeof(int) * n, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dp, prompt_lens, sizeof(int) * n, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(da, answers, sizeof(long long) * n_groups, cudaMemcpyHostToDevice));
        sgb::launch_group_advantages(n_groups, g, dt, stride, dl, dp, da, eps_var, db, db + n, dv, 0);
        SGB_CUDA(cudaDeviceSynchronize());
        SGB_CUDA(cudaMemcpy(rewards, db, sizeof(double) * n, cudaMemcpyDeviceToHost));
        SGB_CUDA(cudaMemcpy(advantages, db + n, sizeof(double) * n, cudaMemcpyDeviceToHost));
        SGB_CUDA(cudaMemcpy(valid, dv, sizeof(int) * n_groups, cudaMemcpyDeviceToHost));
        void* ptrs[] = {dt, dl, dp, dv, da, db};
        for (void* p : ptrs) cudaFree(p);
    });
}

int sgb_allgather_f64(sgb_engine* e, const double* send, int n, double* recv) {
    return guarded([&] {
        DpGroup& g = group_of(e);
        if (n < 0 || !send || !recv) throw std::invalid_argument("allgather: bad arguments");
        cudaStream_t st = E(e).stream();
        const size_t need = static_cast<size_t>(n) * (g.world + 1);
        double* d = g.dbuf;  // the group's 4096-double staging buffer when it fits
        if (need > 4096) SGB_CUDA(cudaMalloc(&d, sizeof(double) * need));
        SGB_CUDA(cudaMemcpyAsync(d, send, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        nccl_check(ncclAllGather(d, d + n, n, ncclFloat64, g.comm, st), "ncclAllGather");
        SGB_CUDA(cudaMemcpyAsync(recv, d + n, sizeof(double) * static_cast<size_t>(n) * g.world, cudaMemcpyDeviceToHost, st));
        SGB_CUDA(cudaStreamSynchronize(st));
        if (d != g.dbuf) SGB_CUDA(cudaFree(d));
    });
}

int sgb_allreduce_sum_f64(sgb_engine* e, double* vals, int n) {
    return guarded([&] { allreduce_host(e, vals, n, ncclFloat64); });
}
int sgb_allreduce_sum_i64(sgb_engine* e, long long* vals, int n) {
    return guarded([&] { allreduce_host(e, vals, n, ncclInt64); });
}

static sgb::Engine::DraftUpdateArgs draft_args(const sgb_adamw* o, float* grad_out) {
    if (!o) throw std::invalid_argument("null AdamW options");
    sgb::Engine::DraftUpdateArgs a;
    a.lr = o->lr;
    a.beta1 = o->beta1;
    a.beta2 = o->beta2;
    a.eps = o->eps;
    a.weight_decay = o->weight_decay;
    a.w_feat = o->w_feat;
    a.w_tok = o->w_tok;
    a.rows_total = o->rows_total;
    a.apply_step = o->apply_step != 0;
    a.grad_out = grad_out;
    return a;
}

static void fill_terms(const sgb::Engine::DraftLossTerms& t, sgb_draft_terms* out) {
    if (!out) return;
    out->feature_loss = t.feature_loss;
    out->token_loss = t.token_loss;
    out->total = t.total;
    out->rows = t.rows;
    out->seconds = t.seconds;
}

int sgb_draft_update(sgb_engine* e, int n_seqs, const int* tokens, const int* lens, const float* features,
                     const sgb_adamw* opt, float* grad_out, sgb_draft_terms* terms) {
    return guarded([&] {
        auto a = draft_args(opt, grad_out);
        if (opt->allreduce_grad) {
            a.grad_hook = grad_allreduce_hook;
            a.hook_ctx = &group_of(e);
        }
        a.n_seqs = n_seqs;
        a.tokens = tokens;
        a.lens = lens;
        a.features = features;
        fill_terms(E(e).draft_update(a), terms);
    });
}

int sgb_policy_enable(sgb_engine* e) {
    return guarded([&] { E(e).policy_enable(); });
}

int sgb_download_target(sgb_engine* e, float* flat, size_t n) {
    return guarded([&] { E(e).download_target(flat, n); });
}

int sgb_policy_update(sgb_engine* e, int n_seqs, const int* tokens, const int* lens, const int* prompt_lens,
                      const double* weights, const sgb_adamw* opt, float* grad_out, sgb_policy_terms* terms) {
    return guarded([&] {
        if (!opt) throw std::invalid_argument("null AdamW options");
        if (n_seqs < 0 || (n_seqs > 0 && (!tokens || !lens || !prompt_lens || !weights)))
            throw std::invalid_argument("policy_update: null sequence arrays");
        sgb::Engine::PolicyArgs a;
        a.n_seqs = n_seqs;
        a.tokens = tokens;
        a.lens = lens;
        a.prompt_lens = prompt_lens;
        a.weights = weights;
        a.lr = opt->lr;
        a.beta1 = opt->beta1;
        a.beta2 = opt->beta2;
        a.eps = opt->eps;
        a.weight_decay = opt->weight_decay;
        a.tokens_total = opt->rows_total;
        a.apply_step = opt->apply_step != 0;
        a.grad_out = grad_out;
        if (opt->allreduce_grad) {
            a.grad_hook = grad_allreduce_hook;
            a.hook_ctx = &group_of(e);
        }
        const auto t = E(e).policy_update(a);
        if (terms) {
            terms->loss = t.loss;
            terms->tokens = t.tokens;
            terms->rows = t.rows;
            terms->seconds = t.seconds;
            terms->skipped = t.skipped ? 1 : 0;
        }
    });
}

int sgb_policy_adamw_state(sgb_engine* e, float* m, float* v, long long* t, int upload) {
    return guarded([&] { E(e).policy_adamw_state(m, v, t, upload != 0); });
}

int sgb_draft_update_last(sgb_engine* e, const sgb_adamw* opt, float* grad_out, sgb_draft_terms* terms) {
    return guarded([&] {
        auto a = draft_args(opt, grad_out);
        if (opt->allreduce_grad) {
            a.grad_hook = grad_allreduce_hook;
            a.hook_ctx = &group_of(e);
        }
        a.use_last_rollout = true;
        fill_terms(E(e).draft_update(a), terms);
    });
}

// ---- C_peak calibration (roofline.cpp:39-108) -------------------------------------------
namespace {
// detect_knee: normalise both axes to the unit box, take the point farthest from the chord
// joining the first and last points; confidence = distance / (sqrt(2)/2).
void knee_of(const int* b, const double* s, int n, int* index, double* confidence) {
    if (n < 4) throw std::invalid_argument("detect_knee: need at least 4 points");
    double xmin = b[0], xmax = b[0], ymin = s[0], ymax = s[0];
    for (int i = 0; i < n; ++i) {
        xmin = std::min(xmin, static_cast<double>(b[i]));
        xmax = std::max(xmax, static_cast<double>(b[i]));
        ymin = std::min(ymin, s[i]);
        ymax = std::max(ymax, s[i]);
    }
    const double xspan = xmax > xmin ? xmax - xmin : 1.0;
    const double yspan = ymax > ymin ? ymax - ymin : 1.0;
    auto nx = [&](int i) { return (b[i] - xmin) / xspan; };
    auto ny = [&](int i) { return (s[i] - ymin) / yspan; };
    const double x0 = nx(0), y0 = ny(0), x1 = nx(n - 1), y1 = ny(n - 1);
    const double cx = x1 - x0, cy = y1 - y0;
    const double clen = std::sqrt(cx * cx + cy * cy);
    double best = -1;
    int bi = 0;
    for (int i = 0; i < n; ++i) {
        double dist;
        if (clen == 0) {
            const double dx = nx(i) - x0, dy = ny(i) - y0;
            dist = std::sqrt(dx * dx + dy * dy);
        } else {
            dist = std::abs(cx * (ny(i) - y0) - cy * (nx(i) - x0)) / clen;
        }
        if (dist > best) {
            best = dist;
            bi = i;
        }
    }
    *index = bi;
    *confidence = std::clamp(best / 0.7071067811865476, 0.0, 1.0);
}
}  // namespace

int sgb_detect_knee(const int* b, const double* s, int n, int* index, double* confidence) {
    return guarded([&] { knee_of(b, s, n, index, confidence); });
}

int sgb_measure_c_peak(sgb_engine* e, int b_max, int warmup, int reps, int* c_peak, double* confidence,
                       int* low_confidence, double* curve_s) {
    return guarded([&] {
        if (b_max < 4) throw std::invalid_argument("measure_c_peak: b_max must be >= 4");
        if (reps < 1) throw std::invalid_argument("measure_c_peak: reps must be >= 1");
        std::vector<int> bs(b_max);
        std::vector<double> ss(b_max);
        for (int b = 1; b <= b_max; ++b) {
            bs[b - 1] = b;
            ss[b - 1] = E(e).latency_probe(b, warmup, reps);
        }
        // non-monotone noise beyond 2% lowers confidence in the knee
        bool low = false;
        for (int i = 1; i < b_max; ++i)
            if (ss[i] < ss[i - 1] * (1.0 - 0.02)) low = true;
        int idx = 0;
        double conf = 0;
        knee_of(bs.data(), ss.data(), b_max, &idx, &conf);
        *confidence = conf;
        if (conf < 0.05) {  // no detectable knee: fall back to b_max
            *c_peak = b_max;
            low = true;
        } else {
            *c_peak = bs[idx];
        }
        *low_confidence = low ? 1 : 0;
        if (curve_s)
            for (int i = 0; i < b_max; ++i) curve_s[i] = ss[i];
    });
}

// ---- SGRPOCK1 checkpoints (src/tinylm.cpp:14-105) ------------------------------------------
// Layout: "SGRPOCK1" | u32 header length | JSON header | param_count little-endian fp32.
// The header is the reference's nlohmann::json dump (keys sorted):
//   {"config":{"d_ff":..,"d_model":..,"max_seq_len":..,"n_heads":..,"n_layers":..,"seed":..,
//    "vocab_size":..},["draft_layers":..,]"kind":"target"|"draft","param_count":..}
namespace {
struct CkptHeader {
    int kind = -1;  // 0 target, 1 draft
    sgb_model_config cfg{};
    int draft_layers = 0;
    size_t param_count = 0;
    size_t data_off = 0;
};

long long json_int(const std::string& h, const char* key) {
    const std::string k = std::string("\"") + key + "\":";
    const size_t p = h.find(k);
    if (p == std::string::npos) throw std::runtime_error(std::string("checkpoint header lacks ") + key);
    return std::stoll(h.substr(p + k.size()));
}

CkptHeader read_header(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open checkpoint: " + path);
    char magic[8];
    uint32_t hl = 0;
    const bool ok = std::fread(magic, 1, 8, f) == 8 && std::memcmp(magic, "SGRPOCK1", 8) == 0 &&
                    std::fread(&hl, 4, 1, f) == 1;
    std::string h(hl, '\0');
    const bool ok2 = ok && std::fread(&h[0], 1, hl, f) == hl;
    std::fclose(f);
    if (!ok) throw std::runtime_error("bad checkpoint magic: " + path);
    if (!ok2) throw std::runtime_error("truncated checkpoint: " + path);
    CkptHeader c;
    const size_t kp = h.find("\"kind\":\"");
    if (kp == std::string::npos) throw std::runtime_error("checkpoint header lacks kind");
    const std::string kind = h.substr(kp + 8, h.find('"', kp + 8) - (kp + 8));
    if (kind == "target") c.kind = 0;
    else if (kind == "draft") c.kind = 1;
    else throw std::runtime_error("unknown checkpoint kind: " + kind);
    c.cfg.vocab_size = static_cast<int>(json_int(h, "vocab_size"));
    c.cfg.d_model = static_cast<int>(json_int(h, "d_model"));
    c.cfg.n_layers = static_cast<int>(json_int(h, "n_layers"));
    c.cfg.n_heads = static_cast<int>(json_int(h, "n_heads"));
    c.cfg.d_ff = static_cast<int>(json_int(h, "d_ff"));
    c.cfg.max_seq_len = static_cast<int>(json_int(h, "max_seq_len"));
    c.cfg.seed = static_cast<unsigned long long>(json_int(h, "seed"));
    c.draft_layers = c.kind == 1 ? static_cast<int>(json_int(h, "draft_layers")) : 0;
    c.param_count = static_cast<size_t>(json_int(h, "param_count"));
    c.data_off = 12 + hl;
    return c;
}

bool same_shape(const sgb_model_config& a, const sgb_model_config& b) {
    return a.vocab_size == b.vocab_size && a.d_model == b.d_model && a.n_layers == b.n_layers &&
           a.n_heads == b.n_heads && a.d_ff == b.d_ff && a.max_seq_len == b.max_seq_len;
}
}  // namespace

int sgb_checkpoint_info(const char* path, int* kind, sgb_model_config* cfg, int* draft_layers, size_t* param_count) {
    return guarded([&] {
        const CkptHeader c = read_header(path);
        if (kind) *kind = c.kind;
        if (cfg) *cfg = c.cfg;
        if (draft_layers) *draft_layers = c.draft_layers;
        if (param_count) *param_count = c.param_count;
    });
}

int sgb_load_checkpoint(sgb_engine* e, const char* path, int* kind_out) {
    return guarded([&] {
        E(e);
        const CkptHeader c = read_header(path);
        if (!same_shape(c.cfg, e->cfg)) throw std::invalid_argument("checkpoint config does not match the engine");
        if (c.kind == 1 && c.draft_layers != e->draft_layers)
            throw std::invalid_argument("checkpoint draft_layers does not match the engine");
        const size_t nt = E(e).target_param_count(), nd = E(e).draft_param_count();
        if (c.param_count != (c.kind == 0 ? nt : nd)) throw std::runtime_error("checkpoint param count mismatch");
        // the payload is mapped, not copied: upload reads it straight from the page cache
        const int fd = open(path, O_RDONLY);
        if (fd < 0) throw std::runtime_error(std::string("cannot open checkpoint: ") + path);
        const size_t bytes = c.data_off + c.param_count * sizeof(float);
        struct stat stt;
        if (fstat(fd, &stt) != 0 || static_cast<size_t>(stt.st_size) < bytes) {
            close(fd);
            throw std::runtime_error(std::string("truncated checkpoint: ") + path);
        }
        void* m = mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE, fd, 0);
        close(fd);
        if (m == MAP_FAILED) throw std::runtime_error("mmap failed for checkpoint");
        const float* flat = reinterpret_cast<const float*>(static_cast<const char*>(m) + c.data_off);
        try {
            if (c.kind == 0) E(e).upload_target(flat, c.param_count);
            else E(e).upload_draft(flat, c.param_count);
        } catch (...) {
            munmap(m, bytes);
            throw;
        }
        munmap(m, bytes);
        if (kind_out) *kind_out = c.kind;
    });
}

int sgb_save_draft_checkpoint(sgb_engine* e, const char* path) {
    return guarded([&] {
        const size_t nd = E(e).draft_param_count();
        std::vector<float> flat(nd);
        E(e).download_draft(flat.data(), nd);
        const sgb_model_config& c = e->cfg;
        const std::string h = "{\"config\":{\"d_ff\":" + std::to_string(c.d_ff) + ",\"d_model\":" +
                              std::to_string(c.d_model) + ",\"max_seq_len\":" + std::to_string(c.max_seq_len) +
                              ",\"n_heads\":" + std::to_string(c.n_heads) + ",\"n_layers\":" +
                              std::to_string(c.n_layers) + ",\"seed\":" + std::to_string(c.seed) +
                              ",\"vocab_size\":" + std::to_string(c.vocab_size) + "},\"draft_layers\":" +
                              std::to_string(e->draft_layers) + ",\"kind\":\"draft\",\"param_count\":" +
                              std::to_string(nd) + "}";
        FILE* f = std::fopen(path, "wb");
        if (!f) throw std::runtime_error(std::string("cannot open checkpoint for writing: ") + path);
        const uint32_t hl = static_cast<uint32_t>(h.size());
        bool ok = std::fwrite("SGRPOCK1", 1, 8, f) == 8 && std::fwrite(&hl, 4, 1, f) == 1 &&
                  std::fwrite(h.data(), 1, hl, f) == hl && std::fwrite(flat.data(), 4, nd, f) == nd;
        ok = (std::fclose(f) == 0) && ok;
        if (!ok) throw std::runtime_error(std::string("checkpoint write failed: ") + path);
    });
}

int sgb_adamw_state(sgb_engine* e, float* m, float* v, long long* t, int upload) {
    return guarded([&] { E(e).adamw_state(m, v, t, upload != 0); });
}

int sgb_rollout_events(sgb_engine* e, int* triples, long long cap, long long* n, double* prefill_seconds) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("null engine");
        const long long m = static_cast<long long>(e->last_events.size() / 3);
        if (n) *n = m;
        if (triples) std::copy(e->last_events.begin(), e->last_events.begin() + 3 * std::min(m, cap), triples);
        if (prefill_seconds) *prefill_seconds = e->last_prefill_s;
    });
}

int sgb_rollout_roofline(sgb_engine* e, double* bytes, double* flops, double* seconds, long long cap, long long* n) {
    return guarded([&] {
        if (!e) throw std::invalid_argument("null engine");
        const long long m = static_cast<long long>(e->last_bytes.size());
        if (n) *n = m;
        const long long k = std::min(m, cap);
        if (bytes) std::copy(e->last_bytes.begin(), e->last_bytes.begin() + k, bytes);
        if (flops) std::copy(e->last_flops.begin(), e->last_flops.begin() + k, flops);
        if (seconds) std::copy(e->last_secs.begin(), e->last_secs.begin() + std::min<long long>(k, e->last_secs.size()), seconds);
    });
}

int sgb_adamw_reset(sgb_engine* e) {
    return guarded([&] { E(e).adamw_reset(); });
}

// GEMM microbenchmark: device-resident random bf16 operands, fused fp32 epilogue,
// average device ms over `iters` launches (CUDA events on the launching stream).
int sgb_bench_gemm(int M, int N, int K, int splits, int iters, double* ms_out) {
    return guarded([&] {
        const int cap = ((M + 255) / 256) * 256;
        // Weights rotate over enough copies to exceed the 126 MB L2, so every launch streams
        // its weights from HBM as in the rollout (28 layers x 74 MB at the c2 shape).
        const size_t wbytes = static_cast<size_t>(N) * K * 2;
        const int ncopy = static_cast<int>(std::max<size_t>(1, (320u << 20) / wbytes + 1));
        std::vector<__nv_bfloat16> hw(static_cast<size_t>(N) * K), hx(static_cast<size_t>(cap) * K);
        uint64_t st = 12345;
        auto rnd = [&]() {
            st = st * 6364136223846793005ULL + 1442695040888963407ULL;
            return static_cast<float>((st >> 40) & 0xFFFF) / 65536.0f - 0.5f;
        };
        for (auto& v : hw) v = __float2bfloat16(0.05f * rnd());
        for (auto& v : hx) v = __float2bfloat16(rnd());
        __nv_bfloat16 *dw = nullptr, *dx = nullptr;
        float* dp = nullptr;
        SGB_CUDA(cudaMalloc(&dw, wbytes * ncopy));
        SGB_CUDA(cudaMalloc(&dx, hx.size() * 2));
        for (int c = 0; c < ncopy; ++c)
            SGB_CUDA(cudaMemcpy(reinterpret_cast<char*>(dw) + c * wbytes, hw.data(), wbytes, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
        std::vector<sgb::GemmWeight> gw(ncopy);
        for (int c = 0; c < ncopy; ++c)
            gw[c].init(reinterpret_cast<const __nv_bfloat16*>(reinterpret_cast<const char*>(dw) + c * wbytes), N, K);
        sgb::GemmAct ga;
        ga.init(dx, cap, K);
        sgb::GemmWorkspace ws;
        ws.cap_floats = sgb::gemm_ws_floats(M, N, K);
        ws.ctr_cap = 1 << 16;
        SGB_CUDA(cudaMalloc(&ws.buf, ws.cap_floats * 4));
        SGB_CUDA(cudaMalloc(&ws.ctr, ws.ctr_cap * sizeof(int)));
        SGB_CUDA(cudaMemset(ws.ctr, 0, ws.ctr_cap * sizeof(int)));
        // splits < 0: kEpiPartials (raw chunk sums, one unit per (tile, chunk))
        const size_t out_floats = static_cast<size_t>(M) * N * (splits < 0 ? sgb::gemm_chunks(N, K) : 1);
        SGB_CUDA(cudaMalloc(&dp, out_floats * 4));
        sgb::GemmEpi epi;
        epi.kind = splits < 0 ? sgb::kEpiPartials : sgb::kEpiF32;
        epi.f32 = dp;
        epi.ld = N;
        if (splits < 0) splits = 0;
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 3; ++i) sgb::gemm_run(gw[i % ncopy], ga, M, epi, ws, 0, splits);
        SGB_CUDA(cudaEventRecord(a, 0));
        for (int i = 0; i < iters; ++i) sgb::gemm_run(gw[(i + 3) % ncopy], ga, M, epi, ws, 0, splits);
        SGB_CUDA(cudaEventRecord(b, 0));
        SGB_CUDA(cudaEventSynchronize(b));
        SGB_KCHECK();
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_out = ms / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(dw);
        cudaFree(dx);
        cudaFree(dp);
        cudaFree(ws.buf);
        cudaFree(ws.ctr);
    });
}

// Attention self-test: row r attends to n_keys[r] keys stored consecutively (rows
// concatenated) in K/V [sum n_keys][H*dh]; the LAST key of every row is addressed through
// the tree-path (chain) slot list, the rest as the contiguous cached prefix. out [B][H*dh].
int sgb_debug_attention(int B, const int* n_keys, int H, int dh, const float* q, const float* k, const float* v,
                        float* out) {
    return guarded([&] {
        if (B <= 0 || H <= 0 || dh <= 0) throw std::invalid_argument("debug_attention: bad shape");
        const int d = H * dh;
        std::vector<long long> base(B), chain(static_cast<size_t>(B) * sgb::kMaxChain, 0);
        std::vector<int> cl(B), chl(B, 1);
        long long tot = 0;
        int maxk = 1;
        double keys = 0;
        for (int b = 0; b < B; ++b) {
            if (n_keys[b] < 1) throw std::invalid_argument("debug_attention: rows need >= 1 key");
            base[b] = tot;
            cl[b] = n_keys[b] - 1;
            chain[static_cast<size_t>(b) * sgb::kMaxChain] = tot + n_keys[b] - 1;
            tot += n_keys[b];
            maxk = std::max(maxk, n_keys[b]);
            keys += n_keys[b];
        }
        std::vector<__nv_bfloat16> hk(tot * d), hv(tot * d);
        for (size_t i = 0; i < hk.size(); ++i) {
            hk[i] = __float2bfloat16(k[i]);
            hv[i] = __float2bfloat16(v[i]);
        }
        __nv_bfloat16 *K = nullptr, *V = nullptr, *o = nullptr;
        float *dq = nullptr, *pacc = nullptr, *pml = nullptr;
        long long *dbase = nullptr, *dchain = nullptr;
        int *dcl = nullptr, *dchl = nullptr;
        const int ns = sgb::attn_splits_for(maxk);
        SGB_CUDA(cudaMalloc(&K, hk.size() * 2));
        SGB_CUDA(cudaMalloc(&V, hv.size() * 2));
        SGB_CUDA(cudaMalloc(&o, static_cast<size_t>(B) * d * 2));
        SGB_CUDA(cudaMalloc(&dq, static_cast<size_t>(B) * d * 4));
        SGB_CUDA(cudaMalloc(&pacc, static_cast<size_t>(B) * d * ns * 4));
        SGB_CUDA(cudaMalloc(&pml, static_cast<size_t>(B) * H * ns * 2 * 4));
        SGB_CUDA(cudaMalloc(&dbase, B * 8));
        SGB_CUDA(cudaMalloc(&dchain, chain.size() * 8));
        SGB_CUDA(cudaMalloc(&dcl, B * 4));
        SGB_CUDA(cudaMalloc(&dchl, B * 4));
        SGB_CUDA(cudaMemcpy(K, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(V, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dq, q, static_cast<size_t>(B) * d * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), B * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), B * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), B * 4, cudaMemcpyHostToDevice));
        sgb::AttnRowsDev ar{dbase, dcl, dchl, dchain};
        sgb::AttnScratch sc{pacc, pml, nullptr, static_cast<long long>(B) * H};
        SGB_CUDA(cudaMalloc(&sc.row_ctr, sc.ctr_cap * 4));
        SGB_CUDA(cudaMemset(sc.row_ctr, 0, sc.ctr_cap * 4));
        sgb::launch_attention(dq, K, V, tot, ar, B, H, d, maxk, keys, sc, o, 0);
        SGB_CUDA(cudaDeviceSynchronize());
        std::vector<__nv_bfloat16> ho(static_cast<size_t>(B) * d);
        SGB_CUDA(cudaMemcpy(ho.data(), o, ho.size() * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < ho.size(); ++i) out[i] = __bfloat162float(ho[i]);
        void* ptrs[] = {K, V, o, dq, pacc, pml, dbase, dchain, dcl, dchl, sc.row_ctr};
        for (void* p : ptrs) cudaFree(p);
    });
}

namespace {
// Device state of a tree-attention case: n_groups sequences, each with ctx_len committed keys
// and a tree of rows (level order, parent within the group) -- the verify rows of one step.
struct TreeAttnCase {
    int M = 0, H = 0, d = 0, max_vlen = 1, n_tiles = 0, qw = 1;
    long long items = 0, n_slots = 0;
    double keys = 0;
    std::vector<void*> ptrs;
    __nv_bfloat16 *K = nullptr, *V = nullptr, *o1 = nullptr, *o2 = nullptr;
    float* q = nullptr;
    sgb::AttnRowsDev ar{};
    sgb::AttnScratch sc{};
    sgb::AttnTileDev* tiles = nullptr;
    std::vector<sgb::TreeGroupDev> tg;
    sgb::TreeGroupDev* dtg = nullptr;
    sgb::TreeTileDev* dtt = nullptr;
    int tw = 1, n_ttiles = 0, max_nodes = 1;
    CUtensorMap kmap, vmap;

    void* dev(size_t bytes) {
        void* p = nullptr;
        SGB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        ptrs.push_back(p);
        return p;
    }
    TreeAttnCase(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H_, int dh,
                 const float* hq, const float* kctx, const float* vctx, const float* knode, const float* vnode)
        : H(H_), d(H_ * dh) {
        if (n_groups <= 0 || H <= 0 || dh <= 0) throw std::invalid_argument("tree_attention: bad shape");
        long long n_ctx = 0;
        for (int g = 0; g < n_groups; ++g) {
            if (ctx_len[g] < 0 || n_rows[g] < 1) throw std::invalid_argument("tree_attention: bad group");
            n_ctx += ctx_len[g];
            M += n_rows[g];
        }
        // KV store: committed keys of every group, then one node slot per row
        const long long slots = n_ctx + M;
        n_slots = slots;
        std::vector<long long> base(M), chain(static_cast<size_t>(M) * sgb::kMaxChain, 0);
        std::vector<int> cl(M), chl(M);
        std::vector<sgb::AttnTileDev> ht;
        std::vector<std::array<int, 4>> groups;
        long long cbase = 0;
        int row = 0;
        for (int g = 0; g < n_groups; ++g) {
            const int r0 = row;
            std::vector<int> depth(n_rows[g]);
            int gmax = 1;
            for (int i = 0; i < n_rows[g]; ++i, ++row) {
                const int p = parent[row];
                if (i == 0 ? p != -1 : (p < 0 || p >= i)) throw std::invalid_argument("tree_attention: bad parent");
                depth[i] = i == 0 ? 0 : depth[p] + 1;
                if (depth[i] + 1 > sgb::kMaxChain) throw std::invalid_argument("tree_attention: tree too deep");
                base[row] = cbase;
                cl[row] = ctx_len[g];
                chl[row] = depth[i] + 1;
                for (int a = i; a >= 0; a = a == 0 ? -1 : parent[r0 + a])
                    chain[static_cast<size_t>(row) * sgb::kMaxChain + depth[a]] = n_ctx + r0 + a;
                gmax = std::max(gmax, ctx_len[g] + depth[i] + 1);
                keys += ctx_len[g] + depth[i] + 1;
            }
            max_vlen = std::max(max_vlen, gmax);
            groups.push_back({r0, n_rows[g], ctx_len[g], gmax});
            cbase += ctx_len[g];
        }
        qw = sgb::attn_tile_qw(groups);
        items = sgb::build_attn_tiles(groups, ht, qw, true);
        n_tiles = static_cast<int>(ht.size());
        const int ns = sgb::attn_splits_for(max_vlen);
        K = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(slots) * d * 2));
        V = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(slots) * d * 2));
        o1 = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(M) * d * 2));
        o2 = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(M) * d * 2));
        q = static_cast<float*>(dev(static_cast<size_t>(M) * d * 4));
        if (hq) {
            std::vector<__nv_bfloat16> hk(static_cast<size_t>(slots) * d), hv(hk.size());
            for (size_t i = 0; i < static_cast<size_t>(n_ctx) * d; ++i) {
                hk[i] = __float2bfloat16(kctx[i]);
                hv[i] = __float2bfloat16(vctx[i]);
            }
            for (size_t i = 0; i < static_cast<size_t>(M) * d; ++i) {
                hk[n_ctx * d + i] = __float2bfloat16(knode[i]);
                hv[n_ctx * d + i] = __float2bfloat16(vnode[i]);
            }
            SGB_CUDA(cudaMemcpy(K, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice));
            SGB_CUDA(cudaMemcpy(V, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice));
            SGB_CUDA(cudaMemcpy(q, hq, static_cast<size_t>(M) * d * 4, cudaMemcpyHostToDevice));
        } else {  // timing only: constant data
            SGB_CUDA(cudaMemset(K, 0x3c, static_cast<size_t>(slots) * d * 2));
            SGB_CUDA(cudaMemset(V, 0x3c, static_cast<size_t>(slots) * d * 2));
            SGB_CUDA(cudaMemset(q, 0, static_cast<size_t>(M) * d * 4));
        }
        auto* pacc = static_cast<float*>(dev(static_cast<size_t>(M) * d * ns * 4));
        auto* pml = static_cast<float*>(dev(static_cast<size_t>(M) * H * ns * 2 * 4));
        auto* dbase = static_cast<long long*>(dev(M * 8));
        auto* dchain = static_cast<long long*>(dev(chain.size() * 8));
        auto* dcl = static_cast<int*>(dev(M * 4));
        auto* dchl = static_cast<int*>(dev(M * 4));
        tiles = static_cast<sgb::AttnTileDev*>(dev(ht.size() * sizeof(sgb::AttnTileDev)));
        // attention_tree.cu: one group per sequence (node rows = its tree rows' own slots)
        {
            long long cb = 0;
            int r = 0, mx = 1;
            for (int g = 0; g < n_groups; ++g) {
                tg.push_back(sgb::TreeGroupDev{r, n_rows[g], ctx_len[g], n_rows[g], n_ctx + r, cb, cb, 0, 0});
                max_nodes = std::max(max_nodes, n_rows[g]);
                mx = std::max(mx, n_rows[g]);
                cb += ctx_len[g];
                r += n_rows[g];
            }
            tw = sgb::tree_attn_warps(mx, n_groups, H, dh, max_nodes);
            std::vector<sgb::TreeTileDev> tt;
            sgb::build_tree_tiles(tg, tw, tt);
            n_ttiles = static_cast<int>(tt.size());
            dtg = static_cast<sgb::TreeGroupDev*>(dev(tg.size() * sizeof(sgb::TreeGroupDev)));
            dtt = static_cast<sgb::TreeTileDev*>(dev(tt.size() * sizeof(sgb::TreeTileDev)));
            SGB_CUDA(cudaMemcpy(dtg, tg.data(), tg.size() * sizeof(sgb::TreeGroupDev), cudaMemcpyHostToDevice));
            SGB_CUDA(cudaMemcpy(dtt, tt.data(), tt.size() * sizeof(sgb::TreeTileDev), cudaMemcpyHostToDevice));
            kmap = sgb::make_kmajor_map(K, static_cast<int>(slots), d, 16);
            vmap = sgb::make_kmajor_map(V, static_cast<int>(slots), d, 16);
        }
        sc = sgb::AttnScratch{pacc, pml, nullptr, static_cast<long long>(M) * H};  // >= rows x head groups
        sc.row_ctr = static_cast<int*>(dev(sc.ctr_cap * 4));
        SGB_CUDA(cudaMemset(sc.row_ctr, 0, sc.ctr_cap * 4));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), M * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), M * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), M * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(tiles, ht.data(), ht.size() * sizeof(sgb::AttnTileDev), cudaMemcpyHostToDevice));
        ar = sgb::AttnRowsDev{dbase, dcl, dchl, dchain};
    }
    ~TreeAttnCase() {
        for (void* p : ptrs) cudaFree(p);
    }
    void run_row() { sgb::launch_attention(q, K, V, n_slots, ar, M, H, d, max_vlen, keys, sc, o1, 0); }
    void run_tree() {
        sgb::launch_attention_tree(q, kmap, vmap, 0, K, V, ar, dtg, dtt, n_ttiles, tw, H, d, max_nodes, o2, 0);
    }
    void run_decode() {
        int mc = 0;
        for (const auto& g : tg) {
            if (g.nrows != 1) throw std::invalid_argument("decode attention: one row per group");
            mc = std::max(mc, g.ctx_len);
        }
        sgb::launch_attention_decode(q, kmap, vmap, 0, K, V, dtg, static_cast<int>(tg.size()), mc, H, d, o2, 0);
    }
    void run_group() { sgb::launch_attention_tiles(q, K, V, n_slots, ar, M, tiles, n_tiles, items, qw, H, d, max_vlen, sc, o2,
                                                    0); }
    void read(const __nv_bfloat16* o, float* out) const {
        std::vector<__nv_bfloat16> ho(static_cast<size_t>(M) * d);
        SGB_CUDA(cudaMemcpy(ho.data(), o, ho.size() * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < ho.size(); ++i) out[i] = __bfloat162float(ho[i]);
    }
};
}  // namespace

int sgb_debug_tree_attention(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H, int dh,
                             const float* q, const float* kctx, const float* vctx, const float* knode,
                             const float* vnode, float* out_row, float* out_group) {
    return guarded([&] {
        if (!q) throw std::invalid_argument("debug_tree_attention: null inputs");
        TreeAttnCase c(n_groups, ctx_len, n_rows, parent, H, dh, q, kctx, vctx, knode, vnode);
        c.run_row();
        c.run_group();
        SGB_CUDA(cudaDeviceSynchronize());
        c.read(c.o1, out_row);
        c.read(c.o2, out_group);
    });
}

int sgb_debug_tree_attention_tree(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H, int dh,
                                  const float* q, const float* kctx, const float* vctx, const float* knode,
                                  const float* vnode, float* out_tree) {
    return guarded([&] {
        if (!q) throw std::invalid_argument("debug_tree_attention: null inputs");
        TreeAttnCase c(n_groups, ctx_len, n_rows, parent, H, dh, q, kctx, vctx, knode, vnode);
        c.run_tree();
        SGB_CUDA(cudaDeviceSynchronize());
        c.read(c.o2, out_tree);
    });
}

// attention_tree.cu's cluster decode kernel (AR steps: one row per group) on the same inputs
int sgb_debug_attention_decode(int n_groups, const int* ctx_len, int H, int dh, const float* q, const float* kctx,
                               const float* vctx, const float* knode, const float* vnode, float* out_row,
                               float* out_decode) {
    return guarded([&] {
        if (!q) throw std::invalid_argument("debug_attention_decode: null inputs");
        std::vector<int> nr(n_groups, 1), par(n_groups, -1);
        TreeAttnCase c(n_groups, ctx_len, nr.data(), par.data(), H, dh, q, kctx, vctx, knode, vnode);
        c.run_row();
        c.run_decode();
        SGB_CUDA(cudaDeviceSynchronize());
        c.read(c.o1, out_row);
        c.read(c.o2, out_decode);
    });
}

// AR attention microbenchmark: B rows with ctx committed keys each; device ms per launch of
// attention.cu (row path), the tree kernel and the cluster decode kernel
int sgb_bench_attention_decode(int B, int ctx, int H, int dh, int iters, double* ms_row, double* ms_tree,
                               double* ms_decode) {
    return guarded([&] {
        if (B <= 0 || iters <= 0) throw std::invalid_argument("bench_attention_decode: bad shape");
        std::vector<int> cl(B, ctx), nr(B, 1), par(B, -1);
        TreeAttnCase c(B, cl.data(), nr.data(), par.data(), H, dh, nullptr, nullptr, nullptr, nullptr, nullptr);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        auto time = [&](auto&& f) {
            for (int i = 0; i < 2; ++i) f();
            SGB_CUDA(cudaEventRecord(a, 0));
            for (int i = 0; i < iters; ++i) f();
            SGB_CUDA(cudaEventRecord(b, 0));
            SGB_CUDA(cudaEventSynchronize(b));
            float ms = 0.f;
            SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
            return static_cast<double>(ms) / iters;
        };
        *ms_row = time([&] { c.run_row(); });
        *ms_tree = time([&] { c.run_tree(); });
        *ms_decode = time([&] { c.run_decode(); });
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

int sgb_bench_tree_attention_tree(int B, int N, int ctx, int H, int dh, int iters, double* ms_tree) {
    return guarded([&] {
        if (B <= 0 || N <= 0 || iters <= 0) throw std::invalid_argument("bench_tree_attention: bad shape");
        std::vector<int> cl(B, ctx), nr(B, N), par;
        for (int b = 0; b < B; ++b) {
            std::vector<int> dep(N, 0);
            for (int i = 0; i < N; ++i) {
                int p = i == 0 ? -1 : (i - 1) / 10;
                if (i) {
                    while (dep[p] + 1 >= sgb::kMaxChain) p = (p - 1) / 10;
                    dep[i] = dep[p] + 1;
                }
                par.push_back(p);
            }
        }
        TreeAttnCase c(B, cl.data(), nr.data(), par.data(), H, dh, nullptr, nullptr, nullptr, nullptr, nullptr);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 2; ++i) c.run_tree();
        SGB_CUDA(cudaEventRecord(a, 0));
        for (int i = 0; i < iters; ++i) c.run_tree();
        SGB_CUDA(cudaEventRecord(b, 0));
        SGB_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_tree = ms / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

// Tree-verify attention microbenchmark: B sequences with ctx committed keys each, an EAGLE-
// shaped tree of N rows per sequence (node i's parent (i-1)/k, depth <= kMaxChain-1); times
// the per-row kernel and the prefix-shared group kernel (CUDA events, default stream).
int sgb_bench_tree_attention(int B, int N, int ctx, int H, int dh, int iters, double* ms_row, double* ms_group) {
    return guarded([&] {
        if (B <= 0 || N <= 0 || iters <= 0) throw std::invalid_argument("bench_tree_attention: bad shape");
        std::vector<int> cl(B, ctx), nr(B, N), par;
        for (int b = 0; b < B; ++b) {
            std::vector<int> dep(N, 0);
            for (int i = 0; i < N; ++i) {
                int p = i == 0 ? -1 : (i - 1) / 10;
                if (i) {
                    while (dep[p] + 1 >= sgb::kMaxChain) p = (p - 1) / 10;
                    dep[i] = dep[p] + 1;
                }
                par.push_back(p);
            }
        }
        TreeAttnCase c(B, cl.data(), nr.data(), par.data(), H, dh, nullptr, nullptr, nullptr, nullptr, nullptr);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        float ms = 0.f;
        for (int pass = 0; pass < 2; ++pass) {
            for (int i = 0; i < 2; ++i) pass ? c.run_group() : c.run_row();
            SGB_CUDA(cudaEventRecord(a, 0));
            for (int i = 0; i < iters; ++i) pass ? c.run_group() : c.run_row();
            SGB_CUDA(cudaEventRecord(b, 0));
            SGB_CUDA(cudaEventSynchronize(b));
            SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
            (pass ? *ms_group : *ms_row) = ms / iters;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

// Decode-attention microbenchmark: B sequences x H heads, each one query row attending to
// ctx cached keys + itself (AR decode shape), KV in a [B*(ctx+1)][d] bf16 store.
int sgb_bench_attention(int B, int ctx, int H, int dh, int iters, double* ms_out) {
    return guarded([&] {
        const int d = H * dh;
        const long long slots = static_cast<long long>(B) * (ctx + 1);
        __nv_bfloat16 *K = nullptr, *V = nullptr, *out = nullptr;
        float *q = nullptr, *pacc = nullptr, *pml = nullptr;
        SGB_CUDA(cudaMalloc(&K, slots * d * 2));
        SGB_CUDA(cudaMalloc(&V, slots * d * 2));
        SGB_CUDA(cudaMemset(K, 0x3c, slots * d * 2));
        SGB_CUDA(cudaMemset(V, 0x3c, slots * d * 2));
        SGB_CUDA(cudaMalloc(&q, static_cast<size_t>(B) * d * 4));
        SGB_CUDA(cudaMemset(q, 0, static_cast<size_t>(B) * d * 4));
        SGB_CUDA(cudaMalloc(&out, static_cast<size_t>(B) * d * 2));
        const int ns = sgb::attn_splits_for(ctx + 1);
        SGB_CUDA(cudaMalloc(&pacc, static_cast<size_t>(B) * d * ns * 4));
        SGB_CUDA(cudaMalloc(&pml, static_cast<size_t>(B) * H * ns * 2 * 4));
        std::vector<long long> base(B), chain(static_cast<size_t>(B) * sgb::kMaxChain, 0);
        std::vector<int> cl(B, ctx), chl(B, 1);
        for (int b = 0; b < B; ++b) {
            base[b] = static_cast<long long>(b) * (ctx + 1);
            chain[static_cast<size_t>(b) * sgb::kMaxChain] = base[b] + ctx;
        }
        long long *dbase = nullptr, *dchain = nullptr;
        int *dcl = nullptr, *dchl = nullptr;
        SGB_CUDA(cudaMalloc(&dbase, B * 8));
        SGB_CUDA(cudaMalloc(&dchain, chain.size() * 8));
        SGB_CUDA(cudaMalloc(&dcl, B * 4));
        SGB_CUDA(cudaMalloc(&dchl, B * 4));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), B * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), B * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), B * 4, cudaMemcpyHostToDevice));
        sgb::AttnRowsDev ar{dbase, dcl, dchl, dchain};
        sgb::AttnScratch sc{pacc, pml, nullptr, static_cast<long long>(B) * H};
        SGB_CUDA(cudaMalloc(&sc.row_ctr, sc.ctr_cap * 4));
        SGB_CUDA(cudaMemset(sc.row_ctr, 0, sc.ctr_cap * 4));
        const double keys = static_cast<double>(B) * (ctx + 1);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 2; ++i) sgb::launch_attention(q, K, V, slots, ar, B, H, d, ctx + 1, keys, sc, out, 0);
        SGB_CUDA(cudaEventRecord(a, 0));
        for (int i = 0; i < iters; ++i) sgb::launch_attention(q, K, V, slots, ar, B, H, d, ctx + 1, keys, sc, out, 0);
        SGB_CUDA(cudaEventRecord(b, 0));
        SGB_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_out = ms / iters;
        void* ptrs[] = {K, V, out, q, pacc, pml, dbase, dchain, dcl, dchl, sc.row_ctr};
        for (void* p : ptrs) cudaFree(p);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

int sgb_profile_enable(sgb_engine* e, int on) {
    return guarded([&] { E(e).set_profiling(on != 0); });
}

int sgb_profile_read(sgb_engine* e, int n_cls, double* ms, double* bytes, double* flops, long long* launches,
                     int reset) {
    return guarded([&] {
        sgb::KernelProfile kp[sgb::kNumCls];
        E(e).read_profile(kp, sgb::kNumCls, reset != 0);
        for (int i = 0; i < n_cls && i < sgb::kNumCls; ++i) {
            if (ms) ms[i] = kp[i].ms;
            if (bytes) bytes[i] = kp[i].bytes;
            if (flops) flops[i] = kp[i].flops;
            if (launches) launches[i] = kp[i].launches;
        }
    });
}

int sgb_debug_gemm(const float* w, const float* x, int M, int N, int K, float* out, int* splits_out) {
    return guarded([&] {
        if (M <= 0 || N <= 0 || K <= 0) throw std::invalid_argument("debug_gemm: bad shape");
        std::vector<__nv_bfloat16> wb(static_cast<size_t>(N) * K), xb(static_cast<size_t>(M) * K);
        for (size_t i = 0; i < wb.size(); ++i) wb[i] = __float2bfloat16(w[i]);
        for (size_t i = 0; i < xb.size(); ++i) xb[i] = __float2bfloat16(x[i]);
        __nv_bfloat16 *dw = nullptr, *dx = nullptr;
        float* dp = nullptr;
        const int cap = ((M + 255) / 256) * 256;
        SGB_CUDA(cudaMalloc(&dw, wb.size() * 2));
        SGB_CUDA(cudaMalloc(&dx, static_cast<size_t>(cap) * K * 2));
        SGB_CUDA(cudaMemset(dx, 0, static_cast<size_t>(cap) * K * 2));
        SGB_CUDA(cudaMemcpy(dw, wb.data(), wb.size() * 2, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dx, xb.data(), xb.size() * 2, cudaMemcpyHostToDevice));
        sgb::GemmWeight gw;
        gw.init(dw, N, K);
        sgb::GemmAct ga;
        ga.init(dx, cap, K);
        sgb::GemmWorkspace ws;
        ws.cap_floats = sgb::gemm_ws_floats(M, N, K);
        ws.ctr_cap = 1 << 14;
        SGB_CUDA(cudaMalloc(&ws.buf, ws.cap_floats * 4));
        SGB_CUDA(cudaMalloc(&ws.ctr, ws.ctr_cap * sizeof(int)));
        SGB_CUDA(cudaMemset(ws.ctr, 0, ws.ctr_cap * sizeof(int)));
        SGB_CUDA(cudaMalloc(&dp, static_cast<size_t>(M) * N * 4));
        sgb::GemmEpi epi;
        epi.kind = sgb::kEpiF32;
        epi.f32 = dp;
        epi.ld = N;
        sgb::gemm_run(gw, ga, M, epi, ws, 0, splits_out ? *splits_out : 0);
        SGB_KCHECK();
        SGB_CUDA(cudaDeviceSynchronize());
        SGB_CUDA(cudaMemcpy(out, dp, static_cast<size_t>(M) * N * 4, cudaMemcpyDeviceToHost));
        if (splits_out) *splits_out = sgb::gemm_splits_for(M, N, K);
        cudaFree(ws.buf);
        cudaFree(ws.ctr);
        cudaFree(dw);
        cudaFree(dx);
        cudaFree(dp);
    });
}

}  // extern "C"

// Concurrency microbenchmark for the two-lane AR step: one decoder layer's attention
// (B rows x (ctx + 1) keys, H heads of dh) on one stream and the layer's four GEMMs at M rows
// (QKV, wo, w1, w2 of width d = H*dh and d_ff) on another, each on a capped persistent grid
// (attn_cap / gemm_cap SMs, 0 = all). out[0..2] = ms per iteration: attention alone, GEMMs
// alone, both streams concurrently.
int sgb_bench_overlap(int B, int ctx, int H, int dh, int dff, int M, int attn_cap, int gemm_cap, int iters,
                      double* out) {
    return guarded([&] {
        if (B <= 0 || M <= 0 || iters <= 0) throw std::invalid_argument("bench_overlap: bad shape");
        const int d = H * dh;
        const long long slots = static_cast<long long>(B) * (ctx + 1);
        std::vector<void*> frees;
        auto dmal = [&](size_t bytes) {
            void* p = nullptr;
            SGB_CUDA(cudaMalloc(&p, bytes));
            SGB_CUDA(cudaMemset(p, 0, bytes));
            frees.push_back(p);
            return p;
        };
        auto* K = static_cast<__nv_bfloat16*>(dmal(slots * d * 2));
        auto* V = static_cast<__nv_bfloat16*>(dmal(slots * d * 2));
        SGB_CUDA(cudaMemset(K, 0x3c, slots * d * 2));
        SGB_CUDA(cudaMemset(V, 0x3c, slots * d * 2));
        auto* q = static_cast<float*>(dmal(static_cast<size_t>(B) * d * 4));
        auto* ao = static_cast<__nv_bfloat16*>(dmal(static_cast<size_t>(B) * d * 2));
        const int ns = sgb::attn_splits_for(ctx + 1);
        sgb::AttnScratch sc{static_cast<float*>(dmal(static_cast<size_t>(B) * d * ns * 4)),
                            static_cast<float*>(dmal(static_cast<size_t>(B) * H * ns * 8)), nullptr,
                            static_cast<long long>(B) * H};
        sc.row_ctr = static_cast<int*>(dmal(sc.ctr_cap * 4));
        std::vector<long long> base(B), chain(static_cast<size_t>(B) * sgb::kMaxChain, 0);
        std::vector<int> cl(B, ctx), chl(B, 1);
        for (int b = 0; b < B; ++b) {
            base[b] = static_cast<long long>(b) * (ctx + 1);
            chain[static_cast<size_t>(b) * sgb::kMaxChain] = base[b] + ctx;
        }
        auto* dbase = static_cast<long long*>(dmal(B * 8));
        auto* dchain = static_cast<long long*>(dmal(chain.size() * 8));
        auto* dcl = static_cast<int*>(dmal(B * 4));
        auto* dchl = static_cast<int*>(dmal(B * 4));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), B * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), B * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), B * 4, cudaMemcpyHostToDevice));
        sgb::AttnRowsDev ar{dbase, dcl, dchl, dchain};
        const double keys = static_cast<double>(B) * (ctx + 1);
        // the layer's GEMMs, weights in rotating copies (> L2) as in the rollout
        const int shp[4][2] = {{3 * d, d}, {d, d}, {dff, d}, {d, dff}};
        const int ncopy = 4;
        std::vector<sgb::GemmWeight> gw(4 * ncopy);
        for (int g = 0; g < 4; ++g)
            for (int c = 0; c < ncopy; ++c) {
                auto* w = static_cast<__nv_bfloat16*>(dmal(static_cast<size_t>(shp[g][0]) * shp[g][1] * 2));
                gw[g * ncopy + c].init(w, shp[g][0], shp[g][1]);
            }
        const int cap = ((M + 255) / 256) * 256;
        auto* xa = static_cast<__nv_bfloat16*>(dmal(static_cast<size_t>(cap) * std::max(d, dff) * 2));
        sgb::GemmAct act_d, act_f;
        act_d.init(xa, cap, d);
        act_f.init(xa, cap, dff);
        auto* yo = static_cast<float*>(dmal(static_cast<size_t>(M) * 3 * std::max(d, dff) * 4));
        sgb::GemmWorkspace ws;
        sgb::GemmEpi epi;
        epi.kind = sgb::kEpiF32;
        epi.f32 = yo;
        cudaStream_t s1, s2;
        SGB_CUDA(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
        SGB_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        cudaEvent_t a, b, j;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        SGB_CUDA(cudaEventCreate(&j));
        int rot = 0;
        auto attn = [&] {
            sgb::g_attn_sm_cap = attn_cap;
            sgb::launch_attention(q, K, V, slots, ar, B, H, d, ctx + 1, keys, sc, ao, s1);
            sgb::g_attn_sm_cap = 0;
        };
        auto gemms = [&] {
            sgb::g_gemm_sm_cap = gemm_cap;
            for (int g = 0; g < 4; ++g) {
                epi.ld = shp[g][0];
                sgb::gemm_run(gw[g * ncopy + rot % ncopy], g == 3 ? act_f : act_d, M, epi, ws, s2, 1);
            }
            ++rot;
            sgb::g_gemm_sm_cap = 0;
        };
        auto time = [&](bool ra, bool rg) {
            for (int w = 0; w < 2; ++w) {
                if (ra) attn();
                if (rg) gemms();
            }
            SGB_CUDA(cudaDeviceSynchronize());
            SGB_CUDA(cudaEventRecord(a, s1));
            SGB_CUDA(cudaStreamWaitEvent(s2, a, 0));
            for (int i = 0; i < iters; ++i) {
                if (ra) attn();
                if (rg) gemms();
            }
            SGB_CUDA(cudaEventRecord(j, s2));
            SGB_CUDA(cudaStreamWaitEvent(s1, j, 0));
            SGB_CUDA(cudaEventRecord(b, s1));
            SGB_CUDA(cudaEventSynchronize(b));
            SGB_KCHECK();
            float ms = 0.f;
            SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
            return static_cast<double>(ms) / iters;
        };
        out[0] = time(true, false);
        out[1] = time(false, true);
        out[2] = time(true, true);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaEventDestroy(j);
        cudaStreamDestroy(s1);
        cudaStreamDestroy(s2);
        for (void* p : frees) cudaFree(p);
    });
}
