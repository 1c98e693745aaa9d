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

}  // extern "C"

