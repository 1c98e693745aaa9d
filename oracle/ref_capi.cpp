// C-ABI shim over the compiled reference (oracle/_ref). TEST INFRASTRUCTURE ONLY.
//
// Exposes the reference's own functions (namespace sgrpo, /root/reference/proj) to
// Python through plain pointers so tests/golden/make_golden.py can pin the numpy
// oracle against the real reference, and bench.py's --impl reference arm can time
// the reference's own generate_dynamic_batch on the host cores. Nothing here
// re-implements reference arithmetic; every call forwards to the reference symbol
// named in its comment.

#include <atomic>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sgrpo/drafttree.hpp"
#include "sgrpo/grpo.hpp"
#include "sgrpo/roofline.hpp"
#include "sgrpo/scheduler.hpp"
#include "sgrpo/tinylm.hpp"

using namespace sgrpo;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

struct CfgC {
    int vocab, d, layers, heads, dff, max_seq;
    unsigned long long seed;
};

ModelConfig to_cfg(const CfgC* c) {
    ModelConfig m;
    m.vocab_size = c->vocab;
    m.d_model = c->d;
    m.n_layers = c->layers;
    m.n_heads = c->heads;
    m.d_ff = c->dff;
    m.max_seq_len = c->max_seq;
    m.seed = c->seed;
    return m;
}

struct TreeC {
    std::vector<int> tok, par, depth;
    std::vector<double> lp, conf;
};

DraftTree tree_from(int n, const int* tok, const int* par, const int* depth, const double* lp,
                    const double* conf) {
    DraftTree t;
    for (int i = 0; i < n; ++i) t.nodes.push_back({tok[i], par[i], depth[i], lp[i], conf[i]});
    return t;
}

}  // namespace

extern "C" {

const char* sgref_last_error() { return g_err.c_str(); }

// ---- rng.hpp:9-65 -------------------------------------------------------------
unsigned long long sgref_mix_key(unsigned long long a, unsigned long long b) { return mix_key(a, b); }
void sgref_splitmix(unsigned long long* state, int n, unsigned long long* out) {
    uint64_t s = *state;
    for (int i = 0; i < n; ++i) out[i] = splitmix64(s);
    *state = s;
}
void sgref_rng_uniforms(unsigned long long seed, int n, double* out) {
    Rng r(seed);
    for (int i = 0; i < n; ++i) out[i] = r.uniform();
}
void sgref_rng_normals(unsigned long long seed, int n, double* out) {
    Rng r(seed);
    for (int i = 0; i < n; ++i) out[i] = r.normal();
}
void sgref_rng_below(unsigned long long seed, unsigned long long m, int n, unsigned long long* out) {
    Rng r(seed);
    for (int i = 0; i < n; ++i) out[i] = r.below(m);
}

// ---- tinylm.hpp:133-189 (init), param counts ------------------------------------
size_t sgref_param_count(const CfgC* c) { return param_count_for(to_cfg(c)); }
size_t sgref_draft_param_count(const CfgC* c, int layers) {
    return draft_param_count_for(to_cfg(c), layers);
}
int sgref_init_model(const CfgC* c, float* out) {
    return guarded([&] {
        auto m = init_model<float>(to_cfg(c));
        std::memcpy(out, m.flat.data(), m.flat.size() * sizeof(float));
    });
}
int sgref_init_draft(const CfgC* c, int layers, float* out) {
    return guarded([&] {
        auto d = init_draft<float>(to_cfg(c), layers);
        std::memcpy(out, d.flat.data(), d.flat.size() * sizeof(float));
    });
}

// Handles: Model / Draft owned by the shim, weights supplied by the caller.
void* sgref_model_new(const CfgC* c, const float* flat) {
    Model* m = nullptr;
    int rc = guarded([&] {
        m = new Model(init_model<float>(to_cfg(c)));
        if (flat) std::memcpy(m->flat.data(), flat, m->flat.size() * sizeof(float));
    });
    return rc == 0 ? m : nullptr;
}
void* sgref_draft_new(const CfgC* c, int layers, const float* flat) {
    Draft* d = nullptr;
    int rc = guarded([&] {
        d = new Draft(init_draft<float>(to_cfg(c), layers));
        if (flat) std::memcpy(d->flat.data(), flat, d->flat.size() * sizeof(float));
    });
    return rc == 0 ? d : nullptr;
}
void sgref_model_free(void* m) { delete static_cast<Model*>(m); }
void sgref_draft_free(void* d) { delete static_cast<Draft*>(d); }
void sgref_draft_get(void* d, float* out) {
    auto* dr = static_cast<Draft*>(d);
    std::memcpy(out, dr->flat.data(), dr->flat.size() * sizeof(float));
}
unsigned long long sgref_target_forward_calls() { return target_forward_calls(); }

// ---- KvCacheT (tinylm.hpp:232-269) ----------------------------------------------
void* sgref_cache_new(int layers, int d) {
    auto* c = new KvCache();
    c->reset(layers, d);
    return c;
}
void* sgref_cache_clone(void* c) { return new KvCache(*static_cast<KvCache*>(c)); }
void sgref_cache_free(void* c) { delete static_cast<KvCache*>(c); }
int sgref_cache_len(void* c) { return static_cast<KvCache*>(c)->len; }
void sgref_cache_get(void* c, float* k, float* v) {
    auto* kc = static_cast<KvCache*>(c);
    size_t n = static_cast<size_t>(kc->len) * kc->d;
    for (int l = 0; l < kc->n_layers; ++l) {
        std::memcpy(k + l * n, kc->k[l].data(), n * sizeof(float));
        std::memcpy(v + l * n, kc->v[l].data(), n * sizeof(float));
    }
}
int sgref_cache_gather_tail(void* c, int base, const int* keep, int n) {
    return guarded([&] { static_cast<KvCache*>(c)->gather_tail(base, std::span<const int>(keep, n)); });
}
int sgref_cache_truncate(void* c, int len) {
    return guarded([&] { static_cast<KvCache*>(c)->truncate(len); });
}

// ---- forward_target (tinylm.hpp:422-463) ------------------------------------------
int sgref_forward_target(void* model, const int* toks, const int* pos, int rows,
                         const unsigned char* mask, void* cache, float* logits, float* hidden) {
    return guarded([&] {
        const Model& m = *static_cast<Model*>(model);
        AttnMask am;
        if (mask) {
            am.rows = rows;
            am.bits.assign(mask, mask + static_cast<size_t>(rows) * rows);
        }
        auto out = forward_target<float>(m, std::span<const int>(toks, rows),
                                         std::span<const int>(pos, rows), mask ? &am : nullptr,
                                         static_cast<KvCache*>(cache));
        if (logits) std::memcpy(logits, out.logits.data(), out.logits.size() * sizeof(float));
        if (hidden) std::memcpy(hidden, out.hidden.data(), out.hidden.size() * sizeof(float));
    });
}

// ---- forward_draft_rows (tinylm.hpp:502-563), cache + optional causal mask ---------
int sgref_forward_draft_rows(void* draft, void* model, const int* toks, const float* prev_feat,
                             const int* pos, int rows, void* cache, int extend, float* feats,
                             float* logits) {
    return guarded([&] {
        const Draft& dr = *static_cast<Draft*>(draft);
        const Model& m = *static_cast<Model*>(model);
        DraftForwardIn<float> in;
        in.tokens = std::span<const int>(toks, rows);
        in.prev_features = std::span<const float>(prev_feat, static_cast<size_t>(rows) * m.config.d_model);
        in.positions = std::span<const int>(pos, rows);
        in.cache = static_cast<KvCache*>(cache);
        in.extend_cache = extend != 0;
        auto out = forward_draft_rows(dr, m, in);
        if (feats) std::memcpy(feats, out.features.data(), out.features.size() * sizeof(float));
        if (logits) std::memcpy(logits, out.logits.data(), out.logits.size() * sizeof(float));
    });
}

// ---- sample_token (tinylm.hpp:591-628) --------------------------------------------
int sgref_sample_token(const float* logits, int n, double temp, unsigned long long key, int* out) {
    return guarded([&] { *out = sample_token<float>(std::span<const float>(logits, n), temp, key); });
}

// Supplied-uniform mode (the exception to "forward only"): sample_token derives u from a key,
// so the parity tests that place u at a chosen CDF boundary need lines 614-627 of tinylm.hpp
// with `rng.uniform()` replaced by the supplied U -- nothing else changes (same std::exp, same
// sequential sums, same comparison). Pinned against the real sample_token by the tests (U =
// Rng(key).uniform() must give sample_token's token for every key).
int sgref_sample_token_u(const float* logits, int n, double temperature, double U, int* out,
                         double* sum_out, double* prefix_out) {
    return guarded([&] {
        double mx = -std::numeric_limits<double>::infinity();
        for (int i = 0; i < n; ++i) mx = std::max(mx, double(logits[i]));
        std::vector<double> p(n);
        double sum = 0;
        for (int i = 0; i < n; ++i) {
            p[i] = std::exp((double(logits[i]) - mx) / temperature);
            sum += p[i];
        }
        double u = U * sum;
        double acc = 0;
        if (prefix_out)
            for (int i = 0; i < n; ++i) prefix_out[i] = acc += p[i];
        acc = 0;
        int tok = n - 1;
        for (int i = 0; i < n; ++i) {
            acc += p[i];
            if (u < acc) {
                tok = i;
                break;
            }
        }
        *out = tok;
        if (sum_out) *sum_out = sum;
    });
}

// std::exp of the reference's libm over an array (the host exp the device restates).
void sgref_exp_array(const double* x, long long n, double* y) {
    for (long long i = 0; i < n; ++i) y[i] = std::exp(x[i]);
}

// Rng(key).uniform() (rng.hpp:28-41)
double sgref_uniform(unsigned long long key) { return Rng(key).uniform(); }

// ---- drafttree (drafttree.cpp) ----------------------------------------------------
long long sgref_max_candidates(int k, int l) { return max_candidates(k, l); }

typedef void (*sgref_lps_fn)(void* ctx, int n_nodes, const int* tokens, const int* parents,
                             const int* depths, int node, double* out_lps);

int sgref_expand_tree_with(int root, int k, int l, int vocab, sgref_lps_fn fn, void* ctx,
                           int cap, int* tok, int* par, int* depth, double* lp, double* conf,
                           int* n_out) {
    return guarded([&] {
        ExpandFn efn = [&](const DraftTree& t, int node) {
            std::vector<int> tt, pp, dd;
            for (const auto& nd : t.nodes) {
                tt.push_back(nd.token);
                pp.push_back(nd.parent);
                dd.push_back(nd.depth);
            }
            std::vector<double> lps(vocab);
            fn(ctx, static_cast<int>(t.nodes.size()), tt.data(), pp.data(), dd.data(), node, lps.data());
            return lps;
        };
        DraftTree t = expand_tree_with(root, k, l, efn);
        if (static_cast<int>(t.nodes.size()) > cap) throw std::runtime_error("tree capacity");
        for (size_t i = 0; i < t.nodes.size(); ++i) {
            tok[i] = t.nodes[i].token;
            par[i] = t.nodes[i].parent;
            depth[i] = t.nodes[i].depth;
            lp[i] = t.nodes[i].log_prob;
            conf[i] = t.nodes[i].confidence;
        }
        *n_out = static_cast<int>(t.nodes.size());
    });
}

int sgref_rerank(int n, const int* tok, const int* par, const int* depth, const double* lp,
                 const double* conf, int n_verify, int* sel, int* n_sel, unsigned char* mask) {
    return guarded([&] {
        DraftTree t = tree_from(n, tok, par, depth, lp, conf);
        SelectedSet s = rerank_candidates(t, n_verify);
        *n_sel = static_cast<int>(s.node_indices.size());
        for (int i = 0; i < *n_sel; ++i) sel[i] = s.node_indices[i];
        if (mask) std::memcpy(mask, s.tree_mask.bits.data(), s.tree_mask.bits.size());
    });
}

int sgref_build_tree_mask(int n, const int* tok, const int* par, const int* depth,
                          const double* lp, const double* conf, const int* sel, int n_sel,
                          unsigned char* mask) {
    return guarded([&] {
        DraftTree t = tree_from(n, tok, par, depth, lp, conf);
        AttnMask m = build_tree_mask(t, std::vector<int>(sel, sel + n_sel));
        std::memcpy(mask, m.bits.data(), m.bits.size());
    });
}

int sgref_verify(int n, const int* tok, const int* par, const int* depth, const double* lp,
                 const double* conf, const int* sel, int n_sel, const float* logits,
                 const float* hidden, int vocab, int d, double temp, unsigned long long seq_seed,
                 int root_pos, int* acc_tokens, int* acc_len, int* bonus, int* acc_rows,
                 float* new_hidden) {
    return guarded([&] {
        DraftTree t = tree_from(n, tok, par, depth, lp, conf);
        SelectedSet s;
        s.node_indices.assign(sel, sel + n_sel);
        s.tree_mask = build_tree_mask(t, s.node_indices);
        VerifyInputs in;
        in.logits = std::span<const float>(logits, static_cast<size_t>(n_sel) * vocab);
        if (hidden) in.hidden = std::span<const float>(hidden, static_cast<size_t>(n_sel) * d);
        in.vocab = vocab;
        in.d = d;
        in.temperature = temp;
        in.seq_seed = seq_seed;
        in.root_pos = root_pos;
        VerifyResult r = verify(t, s, in);
        *acc_len = r.accepted_len;
        *bonus = r.bonus_token;
        for (int i = 0; i < r.accepted_len; ++i) {
            acc_tokens[i] = r.accepted_tokens[i];
            acc_rows[i] = r.accepted_rows[i];
        }
        if (new_hidden && !r.new_hidden.empty())
            std::memcpy(new_hidden, r.new_hidden.data(), r.new_hidden.size() * sizeof(float));
    });
}

// ---- scheduler.cpp:14-54 ------------------------------------------------------------
// GRPO rewards / advantages (src/grpo.cpp:99-136)
double sgref_compute_reward(long long a, long long b, const int* resp, int n) {
    TaskExample ex;
    ex.a = a;
    ex.b = b;
    return compute_reward(ex, std::span<const int>(resp, static_cast<size_t>(n)));
}
int sgref_standardize_advantages(const double* rewards, int g, double eps_var, double* out) {
    std::vector<double> r(rewards, rewards + g);
    auto adv = standardize_advantages(r, eps_var);
    if (!adv) return 0;
    for (int i = 0; i < g; ++i) out[i] = (*adv)[i];
    return 1;
}

int sgref_plan_step(int c_peak, int b, double alpha, int kmax, int lmax, int* out3) {
    return guarded([&] {
        SpecConfig c = plan_step(c_peak, b, alpha, kmax, lmax);
        out3[0] = c.n_verify;
        out3[1] = c.k_draft;
        out3[2] = c.l_draft;
    });
}
int sgref_compute(int which, int a, int b, double alpha, int c, int* out) {
    return guarded([&] {
        if (which == 0) *out = compute_n_verify(a, b);
        else if (which == 1) *out = compute_k_draft(a, b);
        else *out = compute_l_draft(a, alpha, b, c);
    });
}

// ---- generate_dynamic_batch (scheduler.cpp:236-354) -------------------------------------
struct GenArgs {
    double alpha;
    int k_max, l_max, c_peak;
    int mode;  // 0 vanilla, 1 fixed_spec, 2 adaptive_spec
    int early_term;
    double temperature;
    unsigned long long seed;
    int max_new_tokens;
    int fixed_n, fixed_k, fixed_l;
};

static GenOptions to_opts(const GenArgs* a) {
    GenOptions o;
    o.mode = a->mode == 0 ? DecodeMode::vanilla
                          : (a->mode == 1 ? DecodeMode::fixed_spec : DecodeMode::adaptive_spec);
    o.early_term = a->early_term != 0;
    o.temperature = a->temperature;
    o.seed = a->seed;
    o.max_new_tokens = a->max_new_tokens;
    o.fixed.n_verify = a->fixed_n;
    o.fixed.k_draft = a->fixed_k;
    o.fixed.l_draft = a->fixed_l;
    o.fixed.alpha = a->alpha;
    o.fixed.k_max = a->k_max;
    o.fixed.l_max = a->l_max;
    o.fixed.c_peak = a->c_peak;
    return o;
}

void* sgref_generate(void* model, void* draft, const int* prompts, const int* plens, int nprompts,
                     int g, const GenArgs* a) {
    BatchState* bs = nullptr;
    int rc = guarded([&] {
        std::vector<std::vector<int>> pr;
        size_t off = 0;
        for (int i = 0; i < nprompts; ++i) {
            pr.emplace_back(prompts + off, prompts + off + plens[i]);
            off += plens[i];
        }
        SchedParams sp{a->alpha, a->k_max, a->l_max, a->c_peak};
        HardwareProfile prof = desk_profile(a->c_peak);
        bs = new BatchState(generate_dynamic_batch(*static_cast<Model*>(model),
                                                   *static_cast<Draft*>(draft), pr, g, sp, prof,
                                                   to_opts(a)));
    });
    return rc == 0 ? bs : nullptr;
}
void sgref_bs_free(void* h) { delete static_cast<BatchState*>(h); }
int sgref_bs_nseq(void* h) { return static_cast<int>(static_cast<BatchState*>(h)->seqs.size()); }
int sgref_bs_seq(void* h, int i, int* tokens, int cap, int* len, int* prompt_len, int* hit_eos) {
    const auto& s = static_cast<BatchState*>(h)->seqs[i];
    *len = static_cast<int>(s.tokens.size());
    *prompt_len = s.prompt_len;
    *hit_eos = s.hit_eos ? 1 : 0;
    if (tokens) std::memcpy(tokens, s.tokens.data(), std::min<size_t>(cap, s.tokens.size()) * sizeof(int));
    return static_cast<int>(s.features.size());
}
void sgref_bs_features(void* h, int i, float* out) {
    const auto& s = static_cast<BatchState*>(h)->seqs[i];
    std::memcpy(out, s.features.data(), s.features.size() * sizeof(float));
}
int sgref_bs_nsteps(void* h) { return static_cast<int>(static_cast<BatchState*>(h)->stats.steps.size()); }
void sgref_bs_steps(void* h, int* b_cur, int* nkl, int* accepted) {
    const auto& st = static_cast<BatchState*>(h)->stats.steps;
    for (size_t i = 0; i < st.size(); ++i) {
        b_cur[i] = st[i].b_cur;
        nkl[3 * i] = st[i].cfg.n_verify;
        nkl[3 * i + 1] = st[i].cfg.k_draft;
        nkl[3 * i + 2] = st[i].cfg.l_draft;
        accepted[i] = st[i].accepted_total;
    }
}
void sgref_bs_totals(void* h, long long* out2) {
    const auto& st = static_cast<BatchState*>(h)->stats;
    out2[0] = st.total_accepted;
    out2[1] = st.total_verify_slots;
}
int sgref_bs_nevents(void* h) { return static_cast<int>(static_cast<BatchState*>(h)->stats.events.size()); }
void sgref_bs_events(void* h, int* out3) {
    const auto& ev = static_cast<BatchState*>(h)->stats.events;
    for (size_t i = 0; i < ev.size(); ++i) {
        out3[3 * i] = ev[i].step;
        out3[3 * i + 1] = ev[i].seq;
        out3[3 * i + 2] = ev[i].accepted;
    }
}

// Reference arm for bench.py: the reference's own generate_dynamic_batch over disjoint
// prompt shards on `threads` host threads (the reference itself is single-threaded,
// SURVEY.md §8d "N cores"). Returns generated tokens; *seconds = wall time.
long long sgref_generate_threaded(void* model, void* draft, const int* prompts, const int* plens,
                                  int nprompts, int g, const GenArgs* a, int threads,
                                  double* seconds) {
    std::vector<std::vector<int>> pr;
    size_t off = 0;
    for (int i = 0; i < nprompts; ++i) {
        pr.emplace_back(prompts + off, prompts + off + plens[i]);
        off += plens[i];
    }
    if (threads < 1) threads = 1;
    if (threads > nprompts) threads = nprompts;
    std::atomic<long long> total{0};
    std::atomic<int> failed{0};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&, t] {
            std::vector<std::vector<int>> mine;
            for (int i = t; i < nprompts; i += threads) mine.push_back(pr[i]);
            if (mine.empty()) return;
            int rc = guarded([&] {
                SchedParams sp{a->alpha, a->k_max, a->l_max, a->c_peak};
                HardwareProfile prof = desk_profile(a->c_peak);
                BatchState bs = generate_dynamic_batch(*static_cast<Model*>(model),
                                                       *static_cast<Draft*>(draft), mine, g, sp,
                                                       prof, to_opts(a));
                long long n = 0;
                for (const auto& s : bs.seqs) n += static_cast<long long>(s.tokens.size()) - s.prompt_len;
                total += n;
            });
            if (rc) failed++;
        });
    }
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return failed ? -1 : total.load();
}

// ---- draft_loss_grad (grpo.hpp:278-344), AdamW::step (grpo.cpp:142-161),
//      draft_update (grpo.cpp:177-186) ------------------------------------------------
static std::vector<SeqResult> seqs_from(int nseq, const int* tokens, const int* lens,
                                        const float* feats, int d) {
    std::vector<SeqResult> out(nseq);
    size_t to = 0, fo = 0;
    for (int i = 0; i < nseq; ++i) {
        out[i].tokens.assign(tokens + to, tokens + to + lens[i]);
        size_t nf = static_cast<size_t>(std::max(0, lens[i] - 1)) * d;
        out[i].features.assign(feats + fo, feats + fo + nf);
        to += lens[i];
        fo += nf;
    }
    return out;
}

int sgref_draft_loss_grad(void* draft, void* model, int nseq, const int* tokens, const int* lens,
                          const float* feats, double w_feat, double w_tok, float* grad,
                          double* terms4) {
    return guarded([&] {
        const Draft& dr = *static_cast<Draft*>(draft);
        const Model& m = *static_cast<Model*>(model);
        auto seqs = seqs_from(nseq, tokens, lens, feats, m.config.d_model);
        std::vector<const SeqResult*> ptrs;
        for (auto& s : seqs) ptrs.push_back(&s);
        std::vector<float> g(dr.flat.size(), 0.f);
        DraftLossTerms t = draft_loss_grad<float>(dr, m, ptrs, w_feat, w_tok, g);
        std::memcpy(grad, g.data(), g.size() * sizeof(float));
        terms4[0] = t.feature_loss;
        terms4[1] = t.token_loss;
        terms4[2] = t.total;
        terms4[3] = double(t.rows);
    });
}

// policy_loss_grad<float> (grpo.hpp:235-276): the GRPO policy objective's loss and gradient
int sgref_policy_loss_grad(void* model, int nseq, const int* tokens, const int* lens, const int* prompt_lens,
                           const double* weights, float* grad, double* loss) {
    return guarded([&] {
        const Model& m = *static_cast<Model*>(model);
        std::vector<std::vector<int>> toks(nseq);
        std::vector<TrainSeq> ts(nseq);
        size_t off = 0;
        for (int i = 0; i < nseq; ++i) {
            toks[i].assign(tokens + off, tokens + off + lens[i]);
            off += lens[i];
        }
        for (int i = 0; i < nseq; ++i) ts[i] = TrainSeq{&toks[i], prompt_lens[i], weights[i]};
        std::vector<float> g(m.flat.size(), 0.f);
        *loss = policy_loss_grad<float>(m, ts, g);
        std::memcpy(grad, g.data(), g.size() * sizeof(float));
    });
}

struct AdamC {
    double lr, beta1, beta2, eps, wd;
};

void* sgref_adamw_new(const AdamC* a) {
    auto* o = new AdamW();
    o->lr = a->lr;
    o->beta1 = a->beta1;
    o->beta2 = a->beta2;
    o->eps = a->eps;
    o->weight_decay = a->wd;
    return o;
}
void sgref_adamw_free(void* o) { delete static_cast<AdamW*>(o); }
int sgref_adamw_step(void* o, float* params, const float* grad, size_t n) {
    return guarded([&] { static_cast<AdamW*>(o)->step(std::span<float>(params, n), std::span<const float>(grad, n)); });
}

int sgref_draft_update(void* draft, void* model, int nseq, const int* tokens, const int* lens,
                       const float* feats, void* opt, double w_feat, double w_tok, double* terms4) {
    return guarded([&] {
        Draft& dr = *static_cast<Draft*>(draft);
        const Model& m = *static_cast<Model*>(model);
        auto seqs = seqs_from(nseq, tokens, lens, feats, m.config.d_model);
        DraftTrainBatch batch;
        for (auto& s : seqs) batch.seqs.push_back(&s);
        DraftLossTerms t = draft_update(dr, m, batch, *static_cast<AdamW*>(opt), w_feat, w_tok);
        terms4[0] = t.feature_loss;
        terms4[1] = t.token_loss;
        terms4[2] = t.total;
        terms4[3] = double(t.rows);
    });
}

// ---- checkpoints (tinylm.cpp:14-105) -------------------------------------------------
int sgref_save_checkpoint(void* model, const char* path) {
    return guarded([&] { save_checkpoint(path, *static_cast<Model*>(model)); });
}
int sgref_save_draft_checkpoint(void* draft, const char* path) {
    return guarded([&] { save_draft_checkpoint(path, *static_cast<Draft*>(draft)); });
}

}  // extern "C"

// Model with the reference's layout (tinylm.hpp:133-150) and caller-supplied weights,
// skipping init_flat's sequential Box-Muller (33 s at the 1.5B shape); used only by the
// CPU-baseline leg of bench.py, whose timing does not depend on weight values.
extern "C" void* sgref_model_new_weights(const CfgC* c, const float* flat) {
    Model* m = nullptr;
    int rc = guarded([&] {
        ModelConfig cfg = to_cfg(c);
        cfg.validate();
        m = new Model();
        m->config = cfg;
        detail::LayoutBuilder lb;
        const int d = cfg.d_model;
        m->tok_emb = lb.add("tok_emb", cfg.vocab_size, d, Init::normal);
        m->pos_emb = lb.add("pos_emb", cfg.max_seq_len, d, Init::pos_emb);
        for (int l = 0; l < cfg.n_layers; ++l) m->layers.push_back(lb.add_layer(d, cfg.d_ff));
        m->lnf_g = lb.add("lnf_g", 1, d, Init::ones);
        m->lnf_b = lb.add("lnf_b", 1, d, Init::zeros);
        m->lm_head = lb.add("lm_head", d, cfg.vocab_size, Init::normal);
        m->layout = lb.specs;
        m->flat.assign(flat, flat + lb.total);
    });
    return rc == 0 ? m : nullptr;
}
