// The drop-in on the reference side: this translation unit REPLACES src/scheduler.cpp's
// generate_dynamic_batch (scheduler.cpp:236-354, decl scheduler.hpp:99-102) and grpo.cpp's
// draft_update (grpo.cpp:177-186, decl grpo.hpp:115-116) with calls into the B200 C-ABI
// (include/sgrpo_b200.h). Signatures are the reference's own, so train_loop (grpo.cpp:320),
// pretrain_draft (grpo.cpp:229) and the CLI call it unchanged. It compiles against the
// unmodified reference headers (integration/Makefile) and is exercised on the GPU by
// tests/test_gpu_drop_in.py. Link it instead of scheduler.o / grpo.o's definitions.
#include <stdexcept>
#include <string>
#include <vector>

#include "sgrpo/grpo.hpp"
#include "sgrpo/scheduler.hpp"
#include "sgrpo_b200.h"

namespace sgrpo {
namespace {

// C-ABI status -> the reference's exception types
void check(int rc) {
    if (rc == 0) return;
    const std::string m = sgb_last_error();
    switch (rc) {
        case 1: throw std::invalid_argument(m);
        case 2: throw std::out_of_range(m);
        case 4: throw std::domain_error(m);
        default: throw std::runtime_error(m);
    }
}

// One engine per process / GPU; weights re-uploaded on every call (the reference mutates
// Model::flat in policy_update, grpo.cpp:389 -- production code would version-check).
sgb_engine* engine_for(const Model& t, const Draft& d, size_t n_seqs) {
    static sgb_engine* e = nullptr;
    static size_t cap = 0;
    if (e && n_seqs > cap) {
        sgb_engine_destroy(e);
        e = nullptr;
    }
    if (!e) {
        const auto& c = t.config;
        sgb_model_config mc{c.vocab_size, c.d_model, c.n_layers, c.n_heads, c.d_ff, c.max_seq_len, c.seed};
        cap = std::max<size_t>(n_seqs, 8);
        check(sgb_engine_create(&mc, d.n_layers, /*device=*/0, static_cast<int>(cap), /*max_rows=*/2048,
                                /*k_max=*/10, /*l_max=*/6, &e));
    }
    check(sgb_upload_target(e, t.flat.data(), t.flat.size()));
    check(sgb_upload_draft(e, d.flat.data(), d.flat.size()));
    return e;
}
sgb_engine* g_last = nullptr;  // the engine holding the last rollout (draft_update consumes it)

}  // namespace

double GenStats::tau() const {  // scheduler.cpp:72-75 (this TU replaces scheduler.cpp)
    if (total_verify_slots == 0) throw std::domain_error("tau: no verification steps logged");
    return static_cast<double>(total_accepted) / static_cast<double>(total_verify_slots);
}

BatchState generate_dynamic_batch(const Model& target, const Draft& draft, const std::vector<std::vector<int>>& prompts,
                                  int g, const SchedParams& sched, const HardwareProfile& /*profile*/,
                                  const GenOptions& opts) {
    std::vector<int> flat, lens;
    for (const auto& p : prompts) {
        flat.insert(flat.end(), p.begin(), p.end());
        lens.push_back(static_cast<int>(p.size()));
    }
    const int n = static_cast<int>(prompts.size()) * g, T = target.config.max_seq_len, d = target.config.d_model;
    sgb_engine* e = engine_for(target, draft, static_cast<size_t>(std::max(n, 1)));
    g_last = e;
    sgb_gen_options o{sched.alpha, sched.k_max, sched.l_max, sched.c_peak, static_cast<int>(opts.mode),
                      opts.early_term ? 1 : 0, opts.temperature, opts.seed, opts.max_new_tokens,
                      opts.fixed.n_verify, opts.fixed.k_draft, opts.fixed.l_draft, nullptr, 1, 0, nullptr};
    constexpr int kSteps = 1 << 16;
    std::vector<int> toks(static_cast<size_t>(std::max(n, 1)) * T), len(std::max(n, 1)), plen(std::max(n, 1)),
        eos(std::max(n, 1)), rec(5 * kSteps);
    std::vector<double> step_s(kSteps);
    o.step_seconds = step_s.data();  // measured device seconds replace the cost model's
    std::vector<float> feats(static_cast<size_t>(std::max(n, 1)) * (T - 1) * d);
    sgb_rollout_stats st{};
    check(sgb_rollout(e, flat.data(), lens.data(), static_cast<int>(prompts.size()), g, &o, toks.data(), len.data(),
                      plen.data(), eos.data(), feats.data(), rec.data(), kSteps, &st));
    BatchState bs;
    for (int s = 0; s < n; ++s) {
        SeqResult r;
        r.id = s;
        r.tokens.assign(toks.begin() + static_cast<size_t>(s) * T, toks.begin() + static_cast<size_t>(s) * T + len[s]);
        r.prompt_len = plen[s];
        r.hit_eos = eos[s] != 0;
        r.features.assign(feats.begin() + static_cast<size_t>(s) * (T - 1) * d,
                          feats.begin() + static_cast<size_t>(s) * (T - 1) * d + static_cast<size_t>(len[s] - 1) * d);
        bs.seqs.push_back(std::move(r));
    }
    for (int i = 0; i < st.n_steps && i < kSteps; ++i) {
        SpecConfig c;
        c.n_verify = rec[5 * i + 1];
        c.k_draft = rec[5 * i + 2];
        c.l_draft = rec[5 * i + 3];
        bs.stats.steps.push_back(StepRecord{i, rec[5 * i], c, rec[5 * i + 4], step_s[i]});
    }
    bs.stats.total_accepted = st.total_accepted;
    bs.stats.total_verify_slots = st.total_verify_slots;
    bs.stats.total_sim_s = st.seconds;
    return bs;
}

DraftLossTerms draft_update(Draft& draft, const Model& target, const DraftTrainBatch& batch, AdamW& opt, double w_feat,
                            double w_tok) {
    // host sequences -> device (the last-rollout fast path is sgb_draft_update_last)
    sgb_engine* e = g_last ? g_last : engine_for(target, draft, batch.seqs.size());
    std::vector<int> toks, lens;
    std::vector<float> feats;
    for (const SeqResult* s : batch.seqs) {
        toks.insert(toks.end(), s->tokens.begin(), s->tokens.end());
        lens.push_back(static_cast<int>(s->tokens.size()));
        feats.insert(feats.end(), s->features.begin(), s->features.end());
    }
    sgb_adamw a{opt.lr, opt.beta1, opt.beta2, opt.eps, opt.weight_decay, w_feat, w_tok, 0, 1, 0};
    sgb_draft_terms t{};
    check(sgb_draft_update(e, static_cast<int>(lens.size()), toks.data(), lens.data(), feats.data(), &a, nullptr, &t));
    check(sgb_download_draft(e, draft.flat.data(), draft.flat.size()));  // mirror the fp32 master copy
    ++opt.t;                                                              // moments live on the device
    return DraftLossTerms{t.feature_loss, t.token_loss, t.total, t.rows};
}

}  // namespace sgrpo
