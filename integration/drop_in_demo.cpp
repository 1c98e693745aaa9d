// A caller written against the reference's public C++ API only (scheduler.hpp, grpo.hpp,
// tinylm.hpp): init a model + draft, generate_dynamic_batch in vanilla and adaptive mode,
// draft_update on the result. Linked with integration/scheduler_b200.cpp it runs on the B200.
// Prints one JSON line (tests/test_gpu_drop_in.py checks it).
#include <cstdio>
#include <vector>

#include "sgrpo/grpo.hpp"
#include "sgrpo/scheduler.hpp"

using namespace sgrpo;

int main() {
    ModelConfig cfg;
    cfg.vocab_size = 512;
    cfg.d_model = 256;
    cfg.n_layers = 2;
    cfg.n_heads = 4;
    cfg.d_ff = 1024;
    cfg.max_seq_len = 192;
    cfg.seed = 1;
    Model target = init_model<float>(cfg);
    Draft draft = init_draft<float>(cfg, 1);
    Rng rng(mix_key(0, 0x9a01));
    std::vector<std::vector<int>> prompts(8);
    for (auto& p : prompts)
        for (int i = 0; i < 32; ++i) p.push_back(2 + static_cast<int>(rng.below(cfg.vocab_size - 2)));
    SchedParams sched;
    sched.c_peak = 64;
    HardwareProfile prof;
    GenOptions van;
    van.mode = DecodeMode::vanilla;
    van.seed = 7;
    van.max_new_tokens = 64;
    GenOptions ada = van;
    ada.mode = DecodeMode::adaptive_spec;
    BatchState v = generate_dynamic_batch(target, draft, prompts, 4, sched, prof, van);
    BatchState a = generate_dynamic_batch(target, draft, prompts, 4, sched, prof, ada);
    GenOptions hot = ada;  // T=1 keyed sampling: checks seed / sid plumbing through the shim
    hot.temperature = 1.0;
    BatchState h = generate_dynamic_batch(target, draft, prompts, 4, sched, prof, hot);
    bool same = v.seqs.size() == a.seqs.size();
    long long gen = 0;
    for (size_t i = 0; same && i < v.seqs.size(); ++i) {
        same = v.seqs[i].tokens == a.seqs[i].tokens;
        gen += static_cast<long long>(a.seqs[i].tokens.size()) - a.seqs[i].prompt_len;
    }
    DraftTrainBatch batch;
    long long rows = 0;
    for (const auto& s : a.seqs) {
        batch.seqs.push_back(&s);
        rows += static_cast<long long>(s.tokens.size()) >= 3 ? static_cast<long long>(s.tokens.size()) - 2 : 0;
    }
    std::vector<float> before = draft.flat;
    AdamW opt;
    DraftLossTerms t = draft_update(draft, target, batch, opt);
    size_t changed = 0;
    for (size_t i = 0; i < before.size(); ++i) changed += before[i] != draft.flat[i];
    auto dump = [](const char* key, const std::vector<std::vector<int>>& rows) {
        std::printf("\"%s\": [", key);
        for (size_t i = 0; i < rows.size(); ++i) {
            std::printf("%s[", i ? ", " : "");
            for (size_t j = 0; j < rows[i].size(); ++j) std::printf("%s%d", j ? ", " : "", rows[i][j]);
            std::printf("]");
        }
        std::printf("], ");
    };
    auto toks = [](const BatchState& b) {
        std::vector<std::vector<int>> r;
        for (const auto& s : b.seqs) r.push_back(s.tokens);
        return r;
    };
    std::printf("{");
    dump("prompts", prompts);
    dump("tokens_t0", toks(a));
    dump("tokens_t1", toks(h));
    std::printf(
        "\"seqs\": %zu, \"generated\": %lld, \"lossless\": %s, \"tau\": %.6f, \"steps\": %zu, \"spec_steps\": %zu, "
        "\"draft_rows\": %lld, \"expected_rows\": %lld, \"feature_loss\": %.6g, \"token_loss\": %.6g, "
        "\"draft_params_changed\": %zu, \"first_tokens\": [%d, %d, %d, %d]}\n",
        a.seqs.size(), gen, same ? "true" : "false", a.stats.tau(), a.stats.steps.size(),
        static_cast<size_t>(std::count_if(a.stats.steps.begin(), a.stats.steps.end(),
                                          [](const StepRecord& r) { return r.cfg.n_verify > 1; })),
        t.rows, rows, t.feature_loss, t.token_loss, changed, a.seqs[0].tokens[32], a.seqs[0].tokens[33],
        a.seqs[0].tokens[34], a.seqs[0].tokens[35]);
    return same ? 0 : 1;
}
