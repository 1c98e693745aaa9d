// The reference's own strategy benchmark, unmodified: sgrpo::bench (harness.cpp:89-154) runs
// train_loop (grpo.cpp:280-410) once per strategy from one shared initial target/draft and
// checks that every strategy emitted identical token streams (speculation is lossless). This
// main only parses the reference's TrainConfig JSON (train_config_from_json, grpo.cpp:454) and
// prints the reference's bench_table plus one JSON summary line; exit code 3 on a token
// mismatch, like the reference CLI's bench command (tools/sgrpo.cpp:16-17).
//
// Linked two ways (integration/Makefile):
//   ref_bench      -- with integration/scheduler_b200.cpp: generate_dynamic_batch and
//                     draft_update run on the B200 (libsgrpo_b200.so); everything else
//                     (train_loop, policy_update, rewards, harness) is the reference's code
//   ref_bench_cpu  -- the reference alone (its CPU generate_dynamic_batch / draft_update)
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "sgrpo/grpo.hpp"
#include "sgrpo/harness.hpp"

extern "C" __attribute__((weak)) void sgb_shim_counters(long long*, long long*, long long*, long long*, long long*);

using namespace sgrpo;

static unsigned long long fnv(const std::vector<std::vector<std::vector<int>>>& t) {
    unsigned long long h = 1469598103934665603ull;
    for (const auto& it : t)
        for (const auto& s : it) {
            h = (h ^ s.size()) * 1099511628211ull;
            for (int x : s) h = (h ^ static_cast<unsigned>(x)) * 1099511628211ull;
        }
    return h;
}

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s config.json strategy strategy [...]\n", argv[0]);
        return 2;
    }
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    TrainConfig cfg = train_config_from_json(ss.str());
    std::vector<std::string> names(argv + 2, argv + argc);
    BenchResult r = bench(names, cfg);
    std::printf("%s", bench_table(r).c_str());
    std::printf("{\"tokens_identical\": %s, \"entries\": [", r.tokens_identical ? "true" : "false");
    for (size_t i = 0; i < r.entries.size(); ++i) {
        const auto& e = r.entries[i];
        long long gen = 0, accepted = e.result.total_accepted;
        for (const auto& it : e.result.gen_tokens)
            for (const auto& s : it) gen += static_cast<long long>(s.size());
        std::printf("%s{\"name\": \"%s\", \"gen_time_s\": %.6g, \"update_time_s\": %.6g, \"tau\": %.6f, "
                    "\"gen_sr\": %.6f, \"e2e_sr\": %.6f, \"iterations\": %zu, \"accepted\": %lld, "
                    "\"tokens_hash\": \"%016llx\", \"reward_mean_last\": %.6f}",
                    i ? ", " : "", e.name.c_str(), e.metrics.gen_time_s, e.metrics.update_time_s, e.metrics.tau,
                    e.metrics.gen_sr, e.metrics.e2e_sr, e.result.trace.size(), accepted, fnv(e.result.gen_tokens),
                    e.result.trace.empty() ? 0.0 : e.result.trace.back().reward_mean);
    }
    std::printf("]");
    long long pol = 0;
    for (const auto& e : r.entries)
        for (const auto& it : e.result.trace) pol += it.policy_skipped ? 0 : 1;
    std::printf(", \"policy_steps\": %lld", pol);
    if (sgb_shim_counters) {
        long long ro, up, tu, du, pu;
        sgb_shim_counters(&ro, &up, &tu, &du, &pu);
        std::printf(", \"device\": {\"rollouts\": %lld, \"draft_updates\": %lld, \"target_uploads\": %lld, "
                    "\"draft_uploads\": %lld, \"policy_updates\": %lld}", ro, up, tu, du, pu);
    }
    std::printf("}\n");
    return r.tokens_identical ? 0 : 3;
}
