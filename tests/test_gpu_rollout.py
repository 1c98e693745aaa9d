"""GPU rollout (generate_dynamic_batch drop-in) parity: losslessness and oracle agreement."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.gpu_common import C1, SMALL, make_engine

pytestmark = pytest.mark.gpu


def prompts_for(cfg, n, lo=3, hi=9, seed=0):
    rng = np.random.default_rng(seed)
    return [rng.integers(2, cfg.vocab_size, size=int(rng.integers(lo, hi))).tolist() for _ in range(n)]


def first_divergence(a, b):
    for i, (x, y) in enumerate(zip(a, b)):
        if x != y:
            return i
    return min(len(a), len(b)) if len(a) != len(b) else -1


@pytest.mark.parametrize("temp", [0.0, 1.0])
def test_spec_equals_vanilla_bitwise(temp):
    """Speculation is lossless: adaptive/fixed spec tokens == vanilla tokens, bit for bit."""
    e, m, d = make_engine(SMALL, max_seqs=16)
    pr = prompts_for(SMALL, 4)
    kw = dict(c_peak=16, alpha=2.0, k_max=5, l_max=3, temperature=temp, seed=7, max_new_tokens=40)
    van = e.generate(pr, 2, mode="vanilla", **kw)
    ada = e.generate(pr, 2, mode="adaptive_spec", **kw)
    fix = e.generate(pr, 2, mode="fixed_spec", fixed=(8, 4, 3), **kw)
    assert ada.tokens == van.tokens
    assert fix.tokens == van.tokens
    assert ada.hit_eos == van.hit_eos
    for r in (van, ada, fix):
        assert r.total_accepted == sum(len(t) - p - 1 for t, p in zip(r.tokens, r.prompt_len))
        assert r.total_verify_slots == sum(s[0] for s in r.steps)
    # spec verified more rows per step than vanilla
    assert max(s[1] for s in ada.steps) > 1


def _check_divergence_is_near_tie(e, m, gpu_tokens, ref_tokens, slot=15):
    """At the first token where the GPU and the fp32 oracle disagree, the oracle's margin
    between its token and the GPU's token must be explained by the bf16 logit error of
    that very row (GPU forward on the same prefix vs oracle forward)."""
    t = first_divergence(gpu_tokens, ref_tokens)
    if t < 0:
        return None
    prefix = gpu_tokens[:t]
    e.cache_reset(slot)
    lg_gpu, _ = e.forward_target(slot, prefix, list(range(len(prefix))))
    lg_ref, _ = O.forward_target(m, prefix, list(range(len(prefix))))
    g, r = gpu_tokens[t], ref_tokens[t]
    row_g, row_r = lg_gpu[-1], lg_ref[-1]
    assert int(np.argmax(row_g)) == g and int(np.argmax(row_r)) == r
    margin = float(row_r[r] - row_r[g])
    err = float(abs(row_g[r] - row_r[r]) + abs(row_g[g] - row_r[g]))
    assert margin <= err + 1e-6, (t, margin, err)
    return t, margin, err


def test_rollout_matches_oracle_up_to_bf16_near_ties():
    """GPU adaptive rollout vs the fp32 oracle. Decisions are bit-exact given identical logits
    (test_gpu_kernels); over a whole rollout the bf16 logits can only flip a greedy choice
    where the oracle's own top-2 margin is below the bf16 logit error -- checked at every
    first divergence. The controller's (N, K, L) per step equals Eqs. 1-3 of B_cur."""
    e, m, d = make_engine(SMALL, max_seqs=16)
    pr = prompts_for(SMALL, 3, seed=2)
    kw = dict(c_peak=16, alpha=2.0, k_max=5, l_max=3, temperature=0.0, seed=7, max_new_tokens=24)
    gpu = e.generate(pr, 2, mode="adaptive_spec", **kw)
    ref = O.generate_dynamic_batch(m, d, pr, 2, mode="adaptive_spec", **kw)
    for a, b in zip(gpu.tokens, ref.seqs):
        print("divergence", _check_divergence_is_near_tie(e, m, a, b.tokens))
    for b_cur, n, k, l, _ in gpu.steps:
        c = O.plan_step(16, b_cur, 2.0, 5, 3)
        assert (n, k, l) == (c.n_verify, c.k_draft, c.l_draft)
    # features of the committed prefix match the oracle's target hidden states (bf16 tol)
    for a, b, t in zip(gpu.features, ref.seqs, gpu.tokens):
        div = first_divergence(t, b.tokens)
        n = min(len(a), len(b.features), div if div >= 0 else len(a))  # feature j = state after token j
        rel = np.linalg.norm(a[:n] - b.features[:n]) / np.linalg.norm(b.features[:n])
        assert rel < 3e-2


def test_c1_vanilla_vs_oracle():
    """BASELINE configs[0] shape (d=256, L=2): GPU greedy rollout vs oracle; every first
    divergence is a bf16 near-tie; spec == vanilla bitwise."""
    e, m, d = make_engine(C1, max_seqs=8)
    pr = prompts_for(C1, 2, 32, 33, seed=4)
    kw = dict(c_peak=64, temperature=0.0, seed=7, max_new_tokens=24)
    gpu = e.generate(pr, 2, mode="vanilla", **kw)
    ref = O.generate_dynamic_batch(m, d, pr, 2, mode="vanilla", **kw)
    for a, b in zip(gpu.tokens, ref.seqs):
        print("c1 divergence", _check_divergence_is_near_tie(e, m, a, b.tokens, slot=7))
    ada = e.generate(pr, 2, mode="adaptive_spec", **kw)
    assert ada.tokens == gpu.tokens


@pytest.mark.parametrize("mode", ["vanilla", "adaptive_spec"])
def test_rollout_equals_teacher_forced_greedy(mode):
    """Every emitted token equals the argmax of a fresh full-prefix forward of the same
    sequence, bit for bit (batch-invariant kernels; catches any KV-commit/copy error)."""
    e, m, d = make_engine(C1, max_seqs=8)
    pr = prompts_for(C1, 2, 32, 33, seed=4)
    r = e.generate(pr, 2, c_peak=64, mode=mode, temperature=0.0, seed=7, max_new_tokens=24)
    assert r.tokens[0] == r.tokens[1] and r.tokens[2] == r.tokens[3]  # T=0 group members agree
    for s in range(4):
        toks = r.tokens[s]
        e.cache_reset(7)
        lg, _ = e.forward_target(7, toks[:-1], list(range(len(toks) - 1)))
        assert lg.argmax(1)[31:].tolist() == toks[32:], s


def test_group_members_share_prompt_blocks_losslessly():
    """AR steps tile the live members of a query group over their shared prompt blocks
    (prompt >= 2 full 64-key blocks here); the rollout must still equal the teacher-forced
    argmax of each sequence alone, and the speculative rollout must equal it bit for bit."""
    e, m, d = make_engine(C1, max_seqs=8)
    pr = prompts_for(C1, 2, 130, 131, seed=9)
    kw = dict(temperature=0.0, seed=7, max_new_tokens=20)
    van = e.generate(pr, 4, c_peak=4, mode="vanilla", **kw)
    ada = e.generate(pr, 4, c_peak=64, mode="adaptive_spec", **kw)
    assert ada.tokens == van.tokens
    assert max(s[1] for s in ada.steps) > 1
    for s in (0, 5):
        toks = van.tokens[s]
        e.cache_reset(7)
        lg, _ = e.forward_target(7, toks[:-1], list(range(len(toks) - 1)))
        assert lg.argmax(1)[129:].tolist() == toks[130:], s


def test_rollout_errors():
    e, m, d = make_engine(SMALL, max_seqs=4)
    with pytest.raises(ValueError):
        e.generate([], 1, c_peak=4)
    with pytest.raises(ValueError):
        e.generate([[2, 3]], 0, c_peak=4)
    with pytest.raises(ValueError):
        e.generate([[]], 1, c_peak=4)
    with pytest.raises(ValueError):
        e.generate([[2] * SMALL.max_seq_len], 1, c_peak=4)
    with pytest.raises(ValueError):
        e.generate([[2, 3]], 1, c_peak=0)
    with pytest.raises(ValueError):  # k_draft > n_verify - 1
        e.generate([[2, 3]], 1, c_peak=4, mode="fixed_spec", fixed=(2, 3, 1))


def test_gen_stats_jsonl_with_measured_step_seconds():
    """gen_stats_to_jsonl (scheduler.cpp:356-368): one record per step; the B200 build writes
    measured device seconds where the reference writes simulated ones."""
    import json as _json
    from paper_2509_21792_b200 import capi as _c
    e, _, _ = make_engine(SMALL)
    rng = np.random.default_rng(8)
    prompts = [rng.integers(2, SMALL.vocab_size, size=7).tolist() for _ in range(3)]
    r = e.generate(prompts, 2, c_peak=16, mode="adaptive_spec", seed=4, max_new_tokens=20)
    lines = _c.gen_stats_jsonl(r).splitlines()
    assert len(lines) == len(r.steps) == len(r.step_seconds)
    for i, (ln, st) in enumerate(zip(lines, r.steps)):
        j = _json.loads(ln)
        assert j["step"] == i and j["b_cur"] == st[0]
        assert (j["spec_config"]["n_verify"], j["spec_config"]["k_draft"], j["spec_config"]["l_draft"]) == st[1:4]
        assert j["accepted_total"] == st[4] and j["sim_latency_s"] > 0
    assert sum(r.step_seconds) <= r.seconds * 1.0001
