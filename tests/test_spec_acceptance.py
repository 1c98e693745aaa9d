"""The reference SPEC's acceptance criteria that touch the rollout path and ship no test
(SPEC.md "ACCEPTANCE CRITERIA"):

  1. lossless: >= 50 seeded prompts, T=0 adaptive speculation == vanilla greedy for every
     (alpha, k_max, l_max) in a 3x3x3 grid, exact;
  6. tau accounting: streaming tau equals the event-log recount; hand fixture 24 accepted
     over b_cur [4, 3, 1] -> 3.0;
  7. gradient check: the draft loss matches central finite differences at 50 random
     coordinates, relative error < 1e-3 (on the fp64 oracle the device gradient is pinned to);
 10. zero target forwards during draft_update.
"""
import numpy as np
import pytest

from oracle import oracle as O


def test_tau_hand_fixture():
    r = O.GenResult(seqs=[], steps=[(0, 4, 1, 0, 0, 12), (1, 3, 1, 0, 0, 9), (2, 1, 1, 0, 0, 3)],
                    events=[], total_accepted=24, total_verify_slots=4 + 3 + 1)
    assert r.tau() == 3.0
    with pytest.raises(ArithmeticError):
        O.GenResult(seqs=[], steps=[], events=[], total_accepted=0, total_verify_slots=0).tau()


def test_draft_loss_matches_central_finite_differences(monkeypatch):
    """grpo.hpp:278-344 restated in oracle.draft_loss_grad, evaluated in fp64."""
    monkeypatch.setattr(O, "F32", np.float64)
    cfg = O.ModelConfig(vocab_size=48, d_model=32, n_layers=2, n_heads=2, d_ff=64, max_seq_len=24, seed=3)
    t0, d0 = O.init_model(cfg), O.init_draft(cfg, 1)
    tgt = O.Params(cfg, t0.specs, t0.flat.astype(np.float64), t0.n_layers)
    dr = O.Params(cfg, d0.specs, d0.flat.astype(np.float64) * 20, d0.n_layers)  # non-trivial gradients
    rng = np.random.default_rng(0)
    seqs = []
    for n in (9, 12):
        seqs.append(O.SeqResult(id=len(seqs), tokens=rng.integers(2, 48, size=n).tolist(), prompt_len=3,
                                hit_eos=False, features=rng.standard_normal((n - 1, 32))))
    g = np.zeros(dr.flat.size)
    O.draft_loss_grad(dr, tgt, seqs, grad_flat=g)

    def loss(flat):
        return O.draft_loss_grad(O.Params(cfg, dr.specs, flat, dr.n_layers), tgt, seqs,
                                 grad_flat=np.zeros(flat.size))[2]

    idx = rng.choice(np.flatnonzero(np.abs(g) > 1e-6), 50, replace=False)
    for i in idx:
        h = 1e-5 * max(1.0, abs(dr.flat[i]))
        fp, fm = dr.flat.copy(), dr.flat.copy()
        fp[i] += h
        fm[i] -= h
        fd = (loss(fp) - loss(fm)) / (2 * h)
        assert abs(fd - g[i]) <= 1e-3 * max(abs(fd), abs(g[i])), (i, fd, g[i])


@pytest.mark.gpu
def test_lossless_over_50_prompts_and_27_schedules():
    from tests.gpu_common import C1, make_engine
    e, _, _ = make_engine(C1, max_seqs=50)
    rng = np.random.default_rng(2025)
    prompts = [rng.integers(2, C1.vocab_size, size=int(rng.integers(4, 24))).tolist() for _ in range(50)]
    kw = dict(temperature=0.0, seed=11, max_new_tokens=16, want_features=False)
    van = e.generate(prompts, 1, c_peak=4, mode="vanilla", **kw)
    for alpha in (1.0, 2.0, 4.0):
        for k_max in (2, 5, 10):
            for l_max in (1, 3, 6):
                # c_peak 160 over 50 sequences: N_verify = 3 at the start, up to 160 as they finish
                r = e.generate(prompts, 1, c_peak=160, alpha=alpha, k_max=k_max, l_max=l_max,
                               mode="adaptive_spec", **kw)
                assert r.tokens == van.tokens, (alpha, k_max, l_max)


@pytest.mark.gpu
def test_tau_streaming_equals_event_recount():
    from tests.gpu_common import SMALL, make_engine
    e, _, _ = make_engine(SMALL, max_seqs=16)
    rng = np.random.default_rng(7)
    for run in range(20):
        n, g = int(rng.integers(1, 5)), int(rng.integers(1, 4))
        prompts = [rng.integers(2, SMALL.vocab_size, size=int(rng.integers(2, 9))).tolist() for _ in range(n)]
        r = e.generate(prompts, g, c_peak=int(rng.integers(2, 40)), mode="adaptive_spec",
                       temperature=float(rng.choice([0.0, 1.0])), seed=run, max_new_tokens=int(rng.integers(4, 30)),
                       want_features=False)
        # per-step records (b_cur, N, K, L, accepted): the streaming sums, recounted from the log
        assert r.total_verify_slots == sum(s[0] for s in r.steps)
        assert r.total_accepted == sum(s[4] for s in r.steps)
        # and from the committed tokens themselves (the first token is emitted by the prefill)
        assert r.total_accepted == sum(len(t) - p - 1 for t, p in zip(r.tokens, r.prompt_len))
        assert r.tau() == sum(s[4] for s in r.steps) / sum(s[0] for s in r.steps)


@pytest.mark.gpu
def test_draft_update_runs_zero_target_forwards():
    from tests.gpu_common import SMALL, make_engine
    e, _, _ = make_engine(SMALL, max_seqs=8)
    before = e.target_forward_calls()
    r = e.generate([[3, 4, 5], [6, 7, 8, 9]], 2, c_peak=8, mode="adaptive_spec", temperature=0.0, seed=1,
                   max_new_tokens=12)
    after_rollout = e.target_forward_calls()
    assert after_rollout - before == r.target_forwards > 0
    e.draft_update(None, lr=1e-3)
    assert e.target_forward_calls() == after_rollout
