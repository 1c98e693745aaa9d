"""Speculative REJECTION SAMPLING acceptance (north star item 3; BASELINE configs[4]) -- a mode
the reference does not have (it only has keyed strict match, drafttree.cpp:170-222; SPEC.md
lists rejection sampling as a non-goal), so parity is distributional:

* one node, many independent rounds: the emitted token's frequencies match softmax(p / T)
  (chi-square goodness of fit) whatever the draft distribution q, and with one candidate the
  acceptance rate is sum(min(p, q)) (the speculative-sampling identity);
* whole rollouts: the second generated token's marginal frequencies under rejection-sampling
  speculation match those of plain AR sampling (two-sample chi-square), speculation happened,
  and steps without a tree are bit-identical to the strict-match mode.
"""
import numpy as np
import pytest

from tests.gpu_common import SMALL, make_engine

pytestmark = pytest.mark.gpu


def _softmax(l, T):
    z = np.asarray(l, np.float64) / T
    z = np.exp(z - z.max())
    return z / z.sum()


def _chi2_sf(stat, dof):
    from scipy.stats import chi2
    return float(chi2.sf(stat, dof))


def _gof(counts, probs, min_expected=5.0):
    n = counts.sum()
    exp = probs * n
    keep = exp >= min_expected
    obs_k, exp_k = counts[keep], exp[keep]
    obs_r, exp_r = counts[~keep].sum(), exp[~keep].sum()
    stat = float(((obs_k - exp_k) ** 2 / exp_k).sum())
    dof = int(keep.sum()) - 1
    if exp_r >= min_expected:
        stat += (obs_r - exp_r) ** 2 / exp_r
        dof += 1
    return stat, dof


@pytest.fixture(scope="module")
def eng():
    e, _, _ = make_engine(SMALL, max_seqs=64, max_rows=1024)
    yield e
    e.close()


@pytest.mark.parametrize("k,T,shift", [(1, 1.0, 0.5), (3, 1.0, 2.0), (2, 0.7, 0.0), (4, 1.3, 5.0)])
def test_single_node_emits_the_target_distribution(eng, k, T, shift):
    rng = np.random.default_rng(k * 10 + int(shift))
    V = 48
    p = rng.normal(0, 1.5, V).astype(np.float32)
    q = (p + shift * rng.normal(0, 1, V)).astype(np.float32)  # shift 0: q == p
    n = 120_000
    tok, acc = eng.debug_spec_sample(p, q, k, T, n, seed=1000 + k)
    pp, qq = _softmax(p, T), _softmax(q, T)
    stat, dof = _gof(np.bincount(tok, minlength=V).astype(np.float64), pp)
    pv = _chi2_sf(stat, dof)
    print(f"k={k} T={T} shift={shift}: chi2 {stat:.1f} dof {dof} p-value {pv:.3g} accept {acc.mean():.4f}")
    assert pv > 1e-4
    if k == 1:  # P(accept) = sum(min(p, q)) = 1 - TV(p, q)
        want = float(np.minimum(pp, qq).sum())
        assert abs(acc.mean() - want) < 5 * np.sqrt(want * (1 - want) / n) + 1e-9
    if shift == 0.0:
        assert acc.mean() > 0.999  # q == p: the first candidate is always accepted


def test_rollout_marginals_match_ar_sampling(eng):
    """Second generated token: its marginal under rejection-sampling speculation == under AR."""
    prompt = [[5, 17, 200, 41, 2, 99, 7]]
    kw = dict(c_peak=512, alpha=2.0, k_max=6, l_max=3, temperature=1.0, max_new_tokens=6, want_features=False)
    q = len(prompt[0])
    ar, sp, spec_steps, acc, slots = [], [], 0, 0, 0
    for it in range(48):
        a = eng.generate(prompt, 64, mode="vanilla", seed=10_000 + it, **kw)
        r = eng.generate(prompt, 64, mode="adaptive_spec", seed=20_000 + it, acceptance="rejection", **kw)
        # EOS at the first generated token ends a sequence: its own bin (index V)
        ar += [t[q + 1] if len(t) > q + 1 else SMALL.vocab_size for t in a.tokens]
        sp += [t[q + 1] if len(t) > q + 1 else SMALL.vocab_size for t in r.tokens]
        spec_steps += sum(1 for s in r.steps if s[1] > 1)
        acc += r.total_accepted
        slots += r.total_verify_slots
    V = SMALL.vocab_size + 1
    ca = np.bincount(ar, minlength=V).astype(np.float64)
    cs = np.bincount(sp, minlength=V).astype(np.float64)
    keep = (ca + cs) >= 10
    tot_a, tot_s = ca.sum(), cs.sum()
    stat = float(sum((ca[i] * np.sqrt(tot_s / tot_a) - cs[i] * np.sqrt(tot_a / tot_s)) ** 2 / (ca[i] + cs[i])
                     for i in np.nonzero(keep)[0]))
    dof = int(keep.sum()) - 1
    pv = _chi2_sf(stat, dof)
    print(f"two-sample chi2 {stat:.1f} dof {dof} p-value {pv:.3g}; spec steps {spec_steps}, tau {acc / slots:.3f}")
    assert spec_steps > 0
    assert pv > 1e-4


def test_steps_without_tree_equal_strict_mode(eng):
    prompts = [[3, 14, 15, 92, 65, 35], [2, 71, 82, 81]]
    kw = dict(c_peak=16, temperature=1.0, seed=3, max_new_tokens=24, want_features=False)
    a = eng.generate(prompts, 4, mode="vanilla", acceptance="strict", **kw)
    b = eng.generate(prompts, 4, mode="vanilla", acceptance="rejection", **kw)
    assert a.tokens == b.tokens
    # at T = 0 the rejection mode is the greedy strict-match mode (speculation on)
    kw0 = dict(kw, temperature=0.0)
    c = eng.generate(prompts, 2, mode="adaptive_spec", acceptance="strict", **kw0)
    d = eng.generate(prompts, 2, mode="adaptive_spec", acceptance="rejection", **kw0)
    assert c.tokens == d.tokens
