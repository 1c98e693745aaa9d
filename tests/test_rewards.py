"""GRPO rewards and group advantages (src/grpo.cpp:99-136): the numpy oracle against golden
fixtures from the compiled reference (CPU), and the device kernels against the same fixtures
and a rollout's own token table (GPU)."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rewards.json")))
EPS = float.fromhex(GOLD["eps_var"])


def test_oracle_rewards_match_reference_golden():
    for c in GOLD["rewards"]:
        assert O.compute_reward(c["a"], c["b"], c["resp"]) == float.fromhex(c["reward"]), c


def test_oracle_advantages_match_reference_golden_bitwise():
    for grp in GOLD["advantages"]:
        r = [float.fromhex(x) for x in grp["rewards"]]
        adv = O.standardize_advantages(r, EPS)
        if not grp["valid"]:
            assert adv is None
        else:
            assert [a.hex() for a in adv] == grp["adv"], grp
    with pytest.raises(ValueError):
        O.standardize_advantages([1.0], EPS)


def _golden_sequences(g):
    """Reward cases grouped g at a time, each behind a short random prompt."""
    rng = np.random.default_rng(g)
    cases = GOLD["rewards"][: (len(GOLD["rewards"]) // g) * g]
    toks, plens, answers, want = [], [], [], []
    for i in range(0, len(cases), g):
        grp = cases[i:i + g]
        # one answer per group: members score against the group's query (a + b of the first)
        a, b = grp[0]["a"], grp[0]["b"]
        answers.append(a + b)
        for c in grp:
            p = rng.integers(2, 14, size=int(rng.integers(1, 6))).tolist()
            toks.append(p + c["resp"])
            plens.append(len(p))
            want.append(O.compute_reward(a, b, c["resp"]))
    return toks, plens, answers, want


@pytest.mark.gpu
@pytest.mark.parametrize("g", [2, 3, 4, 8])
def test_device_rewards_and_advantages_bit_exact(g):
    from paper_2509_21792_b200 import capi
    toks, plens, answers, want = _golden_sequences(g)
    r, adv, valid = capi.debug_group_advantages(toks, plens, answers, g, EPS)
    assert r.tolist() == want
    for b in range(len(answers)):
        ref = O.standardize_advantages(want[b * g:(b + 1) * g], EPS)
        assert bool(valid[b]) == (ref is not None)
        if ref is not None:
            assert [x.hex() for x in adv[b * g:(b + 1) * g]] == [x.hex() for x in ref]


@pytest.mark.gpu
def test_device_advantages_of_a_rollout():
    """sgb_group_advantages reads the last rollout's tokens straight from HBM."""
    from tests.gpu_common import C1, make_engine, capi
    e, _, _ = make_engine(C1, max_seqs=8)
    rng = np.random.default_rng(5)
    pr = [rng.integers(2, 14, size=8).tolist() for _ in range(2)]
    res = e.generate(pr, 4, c_peak=16, mode="adaptive_spec", temperature=1.0, seed=3, max_new_tokens=24)
    answers = [int(rng.integers(0, 100)) for _ in pr]
    r, adv, valid = e.group_advantages(answers, 4)
    want = [O.compute_reward(answers[s // 4], 0, t[p:]) for s, (t, p) in enumerate(zip(res.tokens, res.prompt_len))]
    assert r.tolist() == want
    for b in range(2):
        ref = O.standardize_advantages(want[b * 4:(b + 1) * 4], EPS)
        assert bool(valid[b]) == (ref is not None)
    with pytest.raises(ValueError):
        e.group_advantages(answers + [1], 4)  # not the last rollout's shape
