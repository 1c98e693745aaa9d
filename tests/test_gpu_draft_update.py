"""GPU online draft learning (draft_update, grpo.cpp:177-186) vs the oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.gpu_common import SMALL, make_engine, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def batch():
    m, d = O.init_model(SMALL), O.init_draft(SMALL, 1)
    rng = np.random.default_rng(7)
    prompts = [rng.integers(2, SMALL.vocab_size, size=int(rng.integers(4, 12))).tolist() for _ in range(4)]
    res = O.generate_dynamic_batch(m, d, prompts, 2, c_peak=16, mode="vanilla", seed=3, max_new_tokens=30)
    return m, d, res.seqs


def test_loss_and_gradient_match_oracle(batch):
    m, d, seqs = batch
    e, _, _ = make_engine(SMALL)
    (fl, tl, tot, rows, secs), grad = e.draft_update([(s.tokens, s.features) for s in seqs], apply_step=False,
                                                     want_grad=True)
    g_ref = np.zeros(d.flat.size, np.float32)
    ref = O.draft_loss_grad(d, m, seqs, 1.0, 0.1, g_ref)
    print("terms gpu", fl, tl, rows, "ref", ref, "grad rel-L2", rel_l2(grad, g_ref), "secs", secs)
    assert rows == ref[3]
    np.testing.assert_allclose([fl, tl], ref[:2], rtol=2e-2)
    assert rel_l2(grad, g_ref) < 5e-2
    # per tensor (tinylm.hpp layout): every block of the gradient matches
    for name, (off, r, c) in d.offsets().items():
        assert rel_l2(grad[off:off + r * c], g_ref[off:off + r * c]) < 8e-2, name


def test_adamw_step_matches_oracle(batch):
    m, d, seqs = batch
    e, _, _ = make_engine(SMALL)
    e.draft_update([(s.tokens, s.features) for s in seqs], lr=1e-3)
    got = e.download_draft()
    d2 = d.copy()
    O.draft_update(d2, m, seqs, O.AdamW(lr=1e-3))
    diff = np.abs(got - d2.flat)
    frac = float((diff > 1e-6).mean())
    print("weights after one AdamW step: frac |dw|>1e-6", frac, "max", diff.max())
    # AdamW's first step moves every weight by ~lr*sign(g): bf16 gradients can only flip
    # the sign of near-zero gradient coordinates
    assert frac < 0.05
    assert diff.max() <= 2e-3 + 1e-6


def test_last_rollout_path_is_bitwise_the_host_path():
    m, d = O.init_model(SMALL), O.init_draft(SMALL, 1)
    e, _, _ = make_engine(SMALL)
    rng = np.random.default_rng(2)
    prompts = [rng.integers(2, SMALL.vocab_size, size=6).tolist() for _ in range(3)]
    r = e.generate(prompts, 2, c_peak=16, mode="vanilla", seed=5, max_new_tokens=20)
    _, g_dev = e.draft_update(None, apply_step=False, want_grad=True)
    _, g_host = e.draft_update(list(zip(r.tokens, r.features)), apply_step=False, want_grad=True)
    assert np.array_equal(g_dev, g_host)


def test_online_learning_raises_acceptance():
    """grpo.cpp:329-345: repeated rollout -> draft_update on the same prompts raises tau."""
    e, m, d = make_engine(SMALL)
    rng = np.random.default_rng(4)
    prompts = [rng.integers(2, SMALL.vocab_size, size=6).tolist() for _ in range(4)]
    kw = dict(c_peak=16, alpha=2.0, k_max=3, l_max=2, mode="adaptive_spec", seed=9, max_new_tokens=24)
    taus = []
    for it in range(30):
        r = e.generate(prompts, 2, **kw)
        taus.append(r.tau())
        e.draft_update(None, lr=3e-3)
    print("tau trajectory", [round(t, 3) for t in taus[::5]], taus[-1])
    assert taus[-1] > taus[0] + 0.1
