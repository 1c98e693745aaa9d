"""Randomised losslessness stress over the attention tilings and schedules: shared-prompt tiles
(group members, prompts of one or more 64-key blocks), tree-verify tiles (8-16 rows), the
weight-balanced and count-balanced splits, T in {0, 1}, fixed and adaptive schedules. Every
speculative rollout must equal the vanilla rollout bit for bit."""
import numpy as np
import pytest

from tests.gpu_common import C1, make_engine

pytestmark = pytest.mark.gpu


def test_random_rollouts_lossless():
    e, _, _ = make_engine(C1, max_seqs=32, max_rows=2048)
    rng = np.random.default_rng(31337)
    for trial in range(24):
        n_q = int(rng.integers(1, 5))
        g = int(rng.choice([1, 2, 4, 8]))
        plen = int(rng.choice([5, 40, 64, 70, 129]))
        prompts = [rng.integers(2, C1.vocab_size, size=plen).tolist() for _ in range(n_q)]
        temp = float(rng.choice([0.0, 1.0]))
        new = int(rng.integers(8, 40))
        caps = [int(rng.integers(1, new + 1)) for _ in range(n_q * g)]
        kw = dict(temperature=temp, seed=trial, max_new_tokens=new, want_features=False, seq_max_new=caps)
        van = e.generate(prompts, g, c_peak=4, mode="vanilla", **kw)
        if rng.random() < 0.5:
            n_v = int(rng.integers(2, 64))
            k = int(rng.integers(1, min(10, n_v - 1) + 1))
            l = int(rng.integers(1, 7))
            spec = e.generate(prompts, g, c_peak=4, mode="fixed_spec", fixed=(n_v, k, l), **kw)
        else:
            spec = e.generate(prompts, g, c_peak=int(rng.integers(8, 300)), mode="adaptive_spec", **kw)
        assert spec.tokens == van.tokens, trial
        assert spec.hit_eos == van.hit_eos, trial


def test_wide_head_rollouts_lossless():
    """> 16 heads: tree-verify and draft-level tiles also take the prefix-end block (attention.cu,
    AttnTileDev.bsh), whose chunks past the common prefix are staged once per row. Prompt lengths
    put the prefix end at every offset inside a 64-key block; spec must equal vanilla bit for bit."""
    from oracle import oracle as O
    from tests.gpu_common import capi
    cfg = O.ModelConfig(vocab_size=512, d_model=28 * 64, n_layers=2, n_heads=28, d_ff=1024, max_seq_len=320, seed=2)
    c = capi()
    e = c.Engine(cfg, 1, 0, 16, 2048, 10, 6)
    e.init_random(2024)
    rng = np.random.default_rng(7)
    for trial in range(8):
        n_q = int(rng.integers(1, 4))
        g = int(rng.choice([1, 2, 4]))
        plen = int(rng.integers(60, 200))
        prompts = [rng.integers(2, cfg.vocab_size, size=plen).tolist() for _ in range(n_q)]
        kw = dict(temperature=float(trial % 2), seed=trial, max_new_tokens=int(rng.integers(20, 60)), want_features=False)
        van = e.generate(prompts, g, c_peak=4, mode="vanilla", **kw)
        spec = e.generate(prompts, g, c_peak=int(rng.choice([64, 211, 300])), mode="adaptive_spec", **kw)
        assert spec.tokens == van.tokens, trial
        assert sum(1 for s in spec.steps if s[1] > 1) > 0, trial  # speculative steps ran
