"""Pins the numpy oracle (oracle/oracle.py) against the real reference.

Two sources of truth, both independent of the numpy oracle and of the CUDA path:
  * golden vectors written by the compiled reference (tests/golden/make_golden.py via
    oracle/_ref/libsgrpo_ref.so);
  * the known-answer tests of the reference's own suite (proj/tests/test_drafttree.cpp,
    proj/tests/test_tinylm.cpp) and the SPEC.md:295-330 scheduler examples.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(G, name)) as f:
        return json.load(f)


def cfg_from(d):
    return O.ModelConfig(**d)


# ---------------------------------------------------------------- rng (rng.hpp:9-65)
def test_rng_golden():
    g = load("rng.json")
    for seed, vals in g["splitmix"].items():
        st = int(seed)
        for v in vals:
            x, st = O.splitmix64(st)
            assert x == int(v)
    for a, b, v in g["mix_key"]:
        assert O.mix_key(int(a), int(b)) == int(v)
    for seed, vals in g["uniform"].items():
        r = O.Rng(int(seed))
        assert [r.uniform() for _ in vals] == vals
    for seed, vals in g["normal"].items():
        r = O.Rng(int(seed))
        assert [r.normal() for _ in vals] == vals
        assert O.normal_stream(int(seed), len(vals)).tolist() == vals
    for seed, vals in g["below"].items():
        r = O.Rng(int(seed))
        assert [r.below(510) for _ in vals] == vals


# ---------------------------------------------------------------- init (tinylm.hpp:83-189)
def test_init_tiny_bit_exact():
    z = np.load(os.path.join(G, "init_tiny.npz"))
    h = load("init_hashes.json")
    cfg = cfg_from(h["tiny"])
    assert np.array_equal(O.init_model(cfg).flat, z["model"])
    assert np.array_equal(O.init_draft(cfg, 1).flat, z["draft1"])
    assert np.array_equal(O.init_draft(cfg, 2).flat, z["draft2"])


def test_init_c1_and_small_hashes():
    h = load("init_hashes.json")
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    for key in ("c1", "small"):
        cfg = cfg_from(h[key])
        assert sha(O.init_model(cfg).flat) == h[f"{key}_model_sha256"]
        assert sha(O.init_draft(cfg, 1).flat) == h[f"{key}_draft_sha256"]


def test_param_count_shape_sum():
    # test_tinylm.cpp:25-50 (independent shape sum)
    c = O.ModelConfig(32, 64, 2, 4, 256, 64, 3)
    expect = 32 * 64 + 64 * 64 + 2 * (64 + 64 + 4 * 64 * 64 + 64 + 64 + 64 * 256 + 256 * 64) + 64 + 64 + 64 * 32
    assert O.param_count(c) == expect


def test_invalid_dimensions_rejected():
    for bad in (dict(d_model=63), dict(vocab_size=3), dict(max_seq_len=4)):
        kw = dict(vocab_size=16, d_model=32, n_layers=2, n_heads=4, d_ff=64, max_seq_len=32, seed=1)
        kw.update(bad)
        with pytest.raises(ValueError):
            O.init_model(O.ModelConfig(**kw))


# ---------------------------------------------------------------- forward (tinylm.hpp:305-563)
def test_forward_golden():
    z = np.load(os.path.join(G, "forward_tiny.npz"))
    meta = load("forward_tiny.json")
    cfg = cfg_from(meta["config"])
    m = O.init_model(cfg)
    lg, hd = O.forward_target(m, meta["tokens"], list(range(8)))
    np.testing.assert_allclose(lg, z["full_logits"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(hd, z["full_hidden"], rtol=1e-5, atol=1e-5)
    cache = O.KvCache(cfg.n_layers, cfg.d_model)
    O.forward_target(m, [2, 7, 5], [0, 1, 2], None, cache)
    lg, hd = O.forward_target(m, [4, 6, 8, 9], [3, 4, 4, 5], z["tree_mask"], cache)
    np.testing.assert_allclose(lg, z["tree_logits"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(np.stack(cache.k), z["tree_cache_k"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(np.stack(cache.v), z["tree_cache_v"], rtol=1e-5, atol=1e-6)
    dr = O.init_draft(cfg, 1)
    dc = O.KvCache(1, cfg.d_model)
    f, l, _, _ = O.forward_draft_rows(dr, m, [3, 5, 7, 2, 9], z["draft_in_feats"], [1, 2, 3, 4, 5], cache=dc)
    np.testing.assert_allclose(f, z["draft_feats"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(l, z["draft_logits"], rtol=1e-5, atol=1e-6)


def test_incremental_equals_full():
    # test_tinylm.cpp:83-117
    cfg = O.ModelConfig(16, 32, 2, 4, 64, 32, 11)
    m = O.init_model(cfg)
    toks = [2, 9, 4, 13, 6, 3, 7, 12]
    full, _ = O.forward_target(m, toks, list(range(8)))
    cache = O.KvCache(2, 32)
    done = 0
    for chunk in (3, 1, 4):
        lg, _ = O.forward_target(m, toks[done:done + chunk], list(range(done, done + chunk)), None, cache)
        np.testing.assert_allclose(lg, full[done:done + chunk], rtol=1e-5, atol=1e-6)
        done += chunk


def test_forward_errors():
    m = O.init_model(O.ModelConfig(16, 32, 2, 4, 64, 32, 1))
    with pytest.raises(IndexError):
        O.forward_target(m, [2], [32])
    with pytest.raises(ValueError):
        O.forward_target(m, [16], [0])


def test_gather_tail_keeps_rows():
    # test_tinylm.cpp:159-176
    m = O.init_model(O.ModelConfig(16, 32, 2, 4, 64, 32, 5))
    c = O.KvCache(2, 32)
    O.forward_target(m, [3, 4, 5, 6, 7], list(range(5)), None, c)
    ref = c.copy()
    c.gather_tail(1, [0, 2])
    assert c.len == 3
    assert np.array_equal(c.k[0][1], ref.k[0][1]) and np.array_equal(c.k[0][2], ref.k[0][3])


# ---------------------------------------------------------------- sampling (tinylm.hpp:591-628)
def test_sample_token_known_answers():
    # test_tinylm.cpp:213-235
    assert O.sample_token([0.0, 3.0, 1.0], 0.0, 1) == 1
    assert O.sample_token([2.0, 2.0, 0.0], 0.0, 1) == 0
    with pytest.raises(ArithmeticError):
        O.sample_token([-np.inf] * 3, 0.0, 1)
    p1 = math.exp(10.0) / (1.0 + math.exp(10.0))
    hits = sum(O.sample_token([0.0, 10.0], 1.0, O.mix_key(42, i)) == 1 for i in range(4000))
    assert abs(hits / 4000 - p1) < 0.02


# ---------------------------------------------------------------- tree (drafttree.cpp)
def test_max_candidates_known_answers():
    # test_drafttree.cpp:47-53
    assert [O.max_candidates(k, l) for k, l in [(3, 3), (1, 1), (7, 3), (0, 5), (4, 1)]] == [22, 2, 106, 1, 5]


def _toy(token):
    probs = {0: [.1, .5, .3, .1], 1: [.05, .05, .2, .7], 2: [.25] * 4, 3: [.7, .1, .1, .1]}
    return [math.log(p) for p in probs[token]]


def test_toy_tree_exact():
    # test_drafttree.cpp:80-103
    t = O.expand_tree_with(0, 2, 2, lambda t, n: _toy(t[n].token))
    assert [(n.token, n.parent) for n in t] == [(0, -1), (1, 0), (2, 0), (3, 1), (2, 1), (0, 2), (1, 2)]
    np.testing.assert_allclose([n.confidence for n in t], [1, .5, .3, .35, .10, .075, .075])


def test_rerank_fixture_and_walk():
    # test_drafttree.cpp:118-126, 212-271
    t = [O.DraftNode(5, -1, 0, 0, 1.0), O.DraftNode(1, 0, 1, math.log(.6), .6),
         O.DraftNode(2, 0, 1, math.log(.3), .3), O.DraftNode(3, 1, 2, math.log(.7), .42)]
    assert O.rerank_candidates(t, 3)[0] == [0, 1, 3]
    t = O.expand_tree_with(0, 2, 2, lambda t, n: _toy(t[n].token))
    sel, _ = O.rerank_candidates(t, 7)

    def row(a):
        r = np.zeros(6, np.float32)
        r[a] = 5
        return r
    rows = [row(0)] * 7
    rows[0], rows[1], rows[3] = row(1), row(3), row(2)
    vr = O.verify(t, sel, np.stack(rows), vocab=6)
    assert vr.accepted_tokens == [1, 3, 2] and vr.accepted_rows == [0, 1, 3] and vr.bonus_token == 2


def test_closure_violation_rejected():
    t = [O.DraftNode(1, -1, 0), O.DraftNode(2, 0, 1), O.DraftNode(3, 1, 2)]
    with pytest.raises(ValueError):
        O.build_tree_mask(t, [0, 2])


def test_trees_golden():
    for case in load("trees.json"):
        calls = iter(case["calls"])
        t = O.expand_tree_with(case["root"], case["k"], case["l"], lambda tr, n: next(calls))
        assert [n.token for n in t] == case["tok"]
        assert [n.parent for n in t] == case["par"]
        assert [n.depth for n in t] == case["dep"]
        assert [n.log_prob for n in t] == case["lp"]
        assert [n.confidence for n in t] == case["conf"]
        for ent in case["rerank"]:
            sel, mask = O.rerank_candidates(t, ent["n_verify"])
            assert sel == ent["sel"]
            assert mask.astype(int).tolist() == ent["mask"]
            lg = np.asarray(ent["logits"], np.float32)
            for v in ent["verify"]:
                vr = O.verify(t, sel, lg, None, case["vocab"], v["temp"], v["seed"], v["root_pos"])
                assert vr.accepted_tokens == v["tokens"]
                assert vr.accepted_rows == v["rows"]
                assert vr.bonus_token == v["bonus"] and vr.accepted_len == v["len"]


# ---------------------------------------------------------------- controller (scheduler.cpp:14-54)
def test_spec_scheduler_examples():
    # SPEC.md:295-330 (verified on the compiled reference)
    assert O.compute_n_verify(64, 16) == 4 and O.compute_n_verify(64, 128) == 1
    assert O.compute_n_verify(600, 7) == 85
    assert O.compute_k_draft(8, 10) == 7 and O.compute_k_draft(64, 10) == 10 and O.compute_k_draft(1, 10) == 0
    assert O.compute_l_draft(16, 2, 6, 5) == 3 and O.compute_l_draft(64, 1, 6, 5) == 6
    assert O.compute_l_draft(2, 4, 6, 1) == 1
    c = O.plan_step(64, 64)
    assert (c.n_verify, c.k_draft, c.l_draft) == (1, 0, 0)
    c = O.plan_step(64, 1, 2, 10, 6)
    assert (c.n_verify, c.k_draft, c.l_draft) == (64, 10, 5)


def test_plan_step_table_golden():
    for c, b, a, km, lm, n, k, l in load("plan_step.json"):
        try:
            s = O.plan_step(c, b, a, km, lm)
            got = (s.n_verify, s.k_draft, s.l_draft)
        except ValueError:
            got = (-1, -1, -1)
        assert got == (n, k, l), (c, b, a, km, lm)


# ---------------------------------------------------------------- rollout (scheduler.cpp:236-354)
def _gen(g, run):
    cfg = cfg_from(g["config"])
    m, d = O.init_model(cfg), O.init_draft(cfg, 1)
    kw = dict(run["kw"])
    fixed = kw.pop("fixed")
    return O.generate_dynamic_batch(m, d, g["prompts"], g["g"], fixed=O.SpecConfig(*fixed, c_peak=kw["c_peak"]), **kw)


def test_generate_small_golden():
    g = load("generate_small.json")
    for run in g["runs"]:
        out = _gen(g, run)
        assert [s.tokens for s in out.seqs] == run["tokens"], run["kw"]
        assert [list(s) for s in out.steps] == run["steps"]
        assert out.total_accepted == run["total_accepted"]
        assert out.total_verify_slots == run["total_verify_slots"]
        assert [s.hit_eos for s in out.seqs] == run["hit_eos"]
        np.testing.assert_allclose([float(s.features.astype(np.float64).sum()) for s in out.seqs],
                                   run["feat_sum"], rtol=1e-4, atol=1e-3)


@pytest.mark.slow
def test_generate_c1_golden():
    g = load("generate_c1.json")
    for run in g["runs"]:
        run = dict(run)
        run["kw"] = dict(run["kw"], fixed=(1, 0, 0))
        out = _gen(g, run)
        assert [s.tokens for s in out.seqs] == run["tokens"]
        assert [list(s) for s in out.steps] == run["steps"]


# ---------------------------------------------------------------- draft update (grpo.hpp:278-344)
def test_draft_update_golden():
    z = np.load(os.path.join(G, "draft_update_small.npz"))
    cfg = cfg_from(load("generate_small.json")["config"])
    m, d = O.init_model(cfg), O.init_draft(cfg, 1)
    assert np.array_equal(d.flat, z["before"])
    seqs, to, fo = [], 0, 0
    for L in z["lens"]:
        seqs.append(O.SeqResult(0, z["tokens"][to:to + L].tolist(), 0, False,
                                z["features"][fo:fo + (L - 1) * cfg.d_model].reshape(L - 1, cfg.d_model)))
        to += L
        fo += (L - 1) * cfg.d_model
    grad = np.zeros(d.flat.size, np.float32)
    terms = O.draft_loss_grad(d, m, seqs, 1.0, 0.1, grad)
    np.testing.assert_allclose(terms[:3], z["terms"][:3], rtol=1e-6)
    assert terms[3] == z["terms"][3]
    scale = np.abs(z["grad"]).max()
    assert np.abs(grad - z["grad"]).max() <= 1e-5 * scale
    O.draft_update(d, m, seqs, O.AdamW(lr=1e-3))
    diff = np.abs(d.flat - z["after"])
    # AdamW's first step is lr*sign(g) except where |g| ~ eps; fp32 summation-order noise can
    # only move those near-zero-gradient coordinates (< 0.01% of the draft).
    assert (diff > 1e-6).mean() < 1e-4
    assert diff.max() <= 2e-3 + 1e-6


def test_checkpoint_roundtrip(tmp_path):
    # test_tinylm.cpp:237-265
    cfg = O.ModelConfig(16, 32, 2, 4, 64, 32, 21)
    m = O.init_model(cfg)
    p1, p2 = tmp_path / "a.ckpt", tmp_path / "b.ckpt"
    O.save_checkpoint(str(p1), m)
    kind, m2 = O.load_checkpoint(str(p1))
    assert kind == "target" and np.array_equal(m2.flat, m.flat)
    O.save_checkpoint(str(p2), m2)
    assert p1.read_bytes() == p2.read_bytes()
