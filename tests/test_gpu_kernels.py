"""GPU parity of the individual kernels (tcgen05 GEMM, forward, sampling, top-k, tree)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from tests.gpu_common import SMALL, capi, make_engine, rel_l2

pytestmark = pytest.mark.gpu

def bf16(a):
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (5, 256, 128), (17, 384, 256), (100, 512, 1024),
                                   (300, 256, 512), (64, 1000, 136), (256, 4608, 1536)])
def test_gemm_matches_fp64_reference(M, N, K):
    c = capi()
    rng = np.random.default_rng(M * 7 + N)
    w = rng.standard_normal((N, K)).astype(np.float32) * 0.05
    x = rng.standard_normal((M, K)).astype(np.float32)
    out, splits = c.debug_gemm(w, x)
    ref = bf16(x).astype(np.float64) @ bf16(w).astype(np.float64).T
    err = np.abs(out - ref).max() / (np.abs(ref).max() + 1e-9)
    assert err < 2e-5, (err, splits)


def test_gemm_batch_invariance():
    """A row's bits must not depend on how many rows share the launch (SURVEY §7 hard part 1)."""
    c = capi()
    rng = np.random.default_rng(3)
    N, K = 512, 768
    w = rng.standard_normal((N, K)).astype(np.float32) * 0.05
    x = rng.standard_normal((300, K)).astype(np.float32)
    full, _ = c.debug_gemm(w, x)
    for m in (1, 3, 16, 17, 33, 64, 65, 128, 129, 256, 257):
        part, _ = c.debug_gemm(w, x[:m])
        assert np.array_equal(part, full[:m]), m
    # the K split decides only which CTA computes which chunk: bits are identical
    for m in (1, 40, 300):
        for s in (1, 2, 3):
            part, _ = c.debug_gemm(w, x[:m], splits=s)
            assert np.array_equal(part, full[:m]), (m, s)


@pytest.mark.parametrize("tiles", [84, 96, 112])
def test_gemm_wide_single_chunk_batch_invariance(tiles):
    """Single-chunk weights of 84-112 tiles (the 7B / 8B QKV and w1 shapes) at every token-tile
    width (16 .. 256-token tiles, partial tiles): every row's bits equal the same row computed at
    any other row count."""
    c = capi()
    rng = np.random.default_rng(tiles)
    N, K = 128 * tiles, 256
    w = rng.standard_normal((N, K)).astype(np.float32) * 0.05
    x = rng.standard_normal((300, K)).astype(np.float32)
    full, _ = c.debug_gemm(w, x)
    for m in (1, 16, 129, 160, 192, 211, 240, 256):
        part, _ = c.debug_gemm(w, x[:m])
        assert np.array_equal(part, full[:m]), m


def test_forward_target_matches_oracle():
    e, m, _ = make_engine(SMALL)
    toks = [2, 9, 4, 13, 6, 3, 7, 12, 200, 31]
    pos = list(range(len(toks)))
    lg, hd = e.forward_target(0, toks, pos)
    rl, rh = O.forward_target(m, toks, pos)
    assert rel_l2(lg, rl) < 2e-2
    assert rel_l2(hd, rh) < 2e-2
    for i in range(len(toks)):
        assert rel_l2(lg[i], rl[i]) < 3e-2


def test_incremental_equals_full_bitwise():
    """test_tinylm.cpp:83-117, but bit-exact on the GPU (batch-invariant kernels)."""
    e, m, _ = make_engine(SMALL)
    toks = [2, 9, 4, 13, 6, 3, 7, 12]
    full, _ = e.forward_target(0, toks, list(range(8)))
    e.cache_reset(1)
    done = 0
    for chunk in (3, 1, 4):
        lg, _ = e.forward_target(1, toks[done:done + chunk], list(range(done, done + chunk)))
        assert np.array_equal(lg, full[done:done + chunk]), chunk
        done += chunk


def test_tree_masked_rows_equal_sequential_paths_bitwise():
    """test_tinylm.cpp:119-157 on the GPU: tree rows == per-path sequential rows, bit-exact."""
    e, m, _ = make_engine(SMALL)
    V = SMALL.vocab_size
    prefix = [2, 7, 5]
    toks, poss, parent = [4, 6, 8, 9], [3, 4, 4, 5], [-1, 0, 0, 1]
    mask = np.zeros((4, 4), np.uint8)
    for i in range(4):
        j = i
        while j != -1:
            mask[i, j] = 1
            j = parent[j]
    e.forward_target(0, prefix, [0, 1, 2])
    tree_lg, _ = e.forward_target(0, toks, poss, mask)
    paths = {0: [4], 1: [4, 6], 2: [4, 8], 3: [4, 6, 9]}
    for row, path in paths.items():
        slot = 1 + row
        e.cache_reset(slot)
        all_t = prefix + path
        lg, _ = e.forward_target(slot, all_t, list(range(len(all_t))))
        assert np.array_equal(lg[-1], tree_lg[row]), row
    # and the oracle agrees within the bf16 tolerance
    cache = O.KvCache(SMALL.n_layers, SMALL.d_model)
    O.forward_target(m, prefix, [0, 1, 2], None, cache)
    rl, _ = O.forward_target(m, toks, poss, mask, cache)
    assert rel_l2(tree_lg, rl) < 2e-2


def test_gather_tail_keeps_rows():
    e, m, _ = make_engine(SMALL)
    e.forward_target(0, [3, 4, 5, 6, 7], list(range(5)))
    k0, v0 = e.cache_read(0)
    e.cache_gather_tail(0, 1, [0, 2])
    assert e.cache_len(0) == 3
    k1, v1 = e.cache_read(0)
    assert np.array_equal(k1[:, 1], k0[:, 1]) and np.array_equal(k1[:, 2], k0[:, 3])
    assert np.array_equal(v1[:, 2], v0[:, 3])


def test_draft_forward_matches_oracle():
    e, m, d = make_engine(SMALL)
    rng = np.random.default_rng(1)
    feats = rng.standard_normal((5, SMALL.d_model)).astype(np.float32)
    f, lg = e.forward_draft_rows(0, [3, 5, 7, 2, 9], feats, [1, 2, 3, 4, 5])
    cache = O.KvCache(1, SMALL.d_model)
    rf, rl, _, _ = O.forward_draft_rows(d, m, [3, 5, 7, 2, 9], feats, [1, 2, 3, 4, 5], cache=cache)
    assert rel_l2(f, rf) < 2e-2
    assert rel_l2(lg, rl) < 3e-2


def test_sampling_bit_exact_given_logits():
    """sample_token (tinylm.hpp:591-628) on identical logits: device == oracle, exactly."""
    e, _, _ = make_engine(SMALL)
    V = SMALL.vocab_size
    rng = np.random.default_rng(5)
    lg = (3 * rng.standard_normal((64, V))).astype(np.float32)
    lg[0, [3, 9, 200]] = lg[0].max() + 1  # exact ties -> lowest index
    lg[1, :] = 0.0
    seeds = rng.integers(0, 2**63, size=64, dtype=np.uint64)
    kp = rng.integers(1, 90, size=64).astype(np.int32)
    for temp in (0.0, 0.7, 1.0, 1.5):
        got = e.sample_rows(lg, temp, seeds, kp)
        want = [O.sample_token(lg[i], temp, O.mix_key(int(seeds[i]), int(kp[i]))) for i in range(64)]
        assert got.tolist() == want, temp
    bad = lg[:2].copy()
    bad[0, 5] = np.nan
    with pytest.raises(ArithmeticError):
        e.sample_rows(bad, 0.0, seeds[:2], kp[:2])


def test_topk_logsoftmax_matches_oracle():
    e, _, _ = make_engine(SMALL)
    V = SMALL.vocab_size
    rng = np.random.default_rng(9)
    lg = (2 * rng.standard_normal((20, V))).astype(np.float32)
    lg[0, [1, 2, 3]] = lg[0].max() + 0.5
    for k in (1, 3, 10, 16):
        tok, lp = e.topk_logsoftmax(lg, k)
        for r in range(20):
            lps = O.log_softmax_row(lg[r])
            want = O.topk_tokens(lps, k)
            assert tok[r].tolist() == want
            np.testing.assert_allclose(lp[r], lps[want], rtol=0, atol=1e-12)


@pytest.mark.parametrize("k,l,nv", [(0, 3, 4), (3, 1, 3), (2, 2, 7), (3, 3, 10), (4, 4, 30), (10, 3, 64),
                                    (10, 6, 211), (5, 5, 1000)])
def test_device_tree_matches_oracle(k, l, nv):
    """expand_tree_with + rerank + build_tree_mask on device vs oracle, decisions bit-exact."""
    e, _, _ = make_engine(SMALL)
    V = SMALL.vocab_size
    rng = np.random.default_rng(k * 31 + l)
    table = {}

    def path_key(node, tok, par):
        path = []
        while node != -1:
            path.append(tok[node])
            node = par[node]
        return tuple(path)

    def logits_for(key):
        if key not in table:
            r = (2.5 * rng.standard_normal(V)).astype(np.float32)
            if rng.random() < 0.3:
                r[rng.integers(0, V, 3)] = r.max()  # exact ties
            table[key] = r
        return table[key]

    def fn(ids, tok, par):
        return np.stack([logits_for(path_key(i, tok, par)) for i in ids])

    root = 17
    dev = e.build_tree(root, k, l, nv, fn)
    ref = O.expand_tree_with(root, k, l, lambda t, n: O.log_softmax_row(
        logits_for(path_key(n, [x.token for x in t], [x.parent for x in t]))))
    assert dev["tok"].tolist() == [x.token for x in ref]
    assert dev["par"].tolist() == [x.parent for x in ref]
    assert dev["dep"].tolist() == [x.depth for x in ref]
    np.testing.assert_allclose(dev["lp"], [x.log_prob for x in ref], rtol=0, atol=1e-12)
    np.testing.assert_allclose(dev["conf"], [x.confidence for x in ref], rtol=1e-12, atol=0)
    sel, mask = O.rerank_candidates(ref, nv)
    assert dev["sel"].tolist() == sel
    assert np.array_equal(dev["mask"], mask)


LARGE_V = O.ModelConfig(vocab_size=70001, d_model=64, n_layers=1, n_heads=1, d_ff=128, max_seq_len=32, seed=2)


def test_multichunk_topk_and_sampling_match_oracle():
    """Rows longer than one 8192-logit chunk: the per-(row, chunk) CTAs and the last-arriver
    merge give the oracle's top-k / log-probs and sample_token results."""
    e, _, _ = make_engine(LARGE_V, max_seqs=2, max_rows=64, seed_models=False)
    V = LARGE_V.vocab_size
    rng = np.random.default_rng(13)
    lg = (3 * rng.standard_normal((24, V))).astype(np.float32)
    lg[0, [5, 8192 + 7, 65536 + 3]] = lg[0].max() + 1  # exact ties in three chunks
    lg[1, :] = 0.0                                       # all equal
    lg[2, :] = -np.inf
    lg[2, [9000, 70000]] = 1.0                           # mostly -inf, winners in two chunks
    lg[3, 8192:] = lg[3].max() + 2                       # mass concentrated after chunk 0
    for k in (1, 10, 16):
        tok, lp = e.topk_logsoftmax(lg, k)
        for r in range(24):
            lps = O.log_softmax_row(lg[r])
            want = O.topk_tokens(lps, k)
            assert tok[r].tolist() == want, (k, r)
            np.testing.assert_allclose(lp[r], lps[want], rtol=0, atol=1e-12)
    seeds = rng.integers(0, 2**63, size=24, dtype=np.uint64)
    kp = rng.integers(1, 90, size=24).astype(np.int32)
    for temp in (0.0, 0.7, 1.0):
        got = e.sample_rows(lg, temp, seeds, kp)
        want = [O.sample_token(lg[i], temp, O.mix_key(int(seeds[i]), int(kp[i]))) for i in range(24)]
        assert got.tolist() == want, temp
    bad = lg[4:6].copy()
    bad[1, 60000] = np.nan
    with pytest.raises(ArithmeticError):
        e.sample_rows(bad, 1.0, seeds[:2], kp[:2])


def _attn_ref(q, k, v, H):
    """fp64 softmax(q.k^T/sqrt(dh)).v per head (tinylm.hpp:335-395) on bf16-rounded K/V."""
    d = q.shape[0]
    dh = d // H
    bf = lambda a: (np.asarray(a, np.float32).view(np.uint32) + 0x7FFF + ((np.asarray(a, np.float32).view(np.uint32) >> 16) & 1)  # noqa: E731
                    & 0xFFFF0000).view(np.float32).astype(np.float64)
    kk, vv = bf(k), bf(v)
    out = np.zeros(d)
    for h in range(H):
        s = kk[:, h * dh:(h + 1) * dh] @ q[h * dh:(h + 1) * dh].astype(np.float64) / np.sqrt(dh)
        p = np.exp(s - s.max())
        out[h * dh:(h + 1) * dh] = (p / p.sum()) @ vv[:, h * dh:(h + 1) * dh]
    return out


@pytest.mark.parametrize("H,dh", [(12, 128), (2, 64), (28, 128)])
def test_attention_long_context_and_launch_shape_invariance(H, dh):
    """The persistent attention kernel vs an fp64 reference at long contexts (rows spread over
    many CTAs, tickets, in-kernel merge), and bitwise invariance of a row's output to the
    batch it is launched with (head grouping and block-to-CTA mapping change with it)."""
    c = pytest.importorskip("paper_2509_21792_b200.capi")
    d = H * dh
    rng = np.random.default_rng(H * 7 + dh)
    lens = [1, 63, 64, 65, 700, 2100, 129, 5]
    qs = rng.standard_normal((len(lens), d)).astype(np.float32)
    ks = [rng.standard_normal((n, d)).astype(np.float32) for n in lens]
    vs = [rng.standard_normal((n, d)).astype(np.float32) for n in lens]
    out = c.debug_attention(qs, ks, vs, H)
    for i, n in enumerate(lens):
        ref = _attn_ref(qs[i], ks[i], vs[i], H)
        err = np.abs(out[i] - ref).max()
        assert err < 2e-2 * max(1.0, np.abs(ref).max()), (n, err)
    # the same rows alone and inside a bigger batch: identical bits
    for i in (0, 4, 5):
        solo = c.debug_attention(qs[i:i + 1], ks[i:i + 1], vs[i:i + 1], H)
        assert np.array_equal(solo[0], out[i]), i
    big_q = np.concatenate([qs, rng.standard_normal((40, d)).astype(np.float32)])
    big_k = ks + [rng.standard_normal((300, d)).astype(np.float32) for _ in range(40)]
    big_v = vs + [rng.standard_normal((300, d)).astype(np.float32) for _ in range(40)]
    big = c.debug_attention(big_q, big_k, big_v, H)
    assert np.array_equal(big[:len(lens)], out)


def test_gemm_pair_bitwise(tmp_path):
    """The CTA-pair (cta_group::2) GEMM (SGB_GEMM_PAIR=1, a separate process: the switch is read
    once) gives the 1-CTA kernel's bits, incl. a forced K split."""
    import os
    import subprocess
    import sys
    c = capi()
    rng = np.random.default_rng(21)
    w = rng.standard_normal((640, 1536)).astype(np.float32) * 0.05
    x = rng.standard_normal((300, 1536)).astype(np.float32)
    np.save(tmp_path / "w.npy", w)
    np.save(tmp_path / "x.npy", x)
    ref = {m: c.debug_gemm(w, x[:m])[0] for m in (65, 128, 211, 300)}
    ref_s = c.debug_gemm(w, x[:200], splits=3)[0]
    code = (
        "import numpy as np, sys; sys.path.insert(0, '.')\n"
        "from paper_2509_21792_b200 import capi as c\n"
        f"w = np.load(r'{tmp_path / 'w.npy'}'); x = np.load(r'{tmp_path / 'x.npy'}')\n"
        "for m in (65, 128, 211, 300): np.save(r'%s/p%%d.npy' %% m, c.debug_gemm(w, x[:m])[0])\n"
        "np.save(r'%s/ps.npy', c.debug_gemm(w, x[:200], splits=3)[0])\n" % (tmp_path, tmp_path))
    env = dict(os.environ, SGB_GEMM_PAIR="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=root, timeout=300)
    for m in (65, 128, 211, 300):
        assert np.array_equal(np.load(tmp_path / f"p{m}.npy"), ref[m]), m
    assert np.array_equal(np.load(tmp_path / "ps.npy"), ref_s)
