"""Prefix-shared tree attention (attention_group.cu) vs the per-row kernel and fp64.

Verify rows of one sequence share its committed K/V; the group kernel stages that prefix
once per tile. Losslessness of the speculative rollout (spec tokens == AR tokens) needs the
group kernel to reproduce the per-row kernel bit for bit, so that is asserted exactly here;
both are also checked against an fp64 reference of build_tree_mask + decode_blocks
(drafttree.cpp:145-168, tinylm.hpp:335-395) within the bf16 tolerance of the K/V store.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _tree(rng, n, max_depth=7):
    par, dep = [-1], [0]
    for i in range(1, n):
        while True:
            p = int(rng.integers(0, i))
            if dep[p] < max_depth:
                break
        par.append(p)
        dep.append(dep[p] + 1)
    return par


def _ref(q, kc, vc, kn, vn, par, H):
    """fp64: row i attends to committed keys then its ancestors-or-self (root first)."""
    bf = lambda a: a.astype(np.float32).view(np.uint32)  # noqa: E731
    # round K/V to bf16 like the device store (round-to-nearest-even)
    def r16(a):
        u = bf(a).astype(np.uint64)
        u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
        return u.astype(np.uint32).view(np.float32).astype(np.float64)
    kc, vc, kn, vn = r16(kc), r16(vc), r16(kn), r16(vn)
    d = q.shape[1]
    dh = d // H
    out = np.zeros(q.shape, np.float64)
    for i in range(len(par)):
        path = []
        a = i
        while a >= 0:
            path.append(a)
            a = par[a]
        path = path[::-1]
        kk = np.concatenate([kc, kn[path]])
        vv = np.concatenate([vc, vn[path]])
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            s = kk[:, sl] @ q[i, sl].astype(np.float64) / np.sqrt(dh)
            p = np.exp(s - s.max())
            out[i, sl] = (p / p.sum()) @ vv[:, sl]
    return out


@pytest.mark.parametrize("H,dh", [(28, 128), (12, 128), (2, 64)])
def test_group_attention_bitwise_equals_per_row_kernel(H, dh):
    from paper_2509_21792_b200 import capi as c
    d = H * dh
    rng = np.random.default_rng(H + dh)
    # (ctx_len, tree rows): tiles of 64 rows, ragged last tiles, chains crossing block edges
    groups = [(1, 13), (63, 8), (64, 64), (65, 65), (300, 211), (127, 2), (700, 40), (190, 1)]
    ctx = [g[0] for g in groups]
    parents = [_tree(rng, g[1]) for g in groups]
    M = sum(g[1] for g in groups)
    q = rng.standard_normal((M, d)).astype(np.float32)
    kc = rng.standard_normal((sum(ctx), d)).astype(np.float32)
    vc = rng.standard_normal((sum(ctx), d)).astype(np.float32)
    kn = rng.standard_normal((M, d)).astype(np.float32)
    vn = rng.standard_normal((M, d)).astype(np.float32)
    o_row, o_grp = c.debug_tree_attention(ctx, parents, q, kc, vc, kn, vn, H)
    assert np.array_equal(o_row, o_grp), np.argwhere(o_row != o_grp)[:5]
    # attention_tree.cu (the engine's tree-verify / draft-level kernel) -- same bits
    o_tree = c.debug_tree_attention_tree(ctx, parents, q, kc, vc, kn, vn, H)
    assert np.array_equal(o_row, o_tree), np.argwhere(o_row != o_tree)[:5]
    # spot-check groups against fp64
    r0 = c0 = 0
    for (cl, n), par in zip(groups, parents):
        if cl <= 300:
            ref = _ref(q[r0:r0 + n], kc[c0:c0 + cl], vc[c0:c0 + cl], kn[r0:r0 + n], vn[r0:r0 + n], par, H)
            err = np.abs(o_grp[r0:r0 + n] - ref).max()
            assert err < 2e-2 * max(1.0, np.abs(ref).max()), (cl, n, err)
        r0 += n
        c0 += cl


def test_group_attention_ragged_and_repeated_launches():
    """Tickets re-arm between launches; a group's rows give the same bits alone and amid others."""
    from paper_2509_21792_b200 import capi as c
    H, dh = 12, 128
    d = H * dh
    rng = np.random.default_rng(3)
    par = _tree(rng, 50)
    q = rng.standard_normal((50, d)).astype(np.float32)
    kc = rng.standard_normal((129, d)).astype(np.float32)
    vc = rng.standard_normal((129, d)).astype(np.float32)
    kn = rng.standard_normal((50, d)).astype(np.float32)
    vn = rng.standard_normal((50, d)).astype(np.float32)
    a_row, a_grp = c.debug_tree_attention([129], [par], q, kc, vc, kn, vn, H)
    b_row, b_grp = c.debug_tree_attention([129], [par], q, kc, vc, kn, vn, H)
    assert np.array_equal(a_grp, b_grp) and np.array_equal(a_row, a_grp)
    # the same group preceded by another one
    par2 = _tree(rng, 20)
    q2 = rng.standard_normal((20, d)).astype(np.float32)
    k2 = rng.standard_normal((40, d)).astype(np.float32)
    n2 = rng.standard_normal((20, d)).astype(np.float32)
    _, g2 = c.debug_tree_attention([40, 129], [par2, par], np.concatenate([q2, q]), np.concatenate([k2, kc]),
                                   np.concatenate([k2, vc]), np.concatenate([n2, kn]), np.concatenate([n2, vn]), H)
    assert np.array_equal(g2[20:], a_grp)


@pytest.mark.gpu
@pytest.mark.parametrize("H,dh", [(28, 128), (4, 64)])
def test_decode_attention_bitwise(H, dh):
    """The cluster decode kernel (AR steps) gives attention.cu's bits: ragged contexts around the
    16-key chunk and 64-key block edges, up to a few thousand keys (clusters of 1..8 CTAs)."""
    from paper_2509_21792_b200 import capi as c
    d = H * dh
    rng = np.random.default_rng(17)
    for ctx in ([1, 15, 16, 17, 63, 64, 65, 127, 200], [640], [4100, 33], [1000] * 3):
        n = sum(ctx)
        q = rng.standard_normal((len(ctx), d)).astype(np.float32)
        kc = rng.standard_normal((n, d)).astype(np.float32)
        vc = rng.standard_normal((n, d)).astype(np.float32)
        kn = rng.standard_normal((len(ctx), d)).astype(np.float32)
        vn = rng.standard_normal((len(ctx), d)).astype(np.float32)
        o_row, o_dec = c.debug_attention_decode(ctx, q, kc, vc, kn, vn, H)
        assert np.array_equal(o_row, o_dec), (ctx, np.argwhere(o_row != o_dec)[:5])
        assert np.isfinite(o_dec).all()
