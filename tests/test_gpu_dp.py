"""Data-parallel protocol on one GPU: the rank-local pieces of the NCCL path.

The driver's GPU box has one GPU, so multi-rank NCCL cannot run here (ranks that wait on each
other must not share a GPU); tests/test_dp_gloo.py covers the world-size-2 host protocol on CPU.
What IS checked on the device:
  * a world-size-1 NCCL group initialises on the engine's stream, and the C2 statistics
    all-reduce and the C1 gradient all-reduce are identities;
  * query-group shards with global sid offsets reproduce the unsharded rollout bit for bit
    (T=1 keyed sampling, so sids matter), as each rank of the data-parallel bench does;
  * shard gradients computed with the GLOBAL row normaliser (grpo.hpp:286-290) sum to the
    full-batch gradient (what ncclAllReduce(sum) produces on N ranks).
"""
import numpy as np
import pytest

from paper_2509_21792_b200 import capi
from tests.gpu_common import SMALL, make_engine, rel_l2

pytestmark = pytest.mark.gpu

GEN = dict(c_peak=16, alpha=2.0, k_max=3, l_max=2, mode="adaptive_spec", temperature=1.0, seed=21,
           max_new_tokens=24)


def _prompts():
    rng = np.random.default_rng(11)
    return [rng.integers(2, SMALL.vocab_size, size=int(rng.integers(4, 10))).tolist() for _ in range(4)]


def test_nccl_world1_allreduce_identity():
    e, _, _ = make_engine(SMALL)
    e.nccl_init(0, 1, capi.nccl_unique_id())
    v = np.array([3, -7, 1 << 40], np.int64)
    assert np.array_equal(e.allreduce_i64(v), v)
    f = np.array([0.25, -1.5e300, 3.0])
    assert np.array_equal(e.allreduce_f64(f), f)
    prompts = _prompts()
    e.generate(prompts, 2, **GEN)
    _, g_plain = e.draft_update(None, apply_step=False, want_grad=True)
    _, g_red = e.draft_update(None, apply_step=False, want_grad=True, allreduce_grad=True)
    assert np.array_equal(g_plain, g_red)


def test_group_shards_reproduce_full_rollout_and_gradient():
    e, _, _ = make_engine(SMALL)
    prompts, g = _prompts(), 2
    full = e.generate(prompts, g, **GEN)
    _, g_full = e.draft_update(None, apply_step=False, want_grad=True)
    rows_total = sum(max(0, len(t) - 2) for t in full.tokens)
    shards, grads, rows = [], [], 0
    for r in range(2):
        mine = prompts[2 * r:2 * r + 2]
        res = e.generate(mine, g, sid_offset=2 * r * g, **GEN)
        shards.append(res)
        (_, _, _, n, _), gr = e.draft_update(None, apply_step=False, want_grad=True, rows_total=rows_total)
        grads.append(gr)
        rows += n
    toks = [t for s in shards for t in s.tokens]
    assert len(toks) == len(full.tokens)
    for a, b in zip(toks, full.tokens):
        assert list(a) == list(b)
    assert rows == rows_total
    summed = grads[0] + grads[1]
    print("shard-sum vs full gradient rel-L2", rel_l2(summed, g_full))
    assert rel_l2(summed, g_full) < 1e-5
