"""Data-parallel host logic on CPU (gloo, world_size 2), SURVEY.md §8(e):
  * the rollout shards by whole query groups and keeps GLOBAL sequence ids, so every
    token stream -- including T>0 keyed sampling -- equals the unsharded run;
  * the online draft update all-reduces gradients computed with the GLOBAL row count
    (grpo.hpp:286-290), so the summed shard gradients equal the full-batch gradient and
    one identical AdamW step follows on every replica (C1);
  * rollout statistics are all-reduced (C2).
The GPU build runs the same protocol with NCCL over NVLink (bench.py / DESIGN.md)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

CFG = O.ModelConfig(vocab_size=64, d_model=64, n_layers=2, n_heads=4, d_ff=128, max_seq_len=48, seed=3)
PROMPTS = [[5, 9, 13], [7, 2, 40, 41], [3, 3, 8], [60, 12, 33, 4, 5]]
G = 2
GEN = dict(c_peak=8, alpha=2.0, k_max=3, l_max=2, mode="adaptive_spec", temperature=1.0, seed=11,
           max_new_tokens=10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, d = O.init_model(CFG), O.init_draft(CFG, 1)
    per = len(PROMPTS) // world
    mine = PROMPTS[rank * per:(rank + 1) * per]
    res = O.generate_dynamic_batch(m, d, mine, G, sid_offset=rank * per * G, **GEN)
    # C2: rollout statistics
    stats = torch.tensor([res.total_accepted, res.total_verify_slots,
                          sum(len(s.tokens) - s.prompt_len for s in res.seqs)], dtype=torch.float64)
    dist.all_reduce(stats)
    # C1: global row count first, then local grads with the global normaliser, then sum
    rows = torch.tensor([sum(max(0, len(s.tokens) - 2) for s in res.seqs)], dtype=torch.int64)
    dist.all_reduce(rows)
    grad = np.zeros(d.flat.size, np.float32)
    terms = O.draft_loss_grad(d, m, res.seqs, 1.0, 0.1, grad, rows_total=int(rows.item()))
    g = torch.from_numpy(grad)
    dist.all_reduce(g)
    loss = torch.tensor([terms[0], terms[1]], dtype=torch.float64)
    dist.all_reduce(loss)
    opt = O.AdamW(lr=1e-3)
    d2 = d.copy()
    opt.step(d2.flat, g.numpy())
    out[rank] = dict(tokens=[s.tokens for s in res.seqs], stats=stats.tolist(), rows=int(rows.item()),
                     grad=g.numpy().copy(), loss=loss.tolist(), weights=d2.flat.copy())
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def sharded():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    return dict(out)


@pytest.fixture(scope="module")
def full():
    m, d = O.init_model(CFG), O.init_draft(CFG, 1)
    res = O.generate_dynamic_batch(m, d, PROMPTS, G, **GEN)
    grad = np.zeros(d.flat.size, np.float32)
    terms = O.draft_loss_grad(d, m, res.seqs, 1.0, 0.1, grad)
    return res, grad, terms


def test_sharded_rollout_keeps_global_sids(sharded, full):
    res = full[0]
    toks = sharded[0]["tokens"] + sharded[1]["tokens"]
    assert toks == [s.tokens for s in res.seqs]


def test_rollout_stats_allreduce(sharded, full):
    res = full[0]
    st = sharded[0]["stats"]
    assert st == sharded[1]["stats"]
    assert st[2] == sum(len(s.tokens) - s.prompt_len for s in res.seqs)
    assert st[0] + st[1] > 0


def test_draft_grad_allreduce_equals_full_batch(sharded, full):
    _, grad, terms = full
    g0, g1 = sharded[0]["grad"], sharded[1]["grad"]
    assert np.array_equal(g0, g1)  # identical after the all-reduce
    assert sharded[0]["rows"] == terms[3]
    assert np.abs(g0 - grad).max() <= 1e-6 * max(1.0, np.abs(grad).max())
    np.testing.assert_allclose(sharded[0]["loss"], terms[:2], rtol=1e-6)


def test_replicas_step_identically(sharded):
    assert np.array_equal(sharded[0]["weights"], sharded[1]["weights"])
