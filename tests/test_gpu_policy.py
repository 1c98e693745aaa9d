"""GRPO policy update on the device: policy_loss_grad (grpo.hpp:235-276) through
target_train_forward / backward (tinylm.hpp:804-866) and one AdamW step (grpo.cpp:142-161),
compared with the COMPILED reference's policy_loss_grad (oracle/_ref) on the same fp32 weights:
loss within 2e-2 relative, gradient rel-L2 <= 5e-2 overall and <= 8e-2 per tensor (bf16 operands,
fp32 accumulation), the AdamW step moves the master like the reference's, and the rebuilt bf16
inference weights are exactly those of a fresh upload of the updated master."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import refc
from tests.gpu_common import C1, SMALL, capi, rel_l2

pytestmark = pytest.mark.gpu


def _seqs(cfg, n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        L = int(rng.integers(6, cfg.max_seq_len - 1))
        q = int(rng.integers(1, L))
        out.append((rng.integers(2, cfg.vocab_size, L).tolist(), q, float(rng.normal(0, 1))))
    out.append((rng.integers(2, cfg.vocab_size, 9).tolist(), 9, 1.0))  # no response: skipped
    return out


@pytest.mark.parametrize("cfg", [SMALL, C1], ids=["small", "c1"])
def test_policy_gradient_matches_reference(cfg):
    if not refc.available():
        pytest.skip("oracle/_ref not built")
    m = O.init_model(cfg)
    e = capi().Engine(cfg, 1, 0, 8, 512, 4, 3)
    e.policy_enable()
    e.upload_target(m.flat)
    e.upload_draft(O.init_draft(cfg, 1).flat)
    seqs = _seqs(cfg, 6, 1)
    (loss, toks, rows, secs, skipped), grad = e.policy_update(seqs, apply_step=False, want_grad=True)
    ref_loss, ref_grad = refc.policy_loss_grad(refc.RefModel(cfg, m.flat), seqs)
    r = rel_l2(grad, ref_grad)
    print(f"{cfg.d_model}: loss {loss:.6e} vs {ref_loss:.6e}; tokens {toks} rows {rows}; grad rel-L2 {r:.2e}; {secs*1e3:.1f} ms")
    assert not skipped and toks == sum(len(t) - q for t, q, _ in seqs)
    assert abs(loss - ref_loss) <= 2e-2 * abs(ref_loss) + 1e-6
    assert r < 5e-2
    for name, (off, rr, cc) in m.offsets().items():
        g, gr = grad[off:off + rr * cc], ref_grad[off:off + rr * cc]
        if np.abs(gr).max() > 0:
            assert rel_l2(g, gr) < 8e-2, name
        else:
            assert np.abs(g).max() == 0, name  # e.g. tok_emb rows of unused tokens


def test_policy_step_and_rebuilt_weights():
    cfg = SMALL
    m = O.init_model(cfg)
    e = capi().Engine(cfg, 1, 0, 8, 512, 4, 3)
    e.policy_enable()
    e.upload_target(m.flat)
    e.upload_draft(O.init_draft(cfg, 1).flat)
    seqs = _seqs(cfg, 5, 2)
    _, g = e.policy_update(seqs, lr=1e-3, apply_step=False, want_grad=True)
    e.policy_update(seqs, lr=1e-3)
    got = e.download_target()
    want = m.flat.copy()
    O.AdamW(lr=1e-3).step(want, g)  # the reference AdamW (oracle restatement) on the device gradient
    diff = np.abs(got - want)
    assert diff.max() < 1e-6, diff.max()
    # the rebuilt inference weights equal a fresh upload of the updated master
    f = capi().Engine(cfg, 1, 0, 8, 512, 4, 3)
    f.upload_target(got)
    f.upload_draft(O.init_draft(cfg, 1).flat)
    toks = [5, 17, 100, 41, 2, 99, 7, 200]
    a, _ = e.forward_target(7, toks, list(range(8)))
    b, _ = f.forward_target(7, toks, list(range(8)))
    assert np.array_equal(a, b)
    # nothing to train: policy_update's logged no-op (grpo.cpp:170)
    (_, toks_n, _, _, skipped), _ = e.policy_update([([3, 4, 5], 3, 1.0)])
    assert skipped and toks_n == 0
