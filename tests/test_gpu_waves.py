"""KV-region admission (waves): a rollout with more sequences than the engine's KV regions runs
its query groups in waves -- a group's regions are recycled once all its members finished and
the next group is admitted and prefilled at that step boundary (the reference admits all at
once, scheduler.cpp:259-294; SURVEY §7 hard part 3, BASELINE configs[4]). Sequence ids, keys and
caps are global, so the tokens, features and EOS flags must equal an all-resident rollout of the
same prompts bit for bit, in every mode."""
import numpy as np
import pytest

from tests.gpu_common import SMALL, make_engine

pytestmark = pytest.mark.gpu


# rejection sampling is lossless in distribution only: its tokens depend on the tree, and the
# adaptive plan depends on the live count, which waves change -- so it is compared under a fixed plan
@pytest.mark.parametrize("mode,temp,acc", [("vanilla", 0.0, "strict"), ("adaptive_spec", 0.0, "strict"),
                                           ("adaptive_spec", 1.0, "strict"), ("fixed_spec", 1.0, "rejection")])
def test_waves_equal_all_resident(mode, temp, acc):
    rng = np.random.default_rng(11)
    prompts = [rng.integers(2, SMALL.vocab_size, size=int(rng.integers(3, 10))).tolist() for _ in range(7)]
    caps = rng.integers(5, 40, size=7 * 4).tolist()  # variable stops: groups finish at different steps
    kw = dict(c_peak=16, alpha=2.0, k_max=4, l_max=3, mode=mode, temperature=temp, seed=9, acceptance=acc,
              seq_max_new=caps, fixed=(6, 3, 2))
    big, _, _ = make_engine(SMALL, max_seqs=32)
    small, _, _ = make_engine(SMALL, max_seqs=8)  # 2 blocks of 4 regions: 7 groups run in 4 waves
    ref = big.generate(prompts, 4, **kw)
    got = small.generate(prompts, 4, **kw)
    assert got.tokens == ref.tokens
    assert got.hit_eos == ref.hit_eos
    for a, b in zip(got.features, ref.features):
        assert np.array_equal(a, b)
    assert got.total_accepted == ref.total_accepted
    with pytest.raises(ValueError):  # the rollout left HBM: the draft update needs its sequences
        small.draft_update(None, apply_step=False)
    big.close()
    small.close()
