import numpy as np, sys
sys.path.insert(0, '.')
from oracle import oracle as O
from tests.gpu_common import C1, make_engine
e, m, d = make_engine(C1, max_seqs=8)
rng = np.random.default_rng(4)
pr = [rng.integers(2, C1.vocab_size, size=32).tolist() for _ in range(2)]
r = e.generate(pr, 2, c_peak=64, mode="vanilla", temperature=0.0, seed=7, max_new_tokens=24)
for s in range(4):
    toks = r.tokens[s]
    e.cache_reset(7)
    lg, _ = e.forward_target(7, toks[:-1], list(range(len(toks)-1)))
    am = lg.argmax(1)
    bad = [t for t in range(31, len(toks)-1) if am[t] != toks[t+1]]
    print(s, "mismatch positions (teacher-forced argmax vs rollout)", bad[:5])
    # incremental: prompt then one at a time
    e.cache_reset(6)
    lg0, _ = e.forward_target(6, toks[:32], list(range(32)))
    print("  prefill last-row equal:", np.array_equal(lg0[-1], lg[31]))
    for t in range(32, 36):
        l1, _ = e.forward_target(6, [toks[t]], [t])
        print("  step", t, "equal", np.array_equal(l1[0], lg[t]), "argmax", l1[0].argmax(), "rollout", toks[t+1])
