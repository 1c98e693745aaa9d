"""Online draft learning at the c2 shape: tau on held-out prompts vs AdamW steps.

Training prompts come from a stream disjoint from the benchmark prompts (SURVEY §8d:
Rng(mix_key(0, 0x7a11 + iter))); each iteration is one rollout (vanilla, greedy, features
kept) followed by S draft_update steps on it (grpo.cpp:329-345), as the paper's online
learning does between GRPO iterations.

    python scripts/warm_draft.py [iters] [S] [lr] [config]
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from bench import WORKLOADS, make_prompts, model_cfg  # noqa: E402
from oracle.oracle import mix_key  # noqa: E402  (integer key derivation only)
from paper_2509_21792_b200 import capi  # noqa: E402


def stream_prompts(key, n, P, V):
    seed = mix_key(0, key)
    with np.errstate(over="ignore"):
        st = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * np.arange(2, n * P + 2, dtype=np.uint64)
        z = (st ^ (st >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z % np.uint64(V - 2) + np.uint64(2)).astype(np.int64).reshape(n, P).tolist()


iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
S = int(sys.argv[2]) if len(sys.argv) > 2 else 4
lr = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
w = dict(WORKLOADS[sys.argv[4] if len(sys.argv) > 4 else "c2"])
w["new"] = 128
cfg = model_cfg(w)
eng = capi.Engine(cfg, 1, 0, 64, 4096, 10, 6)
eng.init_random(1234)
held = make_prompts(w, 0)[:4]


def tau_eval():
    r = eng.generate(held, 1, c_peak=211, mode="adaptive_spec", temperature=0.0, seed=7, max_new_tokens=96,
                     want_features=False)
    ra = eng.generate(held, 1, c_peak=211, mode="vanilla", temperature=0.0, seed=7, max_new_tokens=96,
                      want_features=False)
    same = all(list(a) == list(b) for a, b in zip(r.tokens, ra.tokens))
    return r.tau(), r.generated() / r.seconds, ra.generated() / ra.seconds, same


t0 = time.time()
tau, sp, ar, same = tau_eval()
print(json.dumps(dict(it=0, tau=round(tau, 3), spec_tok_s=round(sp), ar_tok_s=round(ar), lossless=same)), flush=True)
for it in range(1, iters + 1):
    pr = stream_prompts(0x7A11 + it, 32, w["P"], w["V"])
    eng.generate(pr, 2, c_peak=211, mode="vanilla", temperature=0.0, seed=it, max_new_tokens=128, want_features=True)
    for _ in range(S):
        (fl, tl, tot, rows, secs), _ = eng.draft_update(None, lr=lr)
    if it % 5 == 0 or it == iters:
        tau, sp, ar, same = tau_eval()
        print(json.dumps(dict(it=it, steps=it * S, feat_loss=round(fl, 5), tok_loss=round(tl, 4), rows=rows,
                              upd_ms=round(secs * 1e3, 1), tau=round(tau, 3), spec_tok_s=round(sp), ar_tok_s=round(ar),
                              lossless=same, wall=round(time.time() - t0))), flush=True)
