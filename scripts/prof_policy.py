"""GRPO policy update on the device (engine_policy.cu) at a BASELINE shape: one AR rollout, then
policy_update steps over its sequences with synthetic advantages; device time, tokens/s and the
training TFLOP/s (6 x non-embedding params x tokens + the LM head's 6 x d x V per token).

    python scripts/prof_policy.py [config] [n_seqs] [new_tokens] [updates]
"""
import json
import sys

import numpy as np

sys.path.insert(0, '.')
from bench import WORKLOADS, make_prompts, model_cfg  # noqa: E402
from paper_2509_21792_b200 import capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
new = int(sys.argv[3]) if len(sys.argv) > 3 else 512
ups = int(sys.argv[4]) if len(sys.argv) > 4 else 3
w = dict(WORKLOADS[name])
cfg = model_cfg(w)
eng = capi.Engine(cfg, 1, 0, max(64, n), 2048, 10, 6)
eng.policy_enable()
eng.init_random(1234)
r = eng.generate(make_prompts(w, 0)[:n], 1, c_peak=211, mode="vanilla", temperature=0.0, seed=1, max_new_tokens=new)
rng = np.random.default_rng(0)
seqs = [(t, p, float(rng.standard_normal())) for t, p in zip(r.tokens, r.prompt_len)]
d, L, F, V = w["d"], w["L"], w["dff"], w["V"]
P = L * (4 * d * d + 2 * d * F)
for i in range(ups):
    (loss, toks, rows, secs, skipped), _ = eng.policy_update(seqs, lr=2e-5)
    flops = 6.0 * (P + d * V) * rows
    print(json.dumps(dict(config=name, update=i, seqs=n, rows=rows, response_tokens=toks, device_ms=round(secs * 1e3, 1),
                          rows_per_s=round(rows / secs), tflops=round(flops / secs / 1e12, 1), loss=loss,
                          skipped=skipped)), flush=True)
