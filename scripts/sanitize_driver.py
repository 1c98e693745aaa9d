"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family of the
engine at toy shapes -- tcgen05 GEMM incl. split-K finisher and raw-partial paths, attention.cu (per-row,
shared tiles with in-register merge and tickets), attention_tree.cu, sampling (T=0, T>0 keyed + exact
pass, rejection sampling), tree kernels, KV commit, draft update, policy update."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (weights / configs only)
from paper_2509_21792_b200 import capi  # noqa: E402

cfg = O.ModelConfig(vocab_size=256, d_model=128, n_layers=2, n_heads=2, d_ff=256, max_seq_len=96, seed=5)
e = capi.Engine(cfg, 1, 0, 16, 512, 6, 3)
e.policy_enable()
e.upload_target(O.init_model(cfg).flat)
e.upload_draft(O.init_draft(cfg, 1).flat)
rng = np.random.default_rng(0)
prompts = [rng.integers(2, 256, 9).tolist() for _ in range(3)]
for mode, temp, acc in [("vanilla", 0.0, "strict"), ("adaptive_spec", 0.0, "strict"), ("adaptive_spec", 1.0, "strict"),
                        ("adaptive_spec", 1.0, "rejection")]:
    r = e.generate(prompts, 4, c_peak=48, k_max=6, l_max=3, mode=mode, temperature=temp, seed=3, max_new_tokens=12,
                   acceptance=acc)
e.draft_update(None)
e.policy_update([(t, 9, 0.5) for t in r.tokens[:4]])
# the attention self-tests (per-row vs shared tiles vs the tree kernel) and a split-K GEMM
q = rng.standard_normal((30, 256)).astype(np.float32)
kc = rng.standard_normal((70, 256)).astype(np.float32)
kn = rng.standard_normal((30, 256)).astype(np.float32)
par = [[-1, 0, 0, 1, 1, 2, 3, 3, 5, 6, 7, 8, 9, 10, 11], [-1, 0, 1, 2, 3, 4, 5, 0, 0, 8, 9, 10, 11, 12, 13]]
capi.debug_tree_attention([40, 30], par, q, kc, kc, kn, kn, 2)
capi.debug_tree_attention_tree([40, 30], par, q, kc, kc, kn, kn, 2)
capi.debug_gemm(rng.standard_normal((256, 1024)).astype(np.float32), rng.standard_normal((3, 1024)).astype(np.float32),
                splits=4)
print("sanitize driver ok")
