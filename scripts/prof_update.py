"""Draft-update anatomy at the c3/c4 shape: one rollout, then draft_update steps (for ncu).
    python scripts/prof_update.py [config] [n_seqs] [new_tokens] [updates]"""
import sys
import time

sys.path.insert(0, '.')
from bench import WORKLOADS, make_prompts, model_cfg  # noqa: E402
from paper_2509_21792_b200 import capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
new = int(sys.argv[3]) if len(sys.argv) > 3 else 512
ups = int(sys.argv[4]) if len(sys.argv) > 4 else 2
w = dict(WORKLOADS[name])
eng = capi.Engine(model_cfg(w), 1, 0, max(64, n), 2048, 10, 6)
eng.init_random(1234)
r = eng.generate(make_prompts(w, 0)[:n], 1, c_peak=211, mode="vanilla", temperature=0.0, seed=1, max_new_tokens=new)
for i in range(ups):
    t0 = time.time()
    (fl, tl, _, rows, secs), _ = eng.draft_update(None, lr=1e-3)
    print(f"update {i}: rows {rows} device {secs*1e3:.1f} ms wall {(time.time()-t0)*1e3:.1f} ms "
          f"({secs / rows * 1e6:.2f} us/row)", flush=True)
