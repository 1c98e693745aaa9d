"""Per-step device cost of a speculative step vs an AR step at fixed concurrency B.

    python scripts/step_costs.py [c3|c2] [B ...]

For each B: B distinct prompts (g=1), 48 new tokens, vanilla and adaptive_spec rollouts,
median step seconds of each and the kernel-class split of the speculative rollout.
"""
import json
import statistics
import sys

sys.path.insert(0, '.')
from bench import WORKLOADS, make_prompts, model_cfg  # noqa: E402
from paper_2509_21792_b200 import capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
Bs = [int(x) for x in sys.argv[2:]] or [1, 4, 16, 64]
w = dict(WORKLOADS[name])
w["Q"] = max(Bs)
cfg = model_cfg(w)
eng = capi.Engine(cfg, 1, 0, max(Bs), 2048, 10, 6)
eng.init_random(1234)
allp = make_prompts(w, 0)
for B in Bs:
    pr = allp[:B]
    out = dict(B=B)
    for mode in ("vanilla", "adaptive_spec"):
        eng.generate(pr, 1, c_peak=211, mode=mode, temperature=0.0, seed=7, max_new_tokens=8, want_features=False)
        r = eng.generate(pr, 1, c_peak=211, mode=mode, temperature=0.0, seed=7, max_new_tokens=48,
                         want_features=False)
        eng.profile(True)
        eng.generate(pr, 1, c_peak=211, mode=mode, temperature=0.0, seed=7, max_new_tokens=48, want_features=False)
        eng.profile(False)
        prof = eng.read_profile(reset=True)
        st = r.step_seconds[2:] or r.step_seconds
        out[mode] = dict(step_ms=round(1e3 * statistics.median(st), 3), tau=round(r.tau(), 3),
                         plan=r.steps[-1][1:4],
                         classes={k: round(v["ms"] / max(1, len(r.steps)), 3) for k, v in prof.items() if v["ms"]})
    out["ratio"] = round(out["adaptive_spec"]["step_ms"] / out["vanilla"]["step_ms"], 3)
    print(json.dumps(out), flush=True)
