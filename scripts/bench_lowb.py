"""Low-concurrency regime at the c2 (or --config c3) shape: per-step device time of AR vs speculative steps
for B sequences (diagnostic for the concurrency-sweep tail). Timing runs are unprofiled; a
second, profiled run gives the per-class split (events around every launch inflate it). Step
times are the engine's per-decode-step CUDA-event times (prefill excluded); the class split
subtracts a profiled prefill-only run.

    python scripts/bench_lowb.py [B ...] [--ncu] [--config=c3|c3r|c5] [--vanilla] [--ctx=N] [--cpeak=C]
      (--ncu: one short run per mode, for ncu; --vanilla: AR steps only)
"""
import json
import sys

sys.path.insert(0, '.')
from bench import WORKLOADS, make_prompts, model_cfg  # noqa: E402
from paper_2509_21792_b200 import capi  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
ncu = "--ncu" in sys.argv
conf = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--config=")), "c2")
modes = ("vanilla",) if "--vanilla" in sys.argv else ("vanilla", "adaptive_spec")
w = dict(WORKLOADS[conf])
ctx_arg = next((int(a.split("=", 1)[1]) for a in sys.argv[1:] if a.startswith("--ctx=")), 0)
c_peak = next((int(a.split("=", 1)[1]) for a in sys.argv[1:] if a.startswith("--cpeak=")), 211)
if ctx_arg:
    w["P"] = ctx_arg  # long prompts stand in for a long generated context
w["new"] = 64  # the engine's max_seq_len = P + new: keep the KV store small
cfg = model_cfg(w)
eng = capi.Engine(cfg, 1, 0, 64, 2048, 10, 6)
eng.init_random(1234)
prompts = make_prompts(w, 0)
for B in [int(x) for x in (args or ["1", "4", "16", "64"])]:
    pr = prompts[:B]
    for mode in modes:
        kw = dict(c_peak=c_peak, temperature=w.get("temp", 0.0), seed=7, max_new_tokens=8 if ncu else 48,
                  want_features=False, acceptance=w.get("acceptance", "strict"))
        eng.generate(pr, 1, mode=mode, **kw)  # warm
        if ncu:
            continue
        r = eng.generate(pr, 1, mode=mode, **kw)
        eng.profile(True)
        rp = eng.generate(pr, 1, mode=mode, **kw)
        eng.profile(False)
        prof = eng.read_profile(reset=True)
        # prefill alone (no decode step), profiled: subtracted so the classes are decode-only;
        # with --ctx also the first decode step (the draft's catch-up over the long prompt)
        base_new = 2 if ctx_arg else 1
        eng.profile(True)
        eng.generate(pr, 1, mode=mode, **dict(kw, max_new_tokens=base_new))
        eng.profile(False)
        pre = eng.read_profile(reset=True)
        n = len(r.steps)
        dec_s = sum(r.step_seconds) if r.step_seconds else r.seconds
        cls = {k: round((v["ms"] - pre.get(k, {}).get("ms", 0.0)) / max(1, n - (base_new - 1)), 3)
               for k, v in prof.items()}
        med = sorted(r.step_seconds)[n // 2] if r.step_seconds else dec_s / n
        # median: with --ctx the first speculative step carries the draft's catch-up over the whole
        # long prompt (a prefill-like cost the real workloads' 128-token prompts do not have)
        print(json.dumps(dict(B=B, mode=mode, steps=n, ms_per_step=round(1e3 * med, 3),
                              ms_per_step_mean=round(1e3 * dec_s / n, 3),
                              profiled_ms_per_step=round(1e3 * sum(rp.step_seconds) / n, 3) if rp.step_seconds else None,
                              tau=round(r.tau(), 3),
                              tok_s=round(r.generated() / dec_s, 1), nkl=r.steps[-1][1:4],
                              launches_per_step=round(r.kernel_launches / n, 1),
                              cls_ms_per_step=cls)), flush=True)
