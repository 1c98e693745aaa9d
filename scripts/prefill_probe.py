import sys; sys.path.insert(0, '.')
from bench import WORKLOADS, make_prompts, model_cfg
from paper_2509_21792_b200 import capi
w = dict(WORKLOADS["c2"]); w["new"] = 1024
eng = capi.Engine(model_cfg(w), 1, 0, 512, 2048, 10, 6); eng.init_random(1234)
pr = make_prompts(w, 0)
for it in range(2):
    r = eng.generate(pr, 8, c_peak=211, mode="adaptive_spec", temperature=0.0, seed=7, max_new_tokens=16, want_features=False)
    print("rollout s", round(r.seconds, 4), "steps", len(r.step_seconds), "sum steps", round(sum(r.step_seconds), 4), "prefill~", round(r.seconds - sum(r.step_seconds), 4))
