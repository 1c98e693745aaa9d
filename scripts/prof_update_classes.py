"""Draft update at the c3/c4 shape: device time split into the GEMM / LM-head classes (CUDA events
around every GEMM launch) and the rest (training attention, LayerNorm / GELU backward, transposes,
AdamW). python scripts/prof_update_classes.py [n_seqs] [new_tokens]"""
import json
import sys

sys.path.insert(0, '.')
from bench import WORKLOADS, make_prompts, model_cfg  # noqa: E402
from paper_2509_21792_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
new = int(sys.argv[2]) if len(sys.argv) > 2 else 512
w = dict(WORKLOADS["c3"])
eng = capi.Engine(model_cfg(w), 1, 0, max(64, n), 2048, 10, 6)
eng.init_random(1234)
eng.generate(make_prompts(w, 0)[:n], 1, c_peak=211, mode="vanilla", temperature=0.0, seed=1, max_new_tokens=new)
eng.draft_update(None, lr=1e-3)  # warm
(_, _, _, rows, secs), _ = eng.draft_update(None, lr=1e-3)
eng.read_profile(reset=True)
eng.profile(True)
(_, _, _, rows_p, secs_p), _ = eng.draft_update(None, lr=1e-3)
eng.profile(False)
prof = eng.read_profile(reset=True)
gemm_ms = sum(prof[k]["ms"] for k in ("gemm_tcgen05", "lm_head"))
flops = sum(prof[k]["flops"] for k in ("gemm_tcgen05", "lm_head"))
print(json.dumps(dict(rows=rows, device_ms=round(1e3 * secs, 2), profiled_ms=round(1e3 * secs_p, 2),
                      gemm_ms=round(gemm_ms, 2), gemm_tflops=round(flops / (gemm_ms * 1e-3) / 1e12, 1) if gemm_ms else None,
                      gemm_share=round(gemm_ms / (1e3 * secs_p), 3),
                      classes={k: round(v["ms"], 2) for k, v in prof.items()})))
