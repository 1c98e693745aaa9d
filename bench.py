"""Rollout benchmark of the B200-native GRPO-rollout hot path (arXiv 2509.21792).

Metric (BASELINE.json): rollout tokens/s, speedup vs AR decode, mean accept length tau.
Workload (default, BASELINE configs[1] "c2"): Qwen2.5-1.5B-shaped target on the reference
architecture (d=1536, L=28, H=12, d_ff=8960, V=151936) + 1-layer EAGLE-style draft,
64 queries x group 8, 128-token synthetic prompts, 1024 new tokens, greedy, adaptive
speculative decoding (Eqs. 1-3, alpha=2, K_max=10, L_max=6, C_peak=211). Random-init
weights of that architecture drawn on the device (init_flat's distributions).

One "step" = one full rollout (prefill + decode until every sequence finished).
  value  = generated tokens / device time (CUDA events; prompts resident in HBM)
  e2e    = generated tokens / wall time of the public C-ABI call sgb_rollout with host
           prompts in and host tokens + features out (H2D/D2H inside the timed region)
Multi-GPU (torchrun): data-parallel by query group, weak scaling -- every rank runs its own
64x8 shard with global sequence ids; no collective on the data path; time = max over ranks.

--impl reference times the reference's own CPU generate_dynamic_batch (oracle/_ref, the
unmodified reference sources compiled here) on the host cores.
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # V, d, L, H, dff; P prompt tokens, G group, Q queries per GPU, new max new tokens
    "c2": dict(V=151936, d=1536, L=28, H=12, dff=8960, P=128, G=8, Q=64, new=1024, stops=False, online=False, warm=0,
               desc="Qwen2.5-1.5B-shaped target + 1-layer draft, 64 queries x group 8, 128-token prompts, "
                    "1024 new tokens, greedy, adaptive spec (c_peak 211)"),
    # c3 per-GPU shard (BASELINE configs[2] is 128 queries x 8 over the box: 16 x 8 per GPU)
    "c3": dict(V=152064, d=3584, L=28, H=28, dff=18944, P=128, G=8, Q=16, new=1024, stops=True, online=False, warm=24,
               desc="Qwen2.5-7B-shaped target + 1-layer draft, 16 queries x group 8 per GPU (c3's 128 x 8 over 8 "
                    "GPUs), 128-token prompts, variable-length stops 256..1024 new tokens (concurrency sweep "
                    "128 -> 1 per GPU), greedy, adaptive spec, draft warmed online"),
    # c3 sampled at T=1 (the reference TrainConfig default rollout temperature, grpo.hpp:142) with
    # rejection-sampling acceptance: the same shard, stops and warm-up stream as c3
    "c3r": dict(V=152064, d=3584, L=28, H=28, dff=18944, P=128, G=8, Q=16, new=1024, stops=True, online=False,
                warm=24, temp=1.0, acceptance="rejection",
                desc="Qwen2.5-7B-shaped target + 1-layer draft, 16 queries x group 8 per GPU, variable-length stops "
                     "256..1024, T=1.0 rejection-sampling verify (GRPO's sampled rollouts), draft warmed online at T=1"),
    # c4: the c3 shard + the online draft-learning step (NCCL gradient all-reduce) in every step
    "c4": dict(V=152064, d=3584, L=28, H=28, dff=18944, P=128, G=8, Q=16, new=1024, stops=True, online=True, warm=24,
               desc="Qwen2.5-7B-shaped GRPO rollout, data-parallel by query group, 16 queries x group 8 per GPU, "
                    "variable-length stops 256..1024, adaptive spec + one online draft-learning AdamW step with "
                    "NCCL gradient all-reduce per step"),
    # c5 (BASELINE configs[4]): Llama-3-8B shape, rejection-sampling verify at T=1.0, 256 queries x
    # group 16 over 8 GPUs = the full per-GPU shard of 32 queries x 16 = 512 sequences x 4224
    # positions. Its KV (524 KB per token, 1.1 TB) is 6x one GPU's HBM, so the rollout runs in
    # waves over `regions` resident KV regions (engine admission); features are not
    # returned (35 GB per rollout), tokens are
    "c5": dict(V=128256, d=4096, L=32, H=32, dff=14336, P=128, G=16, Q=32, new=4096, stops=False, online=False,
               warm=24, warm_new=256, warm_prompts=24, temp=1.0, acceptance="rejection", features=False, regions=48,
               rows=1024,
               desc="Llama-3-8B-shaped target + 1-layer draft, rejection-sampling verify at T=1.0, 32 queries x "
                    "group 16 per GPU (the full 256 x 16 shard of 8 GPUs), 128-token prompts, 4096 new tokens, "
                    "adaptive spec, KV-region waves (48 resident sequences), draft warmed online (T=1 rollouts of "
                    "256 tokens on a disjoint prompt stream)"),
    "c1": dict(V=512, d=256, L=2, H=4, dff=1024, P=32, G=4, Q=8, new=128, stops=False, online=False, warm=0,
               desc="2-layer d=256 target + 1-layer draft, 8 queries x group 4, 32-token prompts, 128 new tokens"),
}
C_PEAK = 211  # analytic crossover s*F/(2*BW) at the measured sustained peaks


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def model_cfg(w):
    from paper_2509_21792_b200.capi import ModelConfig
    return ModelConfig(w["V"], w["d"], w["L"], w["H"], w["dff"], w["P"] + w["new"], 1)


def make_prompts(w, rank):
    """Uniform ids in [2, V) from a splitmix stream keyed by (run_seed=0, 0x9a01), SURVEY §8d;
    rank r takes global queries [r*Q, (r+1)*Q)."""
    from paper_2509_21792_b200.capi import mix_key
    seed = mix_key(0, 0x9A01)
    n = (rank + 1) * w["Q"] * w["P"]
    with np.errstate(over="ignore"):
        st = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * np.arange(2, n + 2, dtype=np.uint64)
        z = (st ^ (st >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    toks = (z % np.uint64(w["V"] - 2) + np.uint64(2)).astype(np.int64)
    toks = toks[rank * w["Q"] * w["P"]:].reshape(w["Q"], w["P"])
    return [row.tolist() for row in toks]


def _splitmix_stream(seed, n):
    with np.errstate(over="ignore"):
        st = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * np.arange(2, n + 2, dtype=np.uint64)
        z = (st ^ (st >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def stream_prompts(key, n, P, V):
    """Training prompts for online draft learning, disjoint from the benchmark prompts:
    Rng(mix_key(0, key)) (key = 0x7a11 + iteration)."""
    from paper_2509_21792_b200.capi import mix_key
    z = _splitmix_stream(mix_key(0, key), n * P)
    return (z % np.uint64(V - 2) + np.uint64(2)).astype(np.int64).reshape(n, P).tolist()


def stop_caps(w, sid0, n):
    """c3 variable-length stops: per-sequence max_new from Rng(mix_key(0, 0x5709 + sid)),
    uniform in [new/4, new] (max/min = 4x), keyed by GLOBAL sequence id."""
    from paper_2509_21792_b200.capi import mix_key
    lo, hi = w["new"] // 4, w["new"]
    caps = []
    for sid in range(sid0, sid0 + n):
        z = _splitmix_stream(mix_key(0, 0x5709 + sid), 1)[0]
        caps.append(int(lo + int(z % np.uint64(hi - lo + 1))))
    return caps


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].lower() in ("active", "0x1", "yes")})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)]
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def ncu_traffic(name):
    """dram read+write bytes of one attention launch from the committed ncu --set full summary
    (profiles/), with that launch's algorithmic bytes: traffic/algorithmic ~1 means no re-reads."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)
    t = a = None
    try:
        for line in open(path):
            if line.strip().startswith("traffic (dram read+write, bytes)"):
                t = float(line.split()[-1])
            elif line.strip().startswith("algorithmic bytes"):
                a = float(line.split()[-1])
    except OSError:
        return None, None, None
    return t, a, (f"profiles/{name}: ncu --set full of a c2 attention launch inside the bench workload (step 500, 512 rows x 629 keys)" if t else None)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ------------------------------------------------------------------------------ CPU legs
def cpu_reference_sample(w, threads, new_tokens=8, prompt_len=16):
    """The reference's own generate_dynamic_batch (oracle/_ref) on `threads` host threads,
    one sequence per thread, at the full model shape (bounded sample). Returns dict."""
    import ctypes as C
    from oracle import refc as R
    from oracle.oracle import ModelConfig
    cfg = ModelConfig(w["V"], w["d"], w["L"], w["H"], w["dff"], w["P"] + w["new"], 1)
    n = R.lib().sgref_param_count(C.byref(R.cfg_c(cfg)))
    rng = np.random.default_rng(1)
    flat = np.empty(n, np.float32)
    for o in range(0, n, 1 << 26):
        m = min(1 << 26, n - o)
        flat[o:o + m] = rng.standard_normal(m, dtype=np.float32) * np.float32(0.02)
    R.lib().sgref_model_new_weights.restype = C.c_void_p
    h = R.lib().sgref_model_new_weights(C.byref(R.cfg_c(cfg)), flat.ctypes.data_as(C.POINTER(C.c_float)))
    del flat
    model = R.RefModel.__new__(R.RefModel)
    model.cfg, model.h = cfg, h
    draft = R.RefDraft(cfg, 1)
    prompts = [p[:prompt_len] for p in make_prompts(w, 0)[:threads]]
    return model, draft, prompts, dict(c_peak=C_PEAK, mode="vanilla", temperature=0.0, seed=7,
                                       max_new_tokens=new_tokens)


def run_cpu_sample(ctx, threads):
    from oracle import refc as R
    model, draft, prompts, kw = ctx
    n, secs = R.generate_threaded(model, draft, prompts, 1, threads, **kw)
    return n, secs


def cpu_baseline(w, threads):
    """rank 0, N=1 only: one bounded sample of the reference CPU path."""
    from oracle import refc as R
    if not R.available():
        return {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built on this host"}
    ctx = cpu_reference_sample(w, threads)
    n, secs = run_cpu_sample(ctx, threads)
    return {"value": n / secs, "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": f"{threads} sequences x (16-token prompt, 8 new tokens), vanilla greedy, full model shape, "
                      f"{n} tokens in {secs:.1f}s (reference is single-threaded; one sequence per thread)"}


def reference_arm(args, w):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from oracle import refc as R
    threads = max(1, min(os.cpu_count() or 1, 64))
    base = {"impl": "reference", "metric": "rollout tokens/s", "unit": "tokens/s", "n_gpus": args.gpus,
            "higher_is_better": True, "scaling": "weak", "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {w['desc']}", "sample": "bounded CPU sample"}}
    if not R.available():
        base["unavailable"] = "oracle/_ref/libsgrpo_ref.so not built (needs /root/reference at build time)"
        print(json.dumps(base))
        return 0
    ctx = cpu_reference_sample(w, threads)
    for _ in range(args.warmup):
        run_cpu_sample(ctx, threads)
    tot_n, tot_s = 0, 0.0
    for _ in range(args.steps):
        n, s = run_cpu_sample(ctx, threads)
        tot_n += n
        tot_s += s
    v = tot_n / tot_s
    base.update(value=v, steps=args.steps, warmup=args.warmup, ms_per_step=1e3 * tot_s / args.steps,
                vs_baseline=None,
                cpu_baseline={"value": v, "unit": "tokens/s", "cores": threads, "kind": "reference",
                              "sample": f"{threads} sequences x (16-token prompt, 8 new tokens) per step, vanilla "
                                        f"greedy, full {args.config} shape, one sequence per host thread"},
                e2e={"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(base))
    return 0


def per_b_table(rs, ra):
    """Per live-concurrency bucket: mean device seconds of a speculative step vs an AR step at the
    same B, tau there, the break-even tau (= t_spec / t_ar) and the per-step speedup
    tau * t_ar / t_spec (SURVEY §7 hard part 8's table, measured)."""
    def buckets(r):
        out = {}
        for (b, n, k, l, acc), sec in zip(r.steps, r.step_seconds):
            lo = 1 << (max(1, b).bit_length() - 1)  # power-of-two bucket [lo, 2lo)
            e = out.setdefault(lo, [0, 0.0, 0, 0, collections.Counter()])
            e[0] += 1
            e[1] += sec
            e[2] += acc
            e[3] += b
            e[4][(n, k, l)] += 1
        for e in out.values():
            e[4] = e[4].most_common(1)[0][0]  # the bucket's most frequent (N, K, L) plan
        return out
    bs, ba = buckets(rs), buckets(ra)
    rows = []
    for lo in sorted(bs):
        if lo not in ba:
            continue
        ns, ss, acs, bsum, nkl = bs[lo]
        na, sa, _, _, _ = ba[lo]
        ts, ta = ss / ns, sa / na
        tau = acs / bsum if bsum else None
        rows.append({"B": f"{lo}-{2 * lo - 1}", "nkl": list(nkl), "spec_ms": round(1e3 * ts, 3),
                     "ar_ms": round(1e3 * ta, 3), "tau": round(tau, 3) if tau else None,
                     "break_even_tau": round(ts / ta, 3), "step_speedup": round(tau * ta / ts, 3) if tau else None,
                     "spec_steps": ns, "ar_steps": na})
    return rows


def rollout_roofline(eng, hbm, tf):
    """SURVEY §8(d) rollout-level roofline of the last rollout: sum over decode steps of
    max(bytes_t / BW, flops_t / F) vs the measured device time of those steps."""
    b, f, s = eng.rollout_roofline()
    if len(b) == 0:
        return None
    roof = float(np.sum(np.maximum(b / (hbm * 1e9), f / (tf * 1e12))))
    meas = float(np.sum(s))
    return {"roofline_s": round(roof, 4), "measured_s": round(meas, 4), "frac": round(roof / meas, 4) if meas else None,
            "bytes": float(np.sum(b)), "flops": float(np.sum(f)), "steps": int(len(b)),
            "definition": "sum_t max(bytes_t/HBM, flops_t/bf16_sustained) over decode steps (prefill excluded) / "
                          "their CUDA-event time; bytes/flops per SURVEY 8(d): bf16 weights once per target / draft "
                          "pass, every sequence's K/V, verify-row K/V writes, logits"}


# ------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--mode", default="adaptive_spec", choices=["adaptive_spec", "vanilla"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ar", action="store_true", help="skip the AR (vanilla) comparison rollout")
    ap.add_argument("--max-new", type=int, default=0, help="override new tokens (profiling runs)")
    ap.add_argument("--warm-iters", type=int, default=-1, help="online draft-warming iterations (default per config)")
    ap.add_argument("--c-peak", type=int, default=C_PEAK)
    ap.add_argument("--acceptance", default=None, choices=["strict", "rejection"],
                    help="verify acceptance (default per config: c5 rejection sampling, else strict match)")
    ap.add_argument("--warmup-max-new", type=int, default=0,
                    help="new tokens of the warm-up rollouts (0: the workload's); long workloads (c5) warm up short")
    ap.add_argument("--no-profile", action="store_true", help="skip the per-kernel-class profiled rollout")
    args = ap.parse_args()
    w = dict(WORKLOADS[args.config])
    if args.max_new:
        w["new"] = args.max_new
    if args.warm_iters >= 0:
        w["warm"] = args.warm_iters
    if args.acceptance:
        w["acceptance"] = args.acceptance
    if args.impl == "reference":
        return reference_arm(args, w)

    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)  # host plumbing only
    from paper_2509_21792_b200 import capi
    cfg = model_cfg(w)
    n_seq = w["Q"] * w["G"]
    regions = w.get("regions", n_seq)  # resident KV regions (fewer than sequences: waves)
    max_seqs = min(n_seq, regions) if "regions" in w else max(n_seq, 64 if w["warm"] > 0 else 1)
    eng = capi.Engine(cfg, 1, local, max_seqs, w.get("rows", 2048), 10, 6)
    eng.init_random(1234)
    # NCCL data-parallel group over NVLink (C1 gradient all-reduce, C2 statistics)
    uid = [capi.nccl_unique_id() if rank == 0 else None]
    if dist:
        dist.broadcast_object_list(uid, src=0)
    eng.nccl_init(rank, world, uid[0])
    prompts = make_prompts(w, rank)
    caps = stop_caps(w, rank * n_seq, n_seq) if w["stops"] else None
    gen = dict(c_peak=args.c_peak, alpha=2.0, k_max=10, l_max=6, temperature=w.get("temp", 0.0), seed=7,
               max_new_tokens=w["new"], sid_offset=rank * n_seq, seq_max_new=caps,
               acceptance=w.get("acceptance", "strict"))
    want_feats = w.get("features", True)

    def rollout(mode, **over):
        t0 = time.perf_counter()
        r = eng.generate(prompts, w["G"], mode=mode, want_features=want_feats, **dict(gen, **over))
        return r, time.perf_counter() - t0

    adv_stats = {"ms": 0.0, "calls": 0, "groups": 0, "filtered": 0, "reward_mean": 0.0}

    def group_rewards(r, g):
        """group rewards + standardized advantages of this rollout on the device (grpo.cpp:
        99-136, 352-380) and the data-parallel gather of every rank's rewards (NCCL
        all-gather). Synthetic prompts carry no addition task: the answer key is 0."""
        t0 = time.perf_counter()
        rw, _, valid = eng.group_advantages([0] * (len(r.tokens) // g), g)
        allr = eng.allgather_f64(rw, world)
        adv_stats["ms"] += 1e3 * (time.perf_counter() - t0)
        adv_stats["calls"] += 1
        adv_stats["groups"] += len(valid) * world
        adv_stats["filtered"] += int(len(valid) - int(np.sum(valid)))
        adv_stats["reward_mean"] = float(np.mean(allr))

    def draft_step(r, g):
        """one online draft-learning step on this rollout (grpo.cpp:329-345): global row
        count first (int64 all-reduce), local gradient with the global normaliser, NCCL
        all-reduce (sum) of the fp32 gradient, identical AdamW step on every replica."""
        group_rewards(r, g)
        rows = sum(max(0, len(t) - 2) for t in r.tokens)
        rows_total = int(eng.allreduce_i64([rows])[0])  # noqa: F841 (used below)
        t0 = time.perf_counter()
        (fl, tl, _, n, secs), _ = eng.draft_update(None, lr=1e-3, rows_total=rows_total, allreduce_grad=True)
        return secs, time.perf_counter() - t0, fl, tl, rows_total

    # ---- draft warming (untimed): online learning on a disjoint prompt stream
    warm = None
    if w["warm"] > 0:
        t0 = time.perf_counter()
        fl = tl = None
        for it in range(1, w["warm"] + 1):
            tp = stream_prompts(0x7A11 + it + 1000 * rank, w.get("warm_prompts", 32), w["P"], w["V"])
            # training rollouts follow the workload's own length distribution (stop caps keyed by
            # sids disjoint from the benchmark's), so the draft sees the contexts it will serve
            caps_w = stop_caps(w, 1_000_000 + 64 * (it + 1000 * rank), 64) if w["stops"] else None
            rw = eng.generate(tp, 2, c_peak=args.c_peak, mode="vanilla", temperature=w.get("temp", 0.0), seed=it,
                              max_new_tokens=w.get("warm_new", w["new"]), want_features=True, seq_max_new=caps_w)
            for _ in range(4):
                _, _, fl, tl, _ = draft_step(rw, 2)
        warm = {"iterations": w["warm"], "adamw_steps": 4 * w["warm"], "train_seqs_per_iter": 2 * w.get("warm_prompts", 32),
                "feature_loss": round(fl, 5), "token_loss": round(tl, 4), "seconds": round(time.perf_counter() - t0, 1)}

    for _ in range(args.warmup):
        wover = {}
        if args.warmup_max_new:
            wover = dict(max_new_tokens=args.warmup_max_new, seq_max_new=None)
        r, _ = rollout(args.mode, **wover)
        if w["online"]:
            draft_step(r, w["G"])
    eng.read_profile(reset=True)
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    dev_s, wall_s, toks, launches, acc, slots, h2d, d2h = 0.0, 0.0, 0, 0, 0, 0, 0, 0
    spec_steps, upd_s, upd_wall, upd_rows = 0, 0.0, 0.0, 0
    host_gap, host_enq, n_dec = 0.0, 0.0, 0
    terms = None
    last = None
    hbm0, tf0, _ = measured_peaks()
    roof_last = None
    for _ in range(args.steps):
        r, wall = rollout(args.mode)
        last = r
        roof_last = rollout_roofline(eng, hbm0, tf0)
        dev_s += r.seconds
        wall_s += wall
        if w["online"]:
            us, uw, fl, tl, nrows = draft_step(r, w["G"])
            dev_s += us
            wall_s += uw
            upd_s += us
            upd_wall += uw
            upd_rows += nrows
            terms = (fl, tl)
        toks += r.generated()
        launches += r.kernel_launches
        acc += r.total_accepted
        slots += r.total_verify_slots
        h2d += r.h2d_bytes
        d2h += r.d2h_bytes
        spec_steps += sum(1 for s in r.steps if s[1] > 1)
        host_gap += r.host_gap_seconds
        host_enq += r.host_enqueue_seconds
        n_dec += len(r.steps)
    clk = clocks.stop()
    # C2: statistics over the data-parallel group (NCCL); times take the max over ranks
    t_max, w_max = dev_s, wall_s
    tok_all, acc_all, slots_all = toks, acc, slots
    if world > 1:
        import torch
        t = torch.tensor([dev_s, wall_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max, w_max = float(t[0]), float(t[1])
        tok_all, acc_all, slots_all = (int(x) for x in eng.allreduce_i64([toks, acc, slots]))
    ar = None
    if not args.no_ar and args.mode != "vanilla":
        if spec_steps == 0:
            ar = {"value": tok_all / t_max, "unit": "tokens/s", "speedup": 1.0,
                  "note": "every step had B_cur > C_peak, so Eqs. 1-3 planned N_verify=1 (AR) throughout"}
        else:
            rs = last  # the last timed rollout
            ra, _ = rollout("vanilla")
            same = all(list(a) == list(b) for a, b in zip(rs.tokens, ra.tokens))
            ar = {"value": ra.generated() / ra.seconds, "unit": "tokens/s",
                  "spec_value": rs.generated() / rs.seconds,
                  "speedup": (rs.generated() / rs.seconds) / (ra.generated() / ra.seconds),
                  "tokens_identical": same, "note": "rollout only (no draft step), this rank",
                  "per_concurrency": per_b_table(rs, ra)}
            if gen["acceptance"] == "rejection":
                ar["note"] += ("; rejection sampling is lossless in distribution: token streams differ from "
                               "AR sampling by design (the strict-match mode is the token-identical one)")
    # kernel-class breakdown: one more rollout of the same workload with a CUDA-event pair
    # around every launch (kept out of the timed steps: events between launches defeat PDL)
    if not args.no_profile:
        eng.profile(True)
        rollout(args.mode)
        eng.profile(False)
    prof = eng.read_profile(reset=True)
    if rank != 0:
        eng.close()
        if dist:
            dist.destroy_process_group()
        return 0
    hbm, tf, src = measured_peaks()
    att = prof["attention"]
    ach = att["bytes"] / (att["ms"] * 1e-3) / 1e9 if att["ms"] else 0.0
    total_ms = sum(v["ms"] for v in prof.values())
    traffic, traffic_alg, traffic_src = ncu_traffic("r02_attn_c2_inworkload.txt")
    roofline = {"bound": "hbm", "kernel": "attn_kernel (mma.sync tree/paged KV attention: shared-prefix tiles, bulk-DMA ring, in-kernel block merge)",
                "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                "traffic": traffic, "traffic_algorithmic": traffic_alg, "traffic_source": traffic_src,
                "achieved_note": "algorithmic bytes = each sequence's context K/V per layer (SURVEY 8d), prompt "
                                 "included; at <= 16 heads the G members of a group stage their shared prompt "
                                 "once per tile, so DRAM bytes are below the algorithmic bytes",
                "peak_source": src,
                "share_of_step": round(att["ms"] / total_ms, 4) if total_ms else None,
                "measured": "per-launch CUDA events on the engine stream, one profiled rollout after the timed steps",
                "classes": {k: {"ms_per_step": round(v["ms"], 2),
                                "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None,
                                "TFLOPs": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 1) if v["ms"] else None,
                                "launches": v["launches"]} for k, v in prof.items()}}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, max(1, min(os.cpu_count() or 1, 64)))
    config = {"workload": f"{args.config}: {w['desc']}", "mode": args.mode, "c_peak": args.c_peak,
              "acceptance": w.get("acceptance", "strict"), "temperature": w.get("temp", 0.0),
              "sequences_per_gpu": n_seq, "resident_kv_regions": min(n_seq, regions), "new_tokens": w["new"],
              "prompt_len": w["P"], "features_returned": want_feats,
              "l2": "inputs larger than L2 (KV cache of the shard >> 126 MB L2)",
              "parallelism": f"dp{world} (query groups)", "weights": "random init on device"}
    if caps:
        config["stops"] = {"min_new": min(caps), "max_new": max(caps), "mean_new": round(sum(caps) / len(caps), 1)}
    line = {
        "metric": "rollout tokens/s", "value": round(tok_all / t_max, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_max / args.steps, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": config,
        "tau": round(acc_all / slots_all, 4) if slots_all else None, "spec_steps": spec_steps,
        "speedup_vs_ar": ar["speedup"] if ar else None, "ar": ar, "draft_warm": warm,
        "e2e": {"value": round(tok_all / w_max, 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d // args.steps,
                "d2h_bytes_per_step": d2h // args.steps},
        "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
    }
    if roof_last:
        line["roofline"]["rollout"] = roof_last
    if n_dec:
        # the host side of the step loop (one sync per step): device idle from each step's end to
        # the next step's first operation, and host time issuing a step -- what a device-resident
        # (CUDA graph) step loop could remove
        line["host_loop"] = {"decode_steps": n_dec, "gap_us_per_step": round(1e6 * host_gap / n_dec, 1),
                             "gap_share_of_device_time": round(host_gap / dev_s, 4),
                             "enqueue_us_per_step": round(1e6 * host_enq / n_dec, 1),
                             "device_us_per_step": round(1e6 * (dev_s - upd_s) / n_dec, 1)}
    if w["online"]:
        line["online_draft_step"] = {"device_ms_per_step": round(1e3 * upd_s / args.steps, 2),
                                     "wall_ms_per_step": round(1e3 * upd_wall / args.steps, 2),
                                     "global_rows_per_step": upd_rows // args.steps,
                                     "share_of_step": round(upd_s / dev_s, 4),
                                     "feature_loss": round(terms[0], 5), "token_loss": round(terms[1], 4),
                                     "collective": f"ncclAllReduce(sum) fp32 gradient over {world} rank(s)",
                                     "group_advantages": {
                                         "wall_ms_per_step": round(adv_stats["ms"] / max(1, adv_stats["calls"]), 3),
                                         "groups_per_step": w["Q"] * world, "reward_mean": adv_stats["reward_mean"],
                                         "collective": f"ncclAllGather fp64 rewards over {world} rank(s)"}}
    print(json.dumps(line))
    eng.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
