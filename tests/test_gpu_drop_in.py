"""The drop-in, end to end: integration/drop_in_demo is a caller written against the
reference's public C++ API only (scheduler.hpp:99-102 generate_dynamic_batch, grpo.hpp:115-116
draft_update), compiled against the unmodified reference headers and linked with
integration/scheduler_b200.cpp, the translation unit that replaces scheduler.cpp / grpo.cpp's
definitions with C-ABI calls. Built by __graft_entry__.build() where /root/reference exists; the
binary travels to the GPU box with the snapshot.

Checked: adaptive speculation == vanilla through the reference types; the T=0 and T=1 token
tables equal the Python binding's rollout of the same prompts (options, seeds and sequence order
plumbed correctly); draft_update consumed every training row and moved the draft."""
import json
import os
import subprocess

import numpy as np
import pytest

from tests.gpu_common import C1, make_engine

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build",
                   "drop_in_demo")


def test_reference_api_caller_runs_on_b200():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/drop_in_demo not built (needs /root/reference at build time)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["lossless"] and r["seqs"] == 32 and r["generated"] > 0
    assert r["spec_steps"] > 0 and 1.0 <= r["tau"]
    assert r["draft_rows"] == r["expected_rows"] > 0
    assert r["draft_params_changed"] > 0 and np.isfinite(r["feature_loss"]) and np.isfinite(r["token_loss"])

    e, _, _ = make_engine(C1, max_seqs=32, max_rows=2048)
    kw = dict(c_peak=64, mode="adaptive_spec", seed=7, max_new_tokens=64, want_features=False)
    assert e.generate(r["prompts"], 4, temperature=0.0, **kw).tokens == r["tokens_t0"]
    assert e.generate(r["prompts"], 4, temperature=1.0, **kw).tokens == r["tokens_t1"]


BUILD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "_build")
CFG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration", "configs",
                   "drop_in_bench.json")
STRATEGIES = ["vanilla", "vanilla+early_term", "fixed_spec", "adaptive_spec", "adaptive_spec+online_draft"]


def _run_bench(binary, cfg=CFG):
    p = subprocess.run([binary, cfg, *STRATEGIES], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, (p.returncode, p.stdout[-3000:], p.stderr[-3000:])
    return p.stdout, json.loads(p.stdout.strip().splitlines()[-1])


def test_reference_bench_runs_unmodified_reference_on_b200():
    """The reference's own bench() (harness.cpp:89-154) -> train_loop (grpo.cpp:280-410) ->
    pretrain_draft / generate_dynamic_batch / draft_update / policy_update, from the UNMODIFIED
    reference objects, with generate_dynamic_batch and draft_update bound to the B200 drop-in
    (weakened reference definitions, integration/Makefile). Every strategy must emit identical
    tokens (the reference's own check), and the shim's counters prove every rollout and draft
    step of train_loop ran on the device."""
    binary = os.path.join(BUILD, "ref_bench")
    if not os.path.exists(binary):
        pytest.skip("integration/_build/ref_bench not built (needs /root/reference at build time)")
    table, r = _run_bench(binary)
    print(table)
    assert r["tokens_identical"] is True
    cfg = json.load(open(CFG))
    iters = cfg["grpo"]["iterations"]
    dev = r["device"]
    # one rollout per strategy per iteration + bench()'s pretrain_draft corpus rollout
    assert dev["rollouts"] == len(STRATEGIES) * iters + 1
    # pretrain_draft's steps + one per iteration of the online-draft strategy
    assert dev["draft_updates"] == cfg["init"]["draft_pretrain_steps"] + iters
    # the draft is re-uploaded only when the host copy differs from the device copy (each
    # train_loop starts from bench()'s draft0 again); the target only if policy_update moved it
    assert dev["draft_uploads"] <= len(STRATEGIES) + 1
    ent = {e["name"]: e for e in r["entries"]}
    assert all(e["iterations"] == iters for e in ent.values())
    assert ent["adaptive_spec"]["tau"] >= 1.0 and ent["fixed_spec"]["tau"] >= 1.0
    assert len({e["tokens_hash"] for e in ent.values()}) == 1
    cpu = os.path.join(BUILD, "ref_bench_cpu")
    if os.path.exists(cpu):
        _, rc = _run_bench(cpu)
        print("CPU reference tokens_hash", rc["entries"][0]["tokens_hash"], "B200", r["entries"][0]["tokens_hash"])


def test_reference_train_loop_with_device_policy_updates():
    """The same through a configuration whose supervised warm-up (the reference's own host
    code) makes rewards vary, so groups survive the zero-variance filter and train_loop calls
    policy_update: every such step runs on the B200 (policy_update drop-in, engine_policy.cu)
    and the reference's token-identity check still passes across all five strategies."""
    binary = os.path.join(BUILD, "ref_bench")
    if not os.path.exists(binary):
        pytest.skip("integration/_build/ref_bench not built (needs /root/reference at build time)")
    cfg = CFG.replace("drop_in_bench.json", "drop_in_bench_policy.json")
    table, r = _run_bench(binary, cfg)
    print(table)
    assert r["tokens_identical"] is True
    assert r["policy_steps"] > 0
    assert r["device"]["policy_updates"] == r["policy_steps"]
