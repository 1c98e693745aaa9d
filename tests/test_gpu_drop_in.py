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
