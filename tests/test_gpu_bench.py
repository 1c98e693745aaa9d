"""bench.py's GPU arm on the smallest BASELINE config (c1): one JSON line carrying the driver
contract's keys (value, e2e with host<->device bytes, gpu_launches, clocks) and this build's
evidence keys (roofline with the kernel-class split and the rollout-level roofline, host_loop)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpu_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c1", "--steps", "1", "--warmup",
                        "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "tau", "host_loop"):
        assert k in d, k
    assert d["metric"] == "rollout tokens/s" and d["value"] > 0 and d["n_gpus"] == 1 and d["warmup"] >= 3
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["e2e"]["value"] <= d["value"] * 1.01  # end to end includes the host copies
    assert d["gpu_launches"] > 0
    ro = d["roofline"]
    assert ro["bound"] == "hbm" and ro["peak"] > 0 and 0 < ro["frac"] <= 1.2
    assert set(ro["classes"]) >= {"gemm_tcgen05", "attention", "rowops", "lm_head", "sample", "tree", "kv_commit"}
    assert 0 < ro["rollout"]["frac"] <= 1.2
    hl = d["host_loop"]
    assert hl["decode_steps"] > 0 and hl["device_us_per_step"] > 0 and 0 <= hl["gap_share_of_device_time"] < 1
