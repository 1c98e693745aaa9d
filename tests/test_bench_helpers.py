"""bench.py's host-side helpers (no GPU): the per-concurrency break-even table and the c3 stop
caps keyed by global sequence id (so data-parallel shards reproduce the unsharded workload)."""
import os
import sys
from types import SimpleNamespace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _rollout(steps, secs):
    return SimpleNamespace(steps=steps, step_seconds=secs)


def test_per_b_table_buckets_and_break_even():
    # speculative: B = 5 (bucket 4-7) twice with plan (30, 10, 3), once with (1, 0, 0); B = 1 once
    rs = _rollout([(5, 30, 10, 3, 10), (5, 30, 10, 3, 10), (4, 1, 0, 0, 4), (1, 211, 10, 6, 3)],
                  [0.008, 0.008, 0.004, 0.009])
    ra = _rollout([(5, 1, 0, 0, 5), (4, 1, 0, 0, 4), (1, 1, 0, 0, 1)], [0.003, 0.003, 0.002])
    rows = {r["B"]: r for r in bench.per_b_table(rs, ra)}
    assert set(rows) == {"1-1", "4-7"}
    r = rows["4-7"]
    assert r["nkl"] == [30, 10, 3]  # the most frequent plan of the bucket
    assert r["spec_steps"] == 3 and r["ar_steps"] == 2
    ts, ta = (0.008 + 0.008 + 0.004) / 3, 0.003
    assert abs(r["break_even_tau"] - round(ts / ta, 3)) < 1e-9
    tau = 24 / 14
    assert abs(r["tau"] - round(tau, 3)) < 1e-9
    assert abs(r["step_speedup"] - round(tau * ta / ts, 3)) < 1e-9
    assert rows["1-1"]["tau"] == 3.0


def test_stop_caps_keyed_by_global_sid():
    w = dict(bench.WORKLOADS["c3"])
    full = bench.stop_caps(w, 0, 64)
    assert all(w["new"] // 4 <= c <= w["new"] for c in full)
    assert len(set(full)) > 8  # variable-length stops
    # rank r of a data-parallel run computes the caps of its own global sids
    assert bench.stop_caps(w, 16, 16) == full[16:32]
