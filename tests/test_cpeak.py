"""C_peak calibration: detect_knee / measure_c_peak of
src/roofline.cpp:39-108. The oracle restatement is pinned to the reference's own test
cases (tests/test_roofline.cpp:110-190); the library's host implementation (C-ABI
sgb_detect_knee) must pick the same knee on the same curves; the device latency probe
(the reference CLI's latency_fn, tools/sgrpo.cpp:38-49) runs under -m gpu."""
import math
import random

import numpy as np
import pytest

from oracle import oracle as O


def knee_oracle(c):
    """test_roofline.cpp:83-107 brute force."""
    xmin, xmax = c[0][0], c[-1][0]
    ys = [s for _, s in c]
    ymin, ymax = min(ys), max(ys)
    nx = [(b - xmin) / max(1.0, xmax - xmin) for b, _ in c]
    ny = [(s - ymin) / (ymax - ymin if ymax > ymin else 1.0) for _, s in c]
    x0, y0, x1, y1 = nx[0], ny[0], nx[-1], ny[-1]
    best, bd = 0, -1.0
    for i in range(len(c)):
        d = abs((x1 - x0) * (ny[i] - y0) - (y1 - y0) * (nx[i] - x0)) / math.hypot(x1 - x0, y1 - y0)
        if d > bd:
            bd, best = d, i
    return best


def two_segment(k, n=16, slope=0.5):
    return [(b, 1.0 if b <= k else 1.0 + slope * (b - k)) for b in range(1, n + 1)]


def test_oracle_knee_reference_cases():
    c = [(1, 1), (2, 1), (3, 1), (4, 1), (5, 2), (6, 3)]
    i, _ = O.detect_knee(c)
    assert c[i][0] == 4 and i == knee_oracle(c)
    _, conf = O.detect_knee([(b, b) for b in range(1, 6)])
    assert conf == pytest.approx(0.0, abs=1e-9)
    with pytest.raises(ValueError):
        O.detect_knee([(1, 1), (2, 1), (3, 2)])
    for k in range(3, 9):
        c = two_segment(k)
        i, _ = O.detect_knee(c)
        assert abs(c[i][0] - k) <= 1 and i == knee_oracle(c)
    rng = random.Random(77)
    for _ in range(30):
        k = 3 + rng.randrange(10)
        c = [(b, (1.0 if b <= k else 1.0 + 0.4 * (b - k)) * (1.0 + 0.01 * rng.random())) for b in range(1, 21)]
        i1, c1 = O.detect_knee(c)
        i2, c2 = O.detect_knee([(b * 3 + 5, s * 1e-4 + 2.0) for b, s in c])
        assert i1 == i2 and c1 == pytest.approx(c2, abs=1e-9)


def test_oracle_measure_c_peak_reference_cases():
    r = O.measure_c_peak(lambda b: 1.0 if b <= 4 else 1.0 + 0.5 * (b - 4), 16)
    assert r["c_peak"] == 4 and not r["low_confidence"] and len(r["curve"]) == 16
    r = O.measure_c_peak(lambda b: 0.5 * b, 12)
    assert r["c_peak"] == 12 and r["low_confidence"]
    calls = [0]

    def spiky(b):
        calls[0] += 1
        base = 2.0 if b <= 6 else 2.0 + (b - 6)
        return base * 50 if calls[0] % 7 == 0 else base
    assert O.measure_c_peak(spiky, 16, 2, 9)["c_peak"] == 6
    with pytest.raises(ValueError):
        O.measure_c_peak(lambda b: 1.0, 3)


def test_library_knee_matches_oracle():
    from paper_2509_21792_b200 import capi
    rng = np.random.default_rng(3)
    cases = [two_segment(k) for k in range(3, 9)] + [[(1, 1), (2, 1), (3, 1), (4, 1), (5, 2), (6, 3)]]
    for _ in range(200):
        n = int(rng.integers(4, 64))
        k = int(rng.integers(1, n))
        cases.append([(b, (1.0 if b <= k else 1.0 + rng.uniform(0.05, 2) * (b - k)) * (1 + 0.02 * rng.random()))
                      for b in range(1, n + 1)])
    for c in cases:
        assert capi.detect_knee(c)[0] == O.detect_knee(c)[0]
        assert capi.detect_knee(c)[1] == pytest.approx(O.detect_knee(c)[1], abs=1e-12)
    with pytest.raises(ValueError):
        capi.detect_knee([(1, 1.0), (2, 1.0), (3, 2.0)])


@pytest.mark.gpu
def test_device_c_peak_probe():
    from tests.gpu_common import SMALL, make_engine
    e, _, _ = make_engine(SMALL, max_rows=64)
    r = e.measure_c_peak(24, warmup=1, reps=3)
    lat = [s for _, s in r["latency_curve"]]
    print("c_peak", r["c_peak"], "confidence", r["confidence"], "curve", lat)
    assert len(lat) == 24 and all(s > 0 for s in lat)
    assert 1 <= r["c_peak"] <= 24
    assert O.detect_knee([(b, s) for b, s in r["latency_curve"]])[0] + 1 == r["c_peak"] or r["confidence"] < 0.05
