"""Golden fixtures for GRPO rewards / advantages, generated from the REAL reference.

    make -C oracle && python tests/golden/make_golden_rewards.py

compute_reward (src/grpo.cpp:99-116) on crafted responses (well-formed answers, wrong
answers, several '=', an EOS in the middle or at the end, non-digit tokens, > 15 digits,
empty) and standardize_advantages (grpo.cpp:121-136) on reward vectors for G in
{2,3,4,5,8,16} (0/1 patterns as produced by the reward, plus fractional ones). Values come
from oracle/_ref/libsgrpo_ref.so through oracle/ref_capi.cpp; doubles are stored as hex.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import refc as R  # noqa: E402

lib = R.lib()
lib.sgref_compute_reward.restype = C.c_double
lib.sgref_compute_reward.argtypes = [C.c_longlong, C.c_longlong, C.POINTER(C.c_int), C.c_int]
lib.sgref_standardize_advantages.argtypes = [C.POINTER(C.c_double), C.c_int, C.c_double, C.POINTER(C.c_double)]
rng = np.random.default_rng(2509)


def enc(n):
    return [2 + int(c) for c in str(n)]


cases = []
for _ in range(300):
    a, b = int(rng.integers(0, 10 ** int(rng.integers(1, 6)))), int(rng.integers(0, 10 ** int(rng.integers(1, 6))))
    kind = int(rng.integers(0, 9))
    noise = rng.integers(0, 20, size=int(rng.integers(0, 12))).tolist()
    if kind == 0:
        resp = noise + [13] + enc(a + b) + [1]
    elif kind == 1:
        resp = noise + [13] + enc(a + b)
    elif kind == 2:
        resp = noise + [13] + enc(a + b + 1) + [1]
    elif kind == 3:
        resp = [13] + enc(a + b) + [13] + enc(a + b) + [1]
    elif kind == 4:
        resp = noise + [13] + enc(a + b) + [1, 5]
    elif kind == 5:
        resp = noise + [13] + enc(a + b)[:1] + [12] + enc(a + b)[1:]
    elif kind == 6:
        resp = noise + [13] + [2 + int(x) for x in rng.integers(0, 10, size=16)]
    elif kind == 7:
        resp = noise + [13]
    else:
        resp = noise
    arr = (C.c_int * max(1, len(resp)))(*resp)
    cases.append({"a": a, "b": b, "resp": resp, "reward": lib.sgref_compute_reward(a, b, arr, len(resp)).hex()})

groups = []
for g in (2, 3, 4, 5, 8, 16):
    for _ in range(40):
        if rng.random() < 0.8:
            r = rng.integers(0, 2, size=g).astype(np.float64)
        else:
            r = np.round(rng.random(g), 3)
        buf = (C.c_double * g)(*r.tolist())
        out = (C.c_double * g)()
        ok = lib.sgref_standardize_advantages(buf, g, 1e-8, out)
        groups.append({"g": g, "rewards": [float(x).hex() for x in r], "valid": int(ok),
                       "adv": [float(out[i]).hex() for i in range(g)] if ok else None})

json.dump({"rewards": cases, "advantages": groups, "eps_var": (1e-8).hex()},
          open(os.path.join(ROOT, "tests", "golden", "rewards.json"), "w"))
print(len(cases), "reward cases,", len(groups), "groups")
