"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container (needs /root/reference and oracle/_ref/libsgrpo_ref.so, built
by ``make -C oracle``):

    python tests/golden/make_golden.py

Every value written here comes out of the compiled, unmodified reference through
oracle/ref_capi.cpp (never from our numpy oracle or the CUDA path). The fixtures are
small so they are committed; tests/test_oracle_pinning.py checks the numpy oracle
(oracle/oracle.py) against them on any machine, without /root/reference.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import refc as R  # noqa: E402
from oracle.oracle import ModelConfig  # noqa: E402  (plain config record only)

OUT = os.path.dirname(os.path.abspath(__file__))

TINY = ModelConfig(16, 32, 2, 4, 64, 32, 7)          # tests/test_util.hpp:21-31 shape
SMALL = ModelConfig(64, 64, 2, 4, 128, 48, 3)         # rollout / draft-update fixtures
C1 = ModelConfig(512, 256, 2, 4, 1024, 192, 1)        # BASELINE configs[0]


def cfgd(c):
    return dict(vocab_size=c.vocab_size, d_model=c.d_model, n_layers=c.n_layers, n_heads=c.n_heads,
                d_ff=c.d_ff, max_seq_len=c.max_seq_len, seed=c.seed)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rng_fixture():
    L = R.lib()
    out = {"splitmix": {}, "mix_key": [], "uniform": {}, "normal": {}, "below": {}}
    for seed in (0, 1, 42, 0xFFFFFFFFFFFFFFFF):
        st = C.c_ulonglong(seed)
        v = (C.c_ulonglong * 6)()
        L.sgref_splitmix(C.byref(st), 6, v)
        out["splitmix"][str(seed)] = [str(x) for x in v]
        u = np.zeros(6)
        L.sgref_rng_uniforms(C.c_ulonglong(seed), 6, u.ctypes.data_as(C.POINTER(C.c_double)))
        out["uniform"][str(seed)] = u.tolist()
        nn = np.zeros(7)
        L.sgref_rng_normals(C.c_ulonglong(seed), 7, nn.ctypes.data_as(C.POINTER(C.c_double)))
        out["normal"][str(seed)] = nn.tolist()
        b = (C.c_ulonglong * 6)()
        L.sgref_rng_below(C.c_ulonglong(seed), C.c_ulonglong(510), 6, b)
        out["below"][str(seed)] = [int(x) for x in b]
    for a, b in [(0, 0), (7, 3), (1, 2), (123456789, 987654321), (2**63, 5)]:
        out["mix_key"].append([str(a), str(b), str(L.sgref_mix_key(a, b))])
    with open(os.path.join(OUT, "rng.json"), "w") as f:
        json.dump(out, f, indent=1)


def init_fixture():
    m = R.init_model(TINY)
    d1 = R.init_draft(TINY, 1)
    d2 = R.init_draft(TINY, 2)
    np.savez_compressed(os.path.join(OUT, "init_tiny.npz"), model=m, draft1=d1, draft2=d2)
    hashes = {"tiny": cfgd(TINY), "c1": cfgd(C1),
              "c1_model_sha256": sha(R.init_model(C1)), "c1_draft_sha256": sha(R.init_draft(C1, 1)),
              "small": cfgd(SMALL), "small_model_sha256": sha(R.init_model(SMALL)),
              "small_draft_sha256": sha(R.init_draft(SMALL, 1))}
    with open(os.path.join(OUT, "init_hashes.json"), "w") as f:
        json.dump(hashes, f, indent=1)


def forward_fixture():
    """test_tinylm.cpp:83-157 shapes: full, cached incremental, tree-masked."""
    cfg = ModelConfig(16, 32, 2, 4, 64, 32, 23)
    m = R.RefModel(cfg)
    out = {}
    toks = [2, 9, 4, 13, 6, 3, 7, 12]
    out["full_logits"], out["full_hidden"] = R.forward_target(m, toks, list(range(8)))
    # tree over prefix (test_tinylm.cpp:119-157)
    cache = R.RefCache(cfg.n_layers, cfg.d_model)
    R.forward_target(m, [2, 7, 5], [0, 1, 2], None, cache)
    parent = [-1, 0, 0, 1]
    mask = np.zeros((4, 4), np.uint8)
    for i in range(4):
        j = i
        while j != -1:
            mask[i, j] = 1
            j = parent[j]
    out["tree_logits"], out["tree_hidden"] = R.forward_target(m, [4, 6, 8, 9], [3, 4, 4, 5], mask, cache)
    out["tree_mask"] = mask
    k, v = cache.get()
    out["tree_cache_k"], out["tree_cache_v"] = k, v
    # draft rows with cache (draft catch-up shape)
    dr = R.RefDraft(cfg, 1)
    dcache = R.RefCache(1, cfg.d_model)
    feats = np.random.default_rng(3).standard_normal((5, cfg.d_model)).astype(np.float32)
    out["draft_in_feats"] = feats
    out["draft_feats"], out["draft_logits"] = R.forward_draft_rows(dr, m, [3, 5, 7, 2, 9], feats, [1, 2, 3, 4, 5], dcache)
    np.savez_compressed(os.path.join(OUT, "forward_tiny.npz"), **out)
    with open(os.path.join(OUT, "forward_tiny.json"), "w") as f:
        json.dump({"config": cfgd(cfg), "tokens": toks}, f)


def _random_lps(rng, vocab):
    raw = 3.0 * rng.standard_normal(vocab)
    if rng.random() < 0.3:  # inject exact ties to exercise the tie-breaks
        raw[rng.integers(0, vocab, 3)] = raw.max()
    raw = raw - raw.max()
    return raw - np.log(np.exp(raw).sum())


def tree_fixture():
    rng = np.random.default_rng(11)
    cases = []
    for trial in range(30):
        vocab = int(rng.integers(4, 16))
        k = int(rng.integers(0, 6))
        l = int(rng.integers(0, 5))
        lps_by_call = []

        def fn(toks, pars, deps, node):
            lp = _random_lps(rng, vocab)
            lps_by_call.append(lp.tolist())
            return lp

        arrs = R.expand_tree_with(int(rng.integers(0, vocab)), k, l, vocab, fn)
        n = len(arrs[0])
        case = {"vocab": vocab, "k": k, "l": l, "root": int(arrs[0][0]), "calls": lps_by_call,
                "tok": arrs[0].tolist(), "par": arrs[1].tolist(), "dep": arrs[2].tolist(),
                "lp": arrs[3].tolist(), "conf": arrs[4].tolist(), "rerank": []}
        for nv in sorted({1, 2, 3, max(1, n // 2), n, n + 3}):
            sel, mask = R.rerank(arrs, nv)
            ns = len(sel)
            ent = {"n_verify": nv, "sel": sel.tolist(), "mask": mask.astype(int).tolist()}
            # verify with random logits, greedy and sampled, with ties on purpose
            d = 3
            logits = rng.standard_normal((ns, vocab)).astype(np.float32)
            if ns > 1 and vocab > 2:
                # steer some rows to the token of a selected child so walks go deep
                for i in range(ns):
                    kids = [j for j in range(ns) if arrs[1][sel[j]] == sel[i]]
                    if kids and rng.random() < 0.7:
                        logits[i, arrs[0][sel[kids[int(rng.integers(0, len(kids)))]]]] += 6.0
                logits[0, :2] = logits[0].max() + 1.0  # exact tie at the root row
            hidden = rng.standard_normal((ns, d)).astype(np.float32)
            ent["logits"] = logits.tolist()
            ent["verify"] = []
            for temp, seed, root_pos in [(0.0, 5, 3), (1.0, 9, 7), (0.6, 123, 11)]:
                at, al, bonus, rows = R.verify(arrs, sel, logits, hidden, vocab, d, temp, seed, root_pos)
                ent["verify"].append({"temp": temp, "seed": seed, "root_pos": root_pos, "tokens": at,
                                      "len": al, "bonus": bonus, "rows": rows})
            case["rerank"].append(ent)
        cases.append(case)
    with open(os.path.join(OUT, "trees.json"), "w") as f:
        json.dump(cases, f)


def plan_fixture():
    rng = np.random.default_rng(5)
    rows = []
    for _ in range(1000):
        c = int(rng.integers(1, 700))
        b = int(rng.integers(1, 600))
        alpha = float(rng.choice([0.5, 1.0, 2.0, 3.0, 4.0]))
        km = int(rng.integers(0, 12))
        lm = int(rng.integers(0, 8))
        try:
            r = R.plan_step(c, b, alpha, km, lm)
            rows.append([c, b, alpha, km, lm, *r])
        except ValueError:
            rows.append([c, b, alpha, km, lm, -1, -1, -1])
    with open(os.path.join(OUT, "plan_step.json"), "w") as f:
        json.dump(rows, f)


def generate_fixture():
    cfg = SMALL
    m = R.RefModel(cfg)
    dr = R.RefDraft(cfg, 1)
    rng = np.random.default_rng(0)
    prompts = [rng.integers(2, cfg.vocab_size, size=int(rng.integers(3, 9))).tolist() for _ in range(3)]
    runs = []
    for mode, temp, et in [("vanilla", 0.0, True), ("adaptive_spec", 0.0, True), ("adaptive_spec", 1.0, True),
                           ("fixed_spec", 0.7, True), ("adaptive_spec", 0.0, False)]:
        kw = dict(c_peak=16, alpha=2.0, k_max=5, l_max=3, mode=mode, temperature=temp, seed=7,
                  max_new_tokens=20, early_term=et, fixed=(4, 3, 2))
        out = R.generate(m, dr, prompts, 2, **kw)
        runs.append({"kw": kw, "tokens": out["tokens"], "prompt_len": out["prompt_len"],
                     "hit_eos": out["hit_eos"], "steps": out["steps"], "total_accepted": out["total_accepted"],
                     "total_verify_slots": out["total_verify_slots"],
                     "feat_sum": [float(np.float64(f).sum()) for f in out["features"]]})
    with open(os.path.join(OUT, "generate_small.json"), "w") as f:
        json.dump({"config": cfgd(cfg), "prompts": prompts, "g": 2, "runs": runs}, f)
    # draft update on the vanilla rollout
    out = R.generate(m, dr, prompts, 2, c_peak=16, mode="vanilla", seed=7, max_new_tokens=20)

    class S:
        pass
    seqs = []
    for t, fe in zip(out["tokens"], out["features"]):
        s = S()
        s.tokens, s.features = t, fe
        seqs.append(s)
    grad, terms = R.draft_loss_grad(dr, m, seqs)
    before = dr.flat()
    R.draft_update(dr, m, seqs, lr=1e-3)
    after = dr.flat()
    np.savez_compressed(os.path.join(OUT, "draft_update_small.npz"), grad=grad, terms=np.array(terms),
                        before=before, after=after,
                        tokens=np.concatenate([np.asarray(t, np.int32) for t in out["tokens"]]),
                        lens=np.array([len(t) for t in out["tokens"]], np.int32),
                        features=np.concatenate([f.reshape(-1) for f in out["features"]]))


def c1_fixture():
    """BASELINE configs[0] shape, 2 queries x G=2, 24 new tokens (vanilla + adaptive)."""
    cfg = C1
    m = R.RefModel(cfg)
    dr = R.RefDraft(cfg, 1)
    prompts = []
    from oracle.oracle import Rng, mix_key
    r = Rng(mix_key(0, 0x9A01))
    for _ in range(2):
        prompts.append([int(r.below(cfg.vocab_size - 2) + 2) for _ in range(32)])
    runs = []
    for mode in ("vanilla", "adaptive_spec"):
        kw = dict(c_peak=64, mode=mode, temperature=0.0, seed=7, max_new_tokens=24)
        out = R.generate(m, dr, prompts, 2, **kw)
        runs.append({"kw": kw, "tokens": out["tokens"], "steps": out["steps"],
                     "total_accepted": out["total_accepted"], "total_verify_slots": out["total_verify_slots"]})
    with open(os.path.join(OUT, "generate_c1.json"), "w") as f:
        json.dump({"config": cfgd(cfg), "prompts": prompts, "g": 2, "runs": runs}, f)


CKPT = ModelConfig(64, 64, 1, 1, 128, 32, 5)  # head dim 64: loadable by the GPU engine too


def checkpoint_fixture():
    """SGRPOCK1 files written by the reference itself (tinylm.cpp:73-105): a target and a
    1-layer draft with the reference init weights (a perturbed draft, so it is not the init)."""
    m = R.RefModel(CKPT)
    d0 = R.init_draft(CKPT, 1)
    d = R.RefDraft(CKPT, 1, d0 + np.float32(0.001) * np.arange(d0.size, dtype=np.float32) % np.float32(0.01))
    R.check(R.lib().sgref_save_checkpoint(C.c_void_p(m.h), os.path.join(OUT, "ckpt_target.bin").encode()))
    R.check(R.lib().sgref_save_draft_checkpoint(C.c_void_p(d.h), os.path.join(OUT, "ckpt_draft.bin").encode()))
    with open(os.path.join(OUT, "ckpt.json"), "w") as f:
        json.dump({"config": cfgd(CKPT), "draft_layers": 1}, f)


if __name__ == "__main__":
    if not R.available():
        sys.exit("build oracle/_ref first: make -C oracle")
    rng_fixture()
    init_fixture()
    forward_fixture()
    tree_fixture()
    plan_fixture()
    generate_fixture()
    c1_fixture()
    checkpoint_fixture()
    print("golden fixtures written to", OUT)
