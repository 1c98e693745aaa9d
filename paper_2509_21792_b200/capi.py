"""ctypes binding of libsgrpo_b200.so (include/sgrpo_b200.h).

Host-side mirror of the reference's operator API for the rollout path: the same
names (forward_target, forward_draft_rows, sample_token, expand/rerank/verify,
generate_dynamic_batch), argument meaning and error behaviour -- C-ABI status codes are
re-raised as the Python equivalents of the reference's exception types:
  invalid_argument -> ValueError, out_of_range -> IndexError,
  runtime_error -> RuntimeError, domain_error -> ArithmeticError.
There is no CPU fallback: if the shared library is missing this module raises at import.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGB_LIB") or os.path.join(HERE, "libsgrpo_b200.so")  # SGB_LIB: A/B kernel variants

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2509_21792_b200.build` "
                      "(there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)
DEV_LIB_PATH = os.path.join(HERE, "libsgrpo_b200_dev.so")
_dev_lib = None


def _dev():
    """The test-only library (kernel self-tests, microbenchmarks), loaded on first use."""
    global _dev_lib
    if _dev_lib is None:
        if not os.path.exists(DEV_LIB_PATH):
            raise ImportError(f"{DEV_LIB_PATH} is missing: build it with `python -m paper_2509_21792_b200.build`")
        _dev_lib = C.CDLL(DEV_LIB_PATH)
        _dev_lib.sgb_dev_last_error.restype = C.c_char_p
    return _dev_lib


@dataclass
class ModelConfig:
    """ModelConfig (include/sgrpo/tinylm.hpp:16-37), as the engine needs it."""
    vocab_size: int
    d_model: int
    n_layers: int
    n_heads: int
    d_ff: int
    max_seq_len: int
    seed: int = 0


_M64 = (1 << 64) - 1


def _splitmix64(state: int):
    state = (state + 0x9E3779B97F4A7C15) & _M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def mix_key(a: int, b: int) -> int:
    """mix_key (include/sgrpo/rng.hpp:17-20): the keyed-stream combiner the engine derives
    sequence seeds and emission keys with (host integer work, no compute)."""
    s = (a ^ ((b + 0x9E3779B97F4A7C15 + ((a << 6) & _M64) + (a >> 2)) & _M64)) & _M64
    return _splitmix64(s)


class ModelConfigC(C.Structure):
    _fields_ = [("vocab_size", C.c_int), ("d_model", C.c_int), ("n_layers", C.c_int), ("n_heads", C.c_int),
                ("d_ff", C.c_int), ("max_seq_len", C.c_int), ("seed", C.c_ulonglong)]


class GenOptionsC(C.Structure):
    _fields_ = [("alpha", C.c_double), ("k_max", C.c_int), ("l_max", C.c_int), ("c_peak", C.c_int),
                ("mode", C.c_int), ("early_term", C.c_int), ("temperature", C.c_double), ("seed", C.c_ulonglong),
                ("max_new_tokens", C.c_int), ("fixed_n_verify", C.c_int), ("fixed_k_draft", C.c_int),
                ("fixed_l_draft", C.c_int), ("seq_max_new", C.POINTER(C.c_int)), ("want_features", C.c_int),
                ("sid_offset", C.c_int), ("step_seconds", C.POINTER(C.c_double)), ("acceptance", C.c_int)]

ACCEPTANCE = {"strict": 0, "rejection": 1}


class RolloutStatsC(C.Structure):
    _fields_ = [("total_accepted", C.c_longlong), ("total_verify_slots", C.c_longlong), ("n_steps", C.c_int),
                ("target_forwards", C.c_longlong), ("draft_forwards", C.c_longlong),
                ("kernel_launches", C.c_longlong), ("seconds", C.c_double), ("h2d_bytes", C.c_longlong),
                ("d2h_bytes", C.c_longlong), ("host_gap_seconds", C.c_double), ("host_enqueue_seconds", C.c_double)]


LOGITS_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                        C.c_int, C.POINTER(C.c_float))

_lib.sgb_last_error.restype = C.c_char_p
_lib.sgb_engine_create.argtypes = [C.POINTER(ModelConfigC), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_void_p)]
_lib.sgb_engine_destroy.argtypes = [C.c_void_p]

EXPORTED = ["sgb_last_error", "sgb_version", "sgb_device_count", "sgb_engine_create", "sgb_engine_destroy",
            "sgb_param_counts", "sgb_upload_target", "sgb_upload_draft", "sgb_download_draft", "sgb_init_random",
            "sgb_cache_reset", "sgb_cache_len", "sgb_cache_read", "sgb_cache_gather_tail", "sgb_forward_target",
            "sgb_forward_draft_rows", "sgb_sample_rows", "sgb_topk_logsoftmax", "sgb_build_tree", "sgb_rollout",
            "sgb_profile_enable", "sgb_profile_read", "sgb_group_advantages", "sgb_target_forward_calls",
            "sgb_allgather_f64", "sgb_detect_knee", "sgb_measure_c_peak"]
# test-only self-tests / microbenchmarks of libsgrpo_b200_dev.so (include/sgrpo_b200_dev.h)
DEV_EXPORTED = ["sgb_dev_last_error", "sgb_debug_group_advantages", "sgb_bench_gemm", "sgb_bench_attention",
                "sgb_debug_attention", "sgb_debug_tree_attention", "sgb_debug_tree_attention_tree",
                "sgb_bench_tree_attention_tree", "sgb_debug_attention_decode", "sgb_bench_attention_decode",
                "sgb_bench_overlap", "sgb_bench_tree_attention", "sgb_debug_gemm"]

KERNEL_CLASSES = ["gemm_tcgen05", "attention", "rowops", "lm_head", "sample", "tree", "kv_commit"]

_EXC = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: ArithmeticError, 5: RuntimeError}


def _check(rc: int):
    if rc != 0:
        raise _EXC.get(rc, RuntimeError)(_lib.sgb_last_error().decode())


def _check_dev(rc: int):
    if rc != 0:
        raise _EXC.get(rc, RuntimeError)(_dev().sgb_dev_last_error().decode())


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def lib():
    return _lib


def dev_lib():
    return _dev()


def device_count() -> int:
    n = C.c_int()
    _check(_lib.sgb_device_count(C.byref(n)))
    return n.value


def debug_attention(q: np.ndarray, k_rows, v_rows, n_heads: int) -> np.ndarray:
    """Tree/paged attention self-test: q [B][d]; k_rows/v_rows: per row an [n_keys][d]
    array (the last key goes through the tree-path slot list). Returns [B][d] (bf16 values)."""
    q = np.ascontiguousarray(q, np.float32)
    B, d = q.shape
    nk = np.array([len(k) for k in k_rows], np.int32)
    k = np.ascontiguousarray(np.concatenate(k_rows), np.float32)
    v = np.ascontiguousarray(np.concatenate(v_rows), np.float32)
    out = np.zeros((B, d), np.float32)
    _check_dev(_dev().sgb_debug_attention(B, _p(nk, C.c_int), n_heads, d // n_heads, _p(q, C.c_float), _p(k, C.c_float),
                                    _p(v, C.c_float), _p(out, C.c_float)))
    return out


def debug_tree_attention(ctx_len, parents, q, kctx, vctx, knode, vnode, n_heads: int):
    """Prefix-shared tree attention self-test (sgb_debug_tree_attention): per group g,
    ctx_len[g] committed keys and a tree of rows (parents[g], level order, -1 = root).
    Returns (per-row kernel output, group kernel output), each [rows][d] (bf16 values)."""
    q = np.ascontiguousarray(q, np.float32)
    M, d = q.shape
    cl = np.ascontiguousarray(ctx_len, np.int32)
    nr = np.array([len(p) for p in parents], np.int32)
    par = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in parents]), np.int32)
    f = [np.ascontiguousarray(a, np.float32) for a in (kctx, vctx, knode, vnode)]
    o1 = np.zeros((M, d), np.float32)
    o2 = np.zeros((M, d), np.float32)
    _check_dev(_dev().sgb_debug_tree_attention(len(cl), _p(cl, C.c_int), _p(nr, C.c_int), _p(par, C.c_int), n_heads,
                                         d // n_heads, _p(q, C.c_float), *[_p(a, C.c_float) for a in f],
                                         _p(o1, C.c_float), _p(o2, C.c_float)))
    return o1, o2


def debug_group_advantages(tokens, prompt_lens, answers, g: int, eps_var: float = 1e-8):
    """Device rewards + standardized advantages on host token lists (sgb_debug_group_advantages).
    tokens: n_groups*g full sequences; answers: per group a+b. Returns (rewards, adv, valid)."""
    n = len(tokens)
    ng = n // g
    stride = max(1, max(len(t) for t in tokens))
    tab = np.zeros((n, stride), np.int32)
    for i, t in enumerate(tokens):
        tab[i, :len(t)] = t
    lens = np.array([len(t) for t in tokens], np.int32)
    pl = np.ascontiguousarray(prompt_lens, np.int32)
    ans = np.ascontiguousarray(answers, np.int64)
    r = np.zeros(n, np.float64)
    a = np.zeros(n, np.float64)
    v = np.zeros(ng, np.int32)
    _check_dev(_dev().sgb_debug_group_advantages(_p(tab, C.c_int), _p(lens, C.c_int), _p(pl, C.c_int), ng, g, stride,
                                           _p(ans, C.c_longlong), C.c_double(eps_var), _p(r, C.c_double),
                                           _p(a, C.c_double), _p(v, C.c_int)))
    return r, a, v


def debug_gemm(w: np.ndarray, x: np.ndarray, splits: int = 0):
    """out = bf16(x) @ bf16(w).T via the tcgen05 GEMM (optionally forcing the K split);
    returns (out, the split count the auto policy picks)."""
    w = np.ascontiguousarray(w, np.float32)
    x = np.ascontiguousarray(x, np.float32)
    N, K = w.shape
    M = x.shape[0]
    out = np.zeros((M, N), np.float32)
    sp = C.c_int(splits)
    _check_dev(_dev().sgb_debug_gemm(_p(w, C.c_float), _p(x, C.c_float), M, N, K, _p(out, C.c_float), C.byref(sp)))
    return out, sp.value


MODES = {"vanilla": 0, "fixed_spec": 1, "adaptive_spec": 2}


@dataclass
class Rollout:
    """BatchState (scheduler.hpp:91-94) + measurements."""
    tokens: List[List[int]]
    prompt_len: List[int]
    hit_eos: List[bool]
    features: Optional[List[np.ndarray]]
    steps: List[tuple]  # (b_cur, n_verify, k_draft, l_draft, accepted)
    total_accepted: int
    total_verify_slots: int
    target_forwards: int
    draft_forwards: int
    kernel_launches: int
    seconds: float
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    step_seconds: Optional[List[float]] = None  # measured device seconds per decode step
    host_gap_seconds: float = 0.0  # device idle between steps (host planning + launch latency)
    host_enqueue_seconds: float = 0.0  # host wall time issuing the steps

    def tau(self) -> float:
        if self.total_verify_slots == 0:
            raise ArithmeticError("tau: no verification steps logged")
        return self.total_accepted / self.total_verify_slots

    def generated(self) -> int:
        return sum(len(t) - p for t, p in zip(self.tokens, self.prompt_len))


class Engine:
    """One GPU's rollout engine (sgb_engine)."""

    def __init__(self, cfg, draft_layers: int = 1, device: int = 0, max_seqs: int = 64, max_rows: int = 512,
                 k_max: int = 10, l_max: int = 6):
        self.cfg = cfg
        c = ModelConfigC(cfg.vocab_size, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.max_seq_len,
                         getattr(cfg, "seed", 0))
        h = C.c_void_p()
        _check(_lib.sgb_engine_create(C.byref(c), draft_layers, device, max_seqs, max_rows, k_max, l_max,
                                      C.byref(h)))
        self.h = h
        t, d = C.c_size_t(), C.c_size_t()
        _check(_lib.sgb_param_counts(self.h, C.byref(t), C.byref(d)))
        self.n_target, self.n_draft = t.value, d.value

    def close(self):
        if getattr(self, "h", None):
            _lib.sgb_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- weights
    def upload_target(self, flat):
        f = np.ascontiguousarray(flat, np.float32)
        _check(_lib.sgb_upload_target(self.h, _p(f, C.c_float), C.c_size_t(f.size)))

    def upload_draft(self, flat):
        f = np.ascontiguousarray(flat, np.float32)
        _check(_lib.sgb_upload_draft(self.h, _p(f, C.c_float), C.c_size_t(f.size)))

    def download_draft(self) -> np.ndarray:
        out = np.zeros(self.n_draft, np.float32)
        _check(_lib.sgb_download_draft(self.h, _p(out, C.c_float), C.c_size_t(out.size)))
        return out

    def init_random(self, seed: int):
        _check(_lib.sgb_init_random(self.h, C.c_ulonglong(seed)))

    # ---- per-op parity entry points
    def cache_reset(self, slot: int, draft: bool = False):
        _check(_lib.sgb_cache_reset(self.h, slot, int(draft)))

    def cache_len(self, slot: int, draft: bool = False) -> int:
        n = C.c_int()
        _check(_lib.sgb_cache_len(self.h, slot, int(draft), C.byref(n)))
        return n.value

    def cache_read(self, slot: int, draft: bool = False):
        n = self.cache_len(slot, draft)
        L = self.cfg.n_layers if not draft else self.draft_layers
        k = np.zeros((L, n, self.cfg.d_model), np.float32)
        v = np.zeros_like(k)
        _check(_lib.sgb_cache_read(self.h, slot, int(draft), _p(k, C.c_float), _p(v, C.c_float)))
        return k, v

    draft_layers = 1

    def cache_gather_tail(self, slot: int, base: int, keep: Sequence[int]):
        kp = np.ascontiguousarray(keep, np.int32)
        _check(_lib.sgb_cache_gather_tail(self.h, slot, base, _p(kp, C.c_int), kp.size))

    def forward_target(self, slot: int, tokens, positions, mask=None):
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int32)
        n = t.size
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8).reshape(-1)
        logits = np.zeros((n, self.cfg.vocab_size), np.float32)
        hidden = np.zeros((n, self.cfg.d_model), np.float32)
        _check(_lib.sgb_forward_target(self.h, slot, _p(t, C.c_int), _p(p, C.c_int), n, _p(m, C.c_ubyte),
                                       _p(logits, C.c_float), _p(hidden, C.c_float)))
        return logits, hidden

    def forward_draft_rows(self, slot: int, tokens, prev_features, positions, extend_cache=True):
        t = np.ascontiguousarray(tokens, np.int32)
        p = np.ascontiguousarray(positions, np.int32)
        f = np.ascontiguousarray(prev_features, np.float32)
        n = t.size
        feats = np.zeros((n, self.cfg.d_model), np.float32)
        logits = np.zeros((n, self.cfg.vocab_size), np.float32)
        _check(_lib.sgb_forward_draft_rows(self.h, slot, _p(t, C.c_int), _p(f, C.c_float), _p(p, C.c_int), n,
                                           int(extend_cache), _p(feats, C.c_float), _p(logits, C.c_float)))
        return feats, logits

    def sample_rows(self, logits, temperature: float, seeds, key_pos):
        lg = np.ascontiguousarray(logits, np.float32)
        rows, V = lg.shape
        s = np.ascontiguousarray(seeds, np.uint64)
        kp = np.ascontiguousarray(key_pos, np.int32)
        out = np.zeros(rows, np.int32)
        _check(_lib.sgb_sample_rows(self.h, _p(lg, C.c_float), rows, V, C.c_double(temperature),
                                    _p(s, C.c_ulonglong), _p(kp, C.c_int), _p(out, C.c_int)))
        return out

    def topk_logsoftmax(self, logits, k: int):
        lg = np.ascontiguousarray(logits, np.float32)
        rows, V = lg.shape
        kk = min(k, V)
        tok = np.zeros((rows, kk), np.int32)
        lp = np.zeros((rows, kk), np.float64)
        _check(_lib.sgb_topk_logsoftmax(self.h, _p(lg, C.c_float), rows, V, k, _p(tok, C.c_int),
                                        _p(lp, C.c_double)))
        return tok, lp

    def build_tree(self, root_token: int, k: int, l: int, n_verify: int, logits_fn, cap: int = 1024):
        """logits_fn(node_ids, node_tok, node_par) -> [len(node_ids)][V] draft logits."""
        V = self.cfg.vocab_size

        def cb(ctx, n_front, ids, tok, par, n_nodes, out):
            nid = [ids[i] for i in range(n_front)]
            tk = [tok[i] for i in range(n_nodes)]
            pr = [par[i] for i in range(n_nodes)]
            lg = np.ascontiguousarray(logits_fn(nid, tk, pr), np.float32).reshape(-1)
            C.memmove(out, lg.ctypes.data, lg.nbytes)

        cbf = LOGITS_FN(cb)
        tok = np.zeros(cap, np.int32)
        par = np.zeros(cap, np.int32)
        dep = np.zeros(cap, np.int32)
        lp = np.zeros(cap, np.float64)
        conf = np.zeros(cap, np.float64)
        sel = np.zeros(cap, np.int32)
        mask = np.zeros(cap * cap, np.uint8)
        nn, ns = C.c_int(), C.c_int()
        _check(_lib.sgb_build_tree(self.h, root_token, k, l, n_verify, cbf, None, cap, _p(tok, C.c_int),
                                   _p(par, C.c_int), _p(dep, C.c_int), _p(lp, C.c_double), _p(conf, C.c_double),
                                   C.byref(nn), _p(sel, C.c_int), C.byref(ns), _p(mask, C.c_ubyte)))
        n, s = nn.value, ns.value
        return dict(tok=tok[:n], par=par[:n], dep=dep[:n], lp=lp[:n], conf=conf[:n], sel=sel[:s],
                    mask=mask[:s * s].reshape(s, s))

    # ---- the hot path: generate_dynamic_batch
    def generate(self, prompts: Sequence[Sequence[int]], g: int, c_peak: int, alpha: float = 2.0,
                 k_max: int = 10, l_max: int = 6, mode: str = "vanilla", early_term: bool = True,
                 temperature: float = 0.0, seed: int = 0, max_new_tokens: int = 0, fixed=(1, 0, 0),
                 seq_max_new: Optional[Sequence[int]] = None, want_features: bool = True,
                 max_steps_record: int = 1 << 16, sid_offset: int = 0, acceptance: str = "strict") -> Rollout:
        """generate_dynamic_batch. acceptance: "strict" = the reference's keyed strict-match verify
        (drafttree.cpp:170-222), "rejection" = speculative rejection sampling (T > 0, reject.cu)."""
        T, d = self.cfg.max_seq_len, self.cfg.d_model
        n_p = len(prompts)
        ns = n_p * g
        plens = np.array([len(p) for p in prompts], np.int32)
        flat = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts])
                                    if n_p else np.zeros(0, np.int32), np.int32)
        smn = None if seq_max_new is None else np.ascontiguousarray(seq_max_new, np.int32)
        step_s = np.zeros(max_steps_record, np.float64)
        opt = GenOptionsC(alpha, k_max, l_max, c_peak, MODES[mode], int(early_term), temperature, seed,
                          max_new_tokens, fixed[0], fixed[1], fixed[2], _p(smn, C.c_int), int(want_features),
                          sid_offset, _p(step_s, C.c_double), ACCEPTANCE[acceptance])
        toks = np.zeros((max(ns, 1), T), np.int32)
        lens = np.zeros(max(ns, 1), np.int32)
        pl = np.zeros(max(ns, 1), np.int32)
        eos = np.zeros(max(ns, 1), np.int32)
        feats = np.zeros((max(ns, 1), T - 1, d), np.float32) if want_features else None
        rec = np.zeros(5 * max_steps_record, np.int32)
        st = RolloutStatsC()
        _check(_lib.sgb_rollout(self.h, _p(flat, C.c_int), _p(plens, C.c_int), n_p, g, C.byref(opt),
                                _p(toks, C.c_int), _p(lens, C.c_int), _p(pl, C.c_int), _p(eos, C.c_int),
                                _p(feats, C.c_float), _p(rec, C.c_int), max_steps_record, C.byref(st)))
        nst = min(st.n_steps, max_steps_record)
        return Rollout(
            tokens=[toks[i, :lens[i]].tolist() for i in range(ns)], prompt_len=pl[:ns].tolist(),
            hit_eos=[bool(x) for x in eos[:ns]],
            features=[feats[i, :lens[i] - 1] for i in range(ns)] if want_features else None,
            steps=[tuple(int(x) for x in rec[5 * i:5 * i + 5]) for i in range(nst)],
            total_accepted=st.total_accepted, total_verify_slots=st.total_verify_slots,
            target_forwards=st.target_forwards, draft_forwards=st.draft_forwards,
            kernel_launches=st.kernel_launches, seconds=st.seconds, h2d_bytes=st.h2d_bytes,
            d2h_bytes=st.d2h_bytes, step_seconds=step_s[:nst].tolist(), host_gap_seconds=st.host_gap_seconds,
            host_enqueue_seconds=st.host_enqueue_seconds)

    # ---- kernel-class profiler
    def profile(self, on: bool = True):
        _check(_lib.sgb_profile_enable(self.h, int(on)))

    def read_profile(self, reset: bool = True) -> dict:
        n = len(KERNEL_CLASSES)
        ms, by, fl = np.zeros(n), np.zeros(n), np.zeros(n)
        la = np.zeros(n, np.int64)
        _check(_lib.sgb_profile_read(self.h, n, _p(ms, C.c_double), _p(by, C.c_double), _p(fl, C.c_double),
                                     _p(la, C.c_longlong), int(reset)))
        return {k: dict(ms=float(ms[i]), bytes=float(by[i]), flops=float(fl[i]), launches=int(la[i]))
                for i, k in enumerate(KERNEL_CLASSES)}


class AdamWC(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("w_feat", C.c_double), ("w_tok", C.c_double),
                ("rows_total", C.c_longlong), ("apply_step", C.c_int), ("allreduce_grad", C.c_int)]


class DraftTermsC(C.Structure):
    _fields_ = [("feature_loss", C.c_double), ("token_loss", C.c_double), ("total", C.c_double),
                ("rows", C.c_longlong), ("seconds", C.c_double)]


def _draft_update(self, seqs=None, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, w_feat=1.0,
                  w_tok=0.1, rows_total=0, apply_step=True, want_grad=False, allreduce_grad=False):
    """draft_update (grpo.cpp:177-186). seqs: list of (tokens, features[(len-1), d]) or None for
    the engine's last rollout (read from HBM). rows_total: global row normaliser of a data-parallel
    shard (grpo.hpp:286-290); allreduce_grad: NCCL sum of the gradient over the DP group (C1).
    Returns (feature_loss, token_loss, total, rows, seconds) and the fp32 gradient (reference flat
    layout) if want_grad."""
    opt = AdamWC(lr, beta1, beta2, eps, weight_decay, w_feat, w_tok, rows_total, int(apply_step),
                 int(allreduce_grad))
    terms = DraftTermsC()
    grad = np.zeros(self.n_draft, np.float32) if want_grad else None
    if seqs is None:
        _check(_lib.sgb_draft_update_last(self.h, C.byref(opt), _p(grad, C.c_float), C.byref(terms)))
    else:
        toks = np.ascontiguousarray(np.concatenate([np.asarray(t, np.int32) for t, _ in seqs]), np.int32)
        lens = np.array([len(t) for t, _ in seqs], np.int32)
        feats = np.ascontiguousarray(np.concatenate([np.asarray(f, np.float32).reshape(-1) for _, f in seqs]),
                                     np.float32)
        _check(_lib.sgb_draft_update(self.h, len(seqs), _p(toks, C.c_int), _p(lens, C.c_int), _p(feats, C.c_float),
                                     C.byref(opt), _p(grad, C.c_float), C.byref(terms)))
    return (terms.feature_loss, terms.token_loss, terms.total, terms.rows, terms.seconds), grad


def _adamw_reset(self):
    _check(_lib.sgb_adamw_reset(self.h))


Engine.draft_update = _draft_update
Engine.adamw_reset = _adamw_reset
EXPORTED += ["sgb_draft_update", "sgb_draft_update_last", "sgb_adamw_reset"]


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(_lib.sgb_nccl_unique_id(buf))
    return bytes(buf)


def _nccl_init(self, rank: int, world: int, uid: bytes):
    buf = (C.c_ubyte * 128).from_buffer_copy(uid)
    _check(_lib.sgb_nccl_init(self.h, rank, world, buf))


def _group_advantages(self, answers, g: int, eps_var: float = 1e-8):
    """rewards / advantages / valid of the last rollout's groups (sgb_group_advantages)."""
    ans = np.ascontiguousarray(answers, np.int64)
    ng = ans.size
    r = np.zeros(ng * g, np.float64)
    a = np.zeros(ng * g, np.float64)
    v = np.zeros(ng, np.int32)
    _check(_lib.sgb_group_advantages(self.h, _p(ans, C.c_longlong), ng, g, C.c_double(eps_var), _p(r, C.c_double),
                                     _p(a, C.c_double), _p(v, C.c_int)))
    return r, a, v


def _target_forward_calls(self) -> int:
    n = C.c_longlong()
    _check(_lib.sgb_target_forward_calls(self.h, C.byref(n)))
    return n.value


def _allgather_f64(self, vals, world: int):
    s = np.ascontiguousarray(vals, np.float64)
    out = np.zeros(s.size * world, np.float64)
    _check(_lib.sgb_allgather_f64(self.h, _p(s, C.c_double), s.size, _p(out, C.c_double)))
    return out


def _allreduce_f64(self, vals):
    a = np.ascontiguousarray(vals, np.float64).copy()
    _check(_lib.sgb_allreduce_sum_f64(self.h, _p(a, C.c_double), a.size))
    return a


def _allreduce_i64(self, vals):
    a = np.ascontiguousarray(vals, np.int64).copy()
    _check(_lib.sgb_allreduce_sum_i64(self.h, _p(a, C.c_longlong), a.size))
    return a


Engine.nccl_init = _nccl_init
Engine.allreduce_f64 = _allreduce_f64
Engine.allreduce_i64 = _allreduce_i64
Engine.group_advantages = _group_advantages
Engine.target_forward_calls = _target_forward_calls
Engine.allgather_f64 = _allgather_f64
EXPORTED += ["sgb_nccl_unique_id", "sgb_nccl_init", "sgb_allreduce_sum_f64", "sgb_allreduce_sum_i64"]


def detect_knee(curve):
    """detect_knee (roofline.cpp:39-76) on [(b, seconds), ...] -> (index, confidence)."""
    b = np.ascontiguousarray([int(x) for x, _ in curve], np.int32)
    sec = np.ascontiguousarray([float(y) for _, y in curve], np.float64)
    idx, conf = C.c_int(), C.c_double()
    _check(_lib.sgb_detect_knee(_p(b, C.c_int), _p(sec, C.c_double), len(b), C.byref(idx), C.byref(conf)))
    return idx.value, conf.value


def _measure_c_peak(self, b_max: int, warmup: int = 1, reps: int = 3):
    """measure_c_peak (roofline.cpp:78-108) on this engine's device. Returns a dict in the
    reference's HardwareProfile JSON vocabulary (roofline.cpp:188-201)."""
    cp, conf, low = C.c_int(), C.c_double(), C.c_int()
    curve = np.zeros(b_max, np.float64)
    _check(_lib.sgb_measure_c_peak(self.h, b_max, warmup, reps, C.byref(cp), C.byref(conf), C.byref(low),
                                   _p(curve, C.c_double)))
    return dict(c_peak=cp.value, confidence=conf.value, low_confidence=bool(low.value),
                latency_curve=[[b + 1, float(curve[b])] for b in range(b_max)])


Engine.measure_c_peak = _measure_c_peak


def checkpoint_info(path: str) -> dict:
    """SGRPOCK1 header (src/tinylm.cpp:14-105) parsed by the library (host only)."""
    kind, dl, n = C.c_int(), C.c_int(), C.c_size_t()
    cfg = ModelConfigC()
    _check(_lib.sgb_checkpoint_info(path.encode(), C.byref(kind), C.byref(cfg), C.byref(dl), C.byref(n)))
    return dict(kind="target" if kind.value == 0 else "draft", vocab_size=cfg.vocab_size, d_model=cfg.d_model,
                n_layers=cfg.n_layers, n_heads=cfg.n_heads, d_ff=cfg.d_ff, max_seq_len=cfg.max_seq_len,
                seed=cfg.seed, draft_layers=dl.value, param_count=n.value)


def _load_checkpoint(self, path: str) -> str:
    kind = C.c_int()
    _check(_lib.sgb_load_checkpoint(self.h, path.encode(), C.byref(kind)))
    return "target" if kind.value == 0 else "draft"


def _save_draft_checkpoint(self, path: str):
    _check(_lib.sgb_save_draft_checkpoint(self.h, path.encode()))


Engine.load_checkpoint = _load_checkpoint
Engine.save_draft_checkpoint = _save_draft_checkpoint
EXPORTED += ["sgb_checkpoint_info", "sgb_load_checkpoint", "sgb_save_draft_checkpoint"]


def gen_stats_jsonl(r: "Rollout") -> str:
    """gen_stats_to_jsonl (scheduler.cpp:356-368) with MEASURED step seconds in sim_latency_s:
    one JSON object per decode step; accepted_total = tokens appended that step."""
    out = []
    for i, (b, n, k, l, acc) in enumerate(r.steps):
        sec = r.step_seconds[i] if r.step_seconds else 0.0
        out.append(json.dumps({"step": i, "b_cur": b, "spec_config": {"n_verify": n, "k_draft": k, "l_draft": l},
                               "accepted_total": acc, "sim_latency_s": sec}, separators=(",", ":")))
    return "".join(x + "\n" for x in out)


def _sample_rows_u(self, logits, temperature: float, uniforms):
    """sample_token with supplied uniforms (u = uniforms[i] * sum). Returns (tokens, exact_rows):
    exact_rows[i] = 1 where the draw was resolved by the exact sequential pass."""
    lg = np.ascontiguousarray(logits, np.float32)
    rows, V = lg.shape
    u = np.ascontiguousarray(uniforms, np.float64)
    out = np.zeros(rows, np.int32)
    ex = np.zeros(rows, np.int32)
    _check(_lib.sgb_sample_rows_u(self.h, _p(lg, C.c_float), rows, V, C.c_double(temperature), _p(u, C.c_double),
                                  _p(out, C.c_int), _p(ex, C.c_int)))
    return out, ex


def _exact_draws(self) -> int:
    n = C.c_ulonglong()
    _check(_lib.sgb_exact_draws(self.h, C.byref(n)))
    return n.value


def _debug_exp(self, x):
    xx = np.ascontiguousarray(x, np.float64)
    out = np.zeros_like(xx)
    _check(_lib.sgb_debug_exp(self.h, _p(xx, C.c_double), C.c_size_t(xx.size), _p(out, C.c_double)))
    return out


Engine.sample_rows_u = _sample_rows_u
Engine.exact_draws = _exact_draws
Engine.debug_exp = _debug_exp
EXPORTED += ["sgb_sample_rows_u", "sgb_exact_draws", "sgb_debug_exp"]


def _debug_spec_sample(self, p_logits, q_logits, k: int, temperature: float, n_trials: int, seed: int = 1):
    """n_trials rounds of ONE speculative-sampling node (reject.cu): k candidates drawn from
    softmax(q / T), the multi-round rejection against softmax(p / T). Returns (tokens, accepted)."""
    p = np.ascontiguousarray(p_logits, np.float32)
    q = np.ascontiguousarray(q_logits, np.float32)
    tok = np.zeros(n_trials, np.int32)
    acc = np.zeros(n_trials, np.int32)
    _check(_lib.sgb_debug_spec_sample(self.h, _p(p, C.c_float), _p(q, C.c_float), p.size, k, C.c_double(temperature),
                                      n_trials, C.c_ulonglong(seed), _p(tok, C.c_int), _p(acc, C.c_int)))
    return tok, acc


Engine.debug_spec_sample = _debug_spec_sample
EXPORTED += ["sgb_debug_spec_sample", "sgb_adamw_state", "sgb_rollout_events"]


def debug_tree_attention_tree(ctx_len, parents, q, kctx, vctx, knode, vnode, n_heads: int):
    """attention_tree.cu on the debug_tree_attention inputs: out [rows][d] (bf16 values)."""
    cl = np.ascontiguousarray(ctx_len, np.int32)
    nr = np.array([len(p) for p in parents], np.int32)
    par = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in parents]), np.int32)
    q = np.ascontiguousarray(q, np.float32)
    out = np.zeros_like(q)
    _check_dev(_dev().sgb_debug_tree_attention_tree(len(cl), _p(cl, C.c_int), _p(nr, C.c_int), _p(par, C.c_int), n_heads,
                                              q.shape[1] // n_heads, _p(q, C.c_float),
                                              _p(np.ascontiguousarray(kctx, np.float32), C.c_float),
                                              _p(np.ascontiguousarray(vctx, np.float32), C.c_float),
                                              _p(np.ascontiguousarray(knode, np.float32), C.c_float),
                                              _p(np.ascontiguousarray(vnode, np.float32), C.c_float),
                                              _p(out, C.c_float)))
    return out





def debug_attention_decode(ctx_len, q, kctx, vctx, knode, vnode, n_heads: int):
    """attention.cu and the cluster decode kernel on one-row groups: (out_row, out_decode)."""
    cl = np.ascontiguousarray(ctx_len, np.int32)
    q = np.ascontiguousarray(q, np.float32)
    o1, o2 = np.zeros_like(q), np.zeros_like(q)
    _check_dev(_dev().sgb_debug_attention_decode(len(cl), _p(cl, C.c_int), n_heads, q.shape[1] // n_heads, _p(q, C.c_float),
                                           _p(np.ascontiguousarray(kctx, np.float32), C.c_float),
                                           _p(np.ascontiguousarray(vctx, np.float32), C.c_float),
                                           _p(np.ascontiguousarray(knode, np.float32), C.c_float),
                                           _p(np.ascontiguousarray(vnode, np.float32), C.c_float),
                                           _p(o1, C.c_float), _p(o2, C.c_float)))
    return o1, o2


def bench_attention_decode(B: int, ctx: int, n_heads: int, dh: int = 128, iters: int = 20):
    """ms per launch: (attention.cu rows, tree kernel, cluster decode kernel)."""
    r, t, dd = C.c_double(), C.c_double(), C.c_double()
    _check_dev(_dev().sgb_bench_attention_decode(B, ctx, n_heads, dh, iters, C.byref(r), C.byref(t), C.byref(dd)))
    return r.value, t.value, dd.value





def bench_overlap(B: int, ctx: int, n_heads: int, dff: int, M: int, attn_cap: int, gemm_cap: int, dh: int = 128,
                  iters: int = 20):
    """ms per iteration: (attention alone, layer GEMMs alone, both on two streams)."""
    out = (C.c_double * 3)()
    _check_dev(_dev().sgb_bench_overlap(B, ctx, n_heads, dh, dff, M, attn_cap, gemm_cap, iters, out))
    return out[0], out[1], out[2]





class PolicyTermsC(C.Structure):
    _fields_ = [("loss", C.c_double), ("tokens", C.c_longlong), ("rows", C.c_longlong), ("seconds", C.c_double),
                ("skipped", C.c_int)]


def _policy_enable(self):
    """Keep the fp32 target master on the device from the next upload (policy updates)."""
    _check(_lib.sgb_policy_enable(self.h))


def _policy_update(self, seqs, lr=2e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, tokens_total=0,
                   apply_step=True, want_grad=False, allreduce_grad=False):
    """policy_update (grpo.cpp:163-175) on the device. seqs: list of (tokens, prompt_len, advantage).
    Returns (loss, tokens, rows, seconds, skipped) and the fp32 gradient if want_grad."""
    toks = np.ascontiguousarray(np.concatenate([np.asarray(t, np.int32) for t, _, _ in seqs]) if seqs
                                else np.zeros(0, np.int32), np.int32)
    lens = np.array([len(t) for t, _, _ in seqs], np.int32)
    pl = np.array([q for _, q, _ in seqs], np.int32)
    w = np.array([x for _, _, x in seqs], np.float64)
    opt = AdamWC(lr, beta1, beta2, eps, weight_decay, 1.0, 0.1, tokens_total, int(apply_step), int(allreduce_grad))
    grad = np.zeros(self.n_target, np.float32) if want_grad else None
    t = PolicyTermsC()
    _check(_lib.sgb_policy_update(self.h, len(seqs), _p(toks, C.c_int), _p(lens, C.c_int), _p(pl, C.c_int),
                                  _p(w, C.c_double), C.byref(opt), _p(grad, C.c_float), C.byref(t)))
    return (t.loss, t.tokens, t.rows, t.seconds, bool(t.skipped)), grad


def _download_target(self):
    out = np.zeros(self.n_target, np.float32)
    _check(_lib.sgb_download_target(self.h, _p(out, C.c_float), C.c_size_t(out.size)))
    return out


Engine.policy_enable = _policy_enable
Engine.policy_update = _policy_update
Engine.download_target = _download_target
EXPORTED += ["sgb_policy_enable", "sgb_policy_update", "sgb_download_target", "sgb_policy_adamw_state"]


def _rollout_roofline(self):
    """Per-step (algorithmic bytes, flops, measured seconds) of the last rollout."""
    n = C.c_longlong()
    _check(_lib.sgb_rollout_roofline(self.h, None, None, None, 0, C.byref(n)))
    b = np.zeros(n.value, np.float64)
    f = np.zeros(n.value, np.float64)
    s = np.zeros(n.value, np.float64)
    _check(_lib.sgb_rollout_roofline(self.h, _p(b, C.c_double), _p(f, C.c_double), _p(s, C.c_double), n.value,
                                     C.byref(n)))
    return b, f, s


Engine.rollout_roofline = _rollout_roofline
EXPORTED += ["sgb_rollout_roofline"]
