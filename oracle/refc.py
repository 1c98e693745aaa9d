"""ctypes binding of oracle/_ref/libsgrpo_ref.so (the compiled reference + ref_capi.cpp).

TEST INFRASTRUCTURE ONLY (checker / CPU baseline), see oracle/Makefile.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libsgrpo_ref.so")


class CfgC(C.Structure):
    _fields_ = [("vocab", C.c_int), ("d", C.c_int), ("layers", C.c_int), ("heads", C.c_int),
                ("dff", C.c_int), ("max_seq", C.c_int), ("seed", C.c_ulonglong)]


class GenArgs(C.Structure):
    _fields_ = [("alpha", C.c_double), ("k_max", C.c_int), ("l_max", C.c_int), ("c_peak", C.c_int),
                ("mode", C.c_int), ("early_term", C.c_int), ("temperature", C.c_double),
                ("seed", C.c_ulonglong), ("max_new_tokens", C.c_int), ("fixed_n", C.c_int),
                ("fixed_k", C.c_int), ("fixed_l", C.c_int)]


class AdamC(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("wd", C.c_double)]


LPS_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                     C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double))

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.sgref_last_error.restype = C.c_char_p
        _lib.sgref_mix_key.restype = C.c_ulonglong
        _lib.sgref_mix_key.argtypes = [C.c_ulonglong, C.c_ulonglong]
        _lib.sgref_param_count.restype = C.c_size_t
        _lib.sgref_draft_param_count.restype = C.c_size_t
        for n in ("sgref_model_new", "sgref_draft_new", "sgref_cache_new", "sgref_cache_clone",
                  "sgref_generate"):
            getattr(_lib, n).restype = C.c_void_p
        _lib.sgref_model_free.argtypes = [C.c_void_p]
        _lib.sgref_draft_free.argtypes = [C.c_void_p]
        _lib.sgref_cache_free.argtypes = [C.c_void_p]
        _lib.sgref_bs_free.argtypes = [C.c_void_p]
        _lib.sgref_cache_len.argtypes = [C.c_void_p]
        _lib.sgref_cache_clone.argtypes = [C.c_void_p]
        _lib.sgref_max_candidates.restype = C.c_longlong
        _lib.sgref_generate_threaded.restype = C.c_longlong
        _lib.sgref_target_forward_calls.restype = C.c_ulonglong
        _lib.sgref_adamw_new.restype = C.c_void_p
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def check(rc):
    if rc != 0:
        msg = lib().sgref_last_error().decode()
        exc = {1: ValueError, 2: IndexError, 3: RuntimeError, 4: ArithmeticError}.get(rc, RuntimeError)
        raise exc(msg)


def cfg_c(cfg) -> CfgC:
    return CfgC(cfg.vocab_size, cfg.d_model, cfg.n_layers, cfg.n_heads, cfg.d_ff, cfg.max_seq_len, cfg.seed)


def init_model(cfg) -> np.ndarray:
    c = cfg_c(cfg)
    out = np.zeros(lib().sgref_param_count(C.byref(c)), np.float32)
    check(lib().sgref_init_model(C.byref(c), _p(out, C.c_float)))
    return out


def init_draft(cfg, layers=1) -> np.ndarray:
    c = cfg_c(cfg)
    out = np.zeros(lib().sgref_draft_param_count(C.byref(c), layers), np.float32)
    check(lib().sgref_init_draft(C.byref(c), layers, _p(out, C.c_float)))
    return out


class RefModel:
    def __init__(self, cfg, flat: Optional[np.ndarray] = None):
        self.cfg = cfg
        c = cfg_c(cfg)
        f = None if flat is None else np.ascontiguousarray(flat, np.float32)
        self.h = lib().sgref_model_new(C.byref(c), _p(f, C.c_float))

    def __del__(self):
        if getattr(self, "h", None):
            lib().sgref_model_free(self.h)


class RefDraft:
    def __init__(self, cfg, layers=1, flat: Optional[np.ndarray] = None):
        self.cfg, self.layers = cfg, layers
        c = cfg_c(cfg)
        f = None if flat is None else np.ascontiguousarray(flat, np.float32)
        self.h = lib().sgref_draft_new(C.byref(c), layers, _p(f, C.c_float))
        self.n = lib().sgref_draft_param_count(C.byref(c), layers)

    def flat(self) -> np.ndarray:
        out = np.zeros(self.n, np.float32)
        lib().sgref_draft_get(C.c_void_p(self.h), _p(out, C.c_float))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().sgref_draft_free(self.h)


class RefCache:
    def __init__(self, layers, d, h=None):
        self.layers, self.d = layers, d
        self.h = h if h is not None else lib().sgref_cache_new(layers, d)

    def clone(self):
        return RefCache(self.layers, self.d, lib().sgref_cache_clone(self.h))

    @property
    def len(self):
        return lib().sgref_cache_len(self.h)

    def get(self):
        n = self.len
        k = np.zeros((self.layers, n, self.d), np.float32)
        v = np.zeros_like(k)
        lib().sgref_cache_get(C.c_void_p(self.h), _p(k, C.c_float), _p(v, C.c_float))
        return k, v

    def gather_tail(self, base, keep):
        keep = np.ascontiguousarray(keep, np.int32)
        check(lib().sgref_cache_gather_tail(C.c_void_p(self.h), base, _p(keep, C.c_int), len(keep)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().sgref_cache_free(self.h)


def forward_target(model: RefModel, tokens, positions, mask=None, cache: Optional[RefCache] = None):
    cfg = model.cfg
    t = np.ascontiguousarray(tokens, np.int32)
    p = np.ascontiguousarray(positions, np.int32)
    n = len(t)
    m = None if mask is None else np.ascontiguousarray(mask, np.uint8).reshape(-1)
    logits = np.zeros((n, cfg.vocab_size), np.float32)
    hidden = np.zeros((n, cfg.d_model), np.float32)
    check(lib().sgref_forward_target(C.c_void_p(model.h), _p(t, C.c_int), _p(p, C.c_int), n,
                                     _p(m, C.c_ubyte), C.c_void_p(cache.h) if cache else None,
                                     _p(logits, C.c_float), _p(hidden, C.c_float)))
    return logits, hidden


def forward_draft_rows(draft: RefDraft, model: RefModel, tokens, prev_feat, positions,
                       cache: Optional[RefCache] = None, extend=True):
    cfg = model.cfg
    t = np.ascontiguousarray(tokens, np.int32)
    p = np.ascontiguousarray(positions, np.int32)
    f = np.ascontiguousarray(prev_feat, np.float32)
    n = len(t)
    feats = np.zeros((n, cfg.d_model), np.float32)
    logits = np.zeros((n, cfg.vocab_size), np.float32)
    check(lib().sgref_forward_draft_rows(C.c_void_p(draft.h), C.c_void_p(model.h), _p(t, C.c_int),
                                         _p(f, C.c_float), _p(p, C.c_int), n,
                                         C.c_void_p(cache.h) if cache else None, int(extend),
                                         _p(feats, C.c_float), _p(logits, C.c_float)))
    return feats, logits


def sample_token(logits, temp, key):
    l = np.ascontiguousarray(logits, np.float32)
    out = C.c_int()
    check(lib().sgref_sample_token(_p(l, C.c_float), l.size, C.c_double(temp), C.c_ulonglong(key), C.byref(out)))
    return out.value


def sample_token_u(logits, temp, U, want_prefix=False):
    """tinylm.hpp:614-627 with the uniform supplied: (token, sum, sequential prefixes|None)."""
    l = np.ascontiguousarray(logits, np.float32)
    out = C.c_int()
    s = C.c_double()
    pre = np.zeros(l.size, np.float64) if want_prefix else None
    check(lib().sgref_sample_token_u(_p(l, C.c_float), l.size, C.c_double(temp), C.c_double(U), C.byref(out),
                                     C.byref(s), _p(pre, C.c_double)))
    return out.value, s.value, pre


def exp_array(x):
    """std::exp (the reference host's libm) elementwise."""
    xx = np.ascontiguousarray(x, np.float64)
    y = np.zeros_like(xx)
    lib().sgref_exp_array(_p(xx, C.c_double), C.c_longlong(xx.size), _p(y, C.c_double))
    return y


def uniform(key):
    """Rng(key).uniform() (rng.hpp:28-41)."""
    f = lib().sgref_uniform
    f.restype = C.c_double
    return f(C.c_ulonglong(key))


def tree_arrays(tree):
    tok = np.array([n.token for n in tree], np.int32)
    par = np.array([n.parent for n in tree], np.int32)
    dep = np.array([n.depth for n in tree], np.int32)
    lp = np.array([n.log_prob for n in tree], np.float64)
    conf = np.array([n.confidence for n in tree], np.float64)
    return tok, par, dep, lp, conf


def expand_tree_with(root, k, l, vocab, fn, cap=4096):
    """fn(n_nodes, tokens, parents, depths, node) -> log-probs (len vocab)."""
    def cb(ctx, n, tp, pp, dp, node, out):
        toks = [tp[i] for i in range(n)]
        pars = [pp[i] for i in range(n)]
        deps = [dp[i] for i in range(n)]
        lps = np.asarray(fn(toks, pars, deps, node), np.float64)
        for i in range(vocab):
            out[i] = float(lps[i])
    cbf = LPS_FN(cb)
    tok = np.zeros(cap, np.int32)
    par = np.zeros(cap, np.int32)
    dep = np.zeros(cap, np.int32)
    lp = np.zeros(cap, np.float64)
    conf = np.zeros(cap, np.float64)
    n = C.c_int()
    check(lib().sgref_expand_tree_with(root, k, l, vocab, cbf, None, cap, _p(tok, C.c_int), _p(par, C.c_int),
                                       _p(dep, C.c_int), _p(lp, C.c_double), _p(conf, C.c_double), C.byref(n)))
    n = n.value
    return tok[:n], par[:n], dep[:n], lp[:n], conf[:n]


def rerank(arrs, n_verify):
    tok, par, dep, lp, conf = [np.ascontiguousarray(a) for a in arrs]
    n = len(tok)
    sel = np.zeros(n, np.int32)
    ns = C.c_int()
    mask = np.zeros(min(n, n_verify) ** 2, np.uint8)
    check(lib().sgref_rerank(n, _p(tok, C.c_int), _p(par, C.c_int), _p(dep, C.c_int), _p(lp, C.c_double),
                             _p(conf, C.c_double), n_verify, _p(sel, C.c_int), C.byref(ns), _p(mask, C.c_ubyte)))
    k = ns.value
    return sel[:k], mask.reshape(k, k)


def verify(arrs, sel, logits, hidden, vocab, d, temp, seq_seed, root_pos):
    tok, par, dep, lp, conf = [np.ascontiguousarray(a) for a in arrs]
    sel = np.ascontiguousarray(sel, np.int32)
    ns = len(sel)
    lg = np.ascontiguousarray(logits, np.float32)
    hd = None if hidden is None else np.ascontiguousarray(hidden, np.float32)
    acc_t = np.zeros(ns + 1, np.int32)
    acc_r = np.zeros(ns + 1, np.int32)
    L, B = C.c_int(), C.c_int()
    nh = np.zeros((ns + 1) * max(d, 1), np.float32)
    check(lib().sgref_verify(len(tok), _p(tok, C.c_int), _p(par, C.c_int), _p(dep, C.c_int), _p(lp, C.c_double),
                             _p(conf, C.c_double), _p(sel, C.c_int), ns, _p(lg, C.c_float), _p(hd, C.c_float),
                             vocab, d, C.c_double(temp), C.c_ulonglong(seq_seed), root_pos, _p(acc_t, C.c_int),
                             C.byref(L), C.byref(B), _p(acc_r, C.c_int), _p(nh, C.c_float)))
    n = L.value
    return acc_t[:n].tolist(), n, B.value, acc_r[:n].tolist()


def plan_step(c_peak, b, alpha=2.0, kmax=10, lmax=6):
    out = np.zeros(3, np.int32)
    check(lib().sgref_plan_step(c_peak, b, C.c_double(alpha), kmax, lmax, _p(out, C.c_int)))
    return tuple(int(x) for x in out)


MODES = {"vanilla": 0, "fixed_spec": 1, "adaptive_spec": 2}


def gen_args(c_peak, alpha=2.0, k_max=10, l_max=6, mode="vanilla", early_term=True, temperature=0.0,
             seed=0, max_new_tokens=0, fixed=(1, 0, 0)):
    return GenArgs(alpha, k_max, l_max, c_peak, MODES[mode], int(early_term), temperature, seed,
                   max_new_tokens, fixed[0], fixed[1], fixed[2])


def generate(model: RefModel, draft: RefDraft, prompts, g, **kw):
    """Returns dict with tokens, prompt_len, hit_eos, features, steps, totals."""
    plens = np.array([len(p) for p in prompts], np.int32)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts]), np.int32)
    a = gen_args(**kw)
    h = lib().sgref_generate(C.c_void_p(model.h), C.c_void_p(draft.h), _p(flat, C.c_int), _p(plens, C.c_int),
                             len(prompts), g, C.byref(a))
    if not h:
        raise RuntimeError(lib().sgref_last_error().decode())
    h = C.c_void_p(h)
    try:
        ns = lib().sgref_bs_nseq(h)
        d = model.cfg.d_model
        out = dict(tokens=[], prompt_len=[], hit_eos=[], features=[])
        for i in range(ns):
            L, P, E = C.c_int(), C.c_int(), C.c_int()
            cap = model.cfg.max_seq_len
            tk = np.zeros(cap, np.int32)
            nf = lib().sgref_bs_seq(h, i, _p(tk, C.c_int), cap, C.byref(L), C.byref(P), C.byref(E))
            f = np.zeros(nf, np.float32)
            lib().sgref_bs_features(h, i, _p(f, C.c_float))
            out["tokens"].append(tk[:L.value].tolist())
            out["prompt_len"].append(P.value)
            out["hit_eos"].append(bool(E.value))
            out["features"].append(f.reshape(-1, d))
        nst = lib().sgref_bs_nsteps(h)
        b = np.zeros(nst, np.int32)
        nkl = np.zeros(3 * nst, np.int32)
        acc = np.zeros(nst, np.int32)
        lib().sgref_bs_steps(h, _p(b, C.c_int), _p(nkl, C.c_int), _p(acc, C.c_int))
        out["steps"] = [(i, int(b[i]), int(nkl[3 * i]), int(nkl[3 * i + 1]), int(nkl[3 * i + 2]), int(acc[i]))
                        for i in range(nst)]
        tot = np.zeros(2, np.int64)
        lib().sgref_bs_totals(h, _p(tot, C.c_longlong))
        out["total_accepted"], out["total_verify_slots"] = int(tot[0]), int(tot[1])
        return out
    finally:
        lib().sgref_bs_free(h)


def generate_threaded(model, draft, prompts, g, threads, **kw):
    plens = np.array([len(p) for p in prompts], np.int32)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts]), np.int32)
    a = gen_args(**kw)
    secs = C.c_double()
    n = lib().sgref_generate_threaded(C.c_void_p(model.h), C.c_void_p(draft.h), _p(flat, C.c_int),
                                      _p(plens, C.c_int), len(prompts), g, C.byref(a), threads, C.byref(secs))
    if n < 0:
        raise RuntimeError("reference generate failed: " + lib().sgref_last_error().decode())
    return int(n), secs.value


def policy_loss_grad(model: RefModel, seqs):
    """policy_loss_grad<float> (grpo.hpp:235-276) of the compiled reference. seqs: list of
    (tokens, prompt_len, weight). Returns (loss, grad[param_count])."""
    toks = np.ascontiguousarray(np.concatenate([np.asarray(t, np.int32) for t, _, _ in seqs]), np.int32)
    lens = np.array([len(t) for t, _, _ in seqs], np.int32)
    pl = np.array([q for _, q, _ in seqs], np.int32)
    w = np.array([x for _, _, x in seqs], np.float64)
    n = lib().sgref_param_count(C.byref(cfg_c(model.cfg)))
    grad = np.zeros(n, np.float32)
    loss = C.c_double()
    check(lib().sgref_policy_loss_grad(C.c_void_p(model.h), len(seqs), _p(toks, C.c_int), _p(lens, C.c_int),
                                       _p(pl, C.c_int), _p(w, C.c_double), _p(grad, C.c_float), C.byref(loss)))
    return loss.value, grad


def _seq_arrays(seqs, d):
    toks = np.ascontiguousarray(np.concatenate([np.asarray(s.tokens, np.int32) for s in seqs]), np.int32)
    lens = np.array([len(s.tokens) for s in seqs], np.int32)
    feats = np.ascontiguousarray(np.concatenate([np.asarray(s.features, np.float32).reshape(-1) for s in seqs]),
                                 np.float32)
    return toks, lens, feats


def draft_loss_grad(draft: RefDraft, model: RefModel, seqs, w_feat=1.0, w_tok=0.1):
    toks, lens, feats = _seq_arrays(seqs, model.cfg.d_model)
    grad = np.zeros(draft.n, np.float32)
    terms = np.zeros(4, np.float64)
    check(lib().sgref_draft_loss_grad(C.c_void_p(draft.h), C.c_void_p(model.h), len(seqs), _p(toks, C.c_int),
                                      _p(lens, C.c_int), _p(feats, C.c_float), C.c_double(w_feat),
                                      C.c_double(w_tok), _p(grad, C.c_float), _p(terms, C.c_double)))
    return grad, tuple(terms)


def draft_update(draft: RefDraft, model: RefModel, seqs, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0,
                 w_feat=1.0, w_tok=0.1, opt=None):
    toks, lens, feats = _seq_arrays(seqs, model.cfg.d_model)
    own = opt is None
    if own:
        a = AdamC(lr, beta1, beta2, eps, wd)
        opt = lib().sgref_adamw_new(C.byref(a))
    terms = np.zeros(4, np.float64)
    check(lib().sgref_draft_update(C.c_void_p(draft.h), C.c_void_p(model.h), len(seqs), _p(toks, C.c_int),
                                   _p(lens, C.c_int), _p(feats, C.c_float), C.c_void_p(opt), C.c_double(w_feat),
                                   C.c_double(w_tok), _p(terms, C.c_double)))
    if own:
        lib().sgref_adamw_free(C.c_void_p(opt))
    return tuple(terms)
