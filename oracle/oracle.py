"""CPU restatement (numpy) of the reference's GRPO-rollout hot path.

TEST INFRASTRUCTURE ONLY -- this module is the *checker*. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg may import it.
The product path (``paper_2509_21792_b200``) never imports it and has no CPU
fallback.

Every function restates the reference algorithm of arXiv 2509.21792's desk-scale
C++ implementation (``/root/reference/proj``); each docstring cites the file:line it
follows. Paths are relative to ``/root/reference/proj``.

Pinning: ``tests/test_oracle_pinning.py`` checks this module against golden vectors
produced by the compiled reference itself (``oracle/_ref/libsgrpo_ref.so``, built by
``oracle/Makefile`` from the unmodified reference sources; fixtures written by
``tests/golden/make_golden.py``) and against the known-answer tests of the
reference's own test-suite (``tests/test_drafttree.cpp``, ``tests/test_tinylm.cpp``,
``SPEC.md:295-330``).

Arithmetic notes:
* fp32 tensors are float32 numpy arrays; BLAS summation order differs from the
  reference's i-k-j loops (``include/sgrpo/nn.hpp:15-29``), so fp32 outputs agree to
  ~1e-6 relative, not bitwise. Integer / index / tree decisions agree exactly.
* Sequential fp64 sums of the reference (``nn.hpp:172-180``, ``tinylm.hpp:614-627``)
  are reproduced with ``np.cumsum`` (sequential) and ``math`` (glibc) so sampling and
  confidences match bit-for-bit given identical logits.
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
PAD_TOKEN = 0  # tinylm.hpp:40
EOS_TOKEN = 1  # tinylm.hpp:41


# ----------------------------------------------------------------------------------
# RNG -- include/sgrpo/rng.hpp:9-65
# ----------------------------------------------------------------------------------
def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def splitmix64(state: int):
    """rng.hpp:9-14. Returns (value, new_state)."""
    state = (state + GOLDEN) & MASK64
    return _mix64(state), state


def mix_key(a: int, b: int, c: Optional[int] = None) -> int:
    """rng.hpp:17-24."""
    if c is not None:
        return mix_key(mix_key(a, b), c)
    a &= MASK64
    b &= MASK64
    s = (a ^ ((b + GOLDEN + ((a << 6) & MASK64) + (a >> 2)) & MASK64)) & MASK64
    return splitmix64(s)[0]


class Rng:
    """rng.hpp:28-65 (constructor discards one draw)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64
        _, self.state = splitmix64(self.state)
        self._spare = None

    def next_u64(self) -> int:
        v, self.state = splitmix64(self.state)
        return v

    def uniform(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def normal(self) -> float:
        if self._spare is not None:
            s, self._spare = self._spare, None
            return s
        u1 = self.uniform()
        u2 = self.uniform()
        while u1 <= 1e-300:
            u1 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        th = 6.283185307179586476925286766559 * u2
        self._spare = r * math.sin(th)
        return r * math.cos(th)

    def below(self, n: int) -> int:
        return self.next_u64() % n


def _u64_stream(seed: int, n: int) -> np.ndarray:
    """The first n next_u64() outputs of Rng(seed), vectorised (rng.hpp:30-37)."""
    with np.errstate(over="ignore"):
        st = np.uint64(seed & MASK64) + np.uint64(GOLDEN) * np.arange(2, n + 2, dtype=np.uint64)
        z = st
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def normal_stream(seed: int, n: int) -> np.ndarray:
    """First n Rng(seed).normal() values (Box-Muller pairs, spare cached; rng.hpp:40-53).

    Transcendentals go through ``math`` (the C library), exactly as the reference."""
    npairs = (n + 1) // 2
    u = (_u64_stream(seed, 2 * npairs) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    u1, u2 = u[0::2], u[1::2]
    if np.any(u1 <= 1e-300):  # the resample branch (probability 2^-53): fall back
        r = Rng(seed)
        return np.array([r.normal() for _ in range(n)])
    log, sqrt, sin, cos = math.log, math.sqrt, math.sin, math.cos
    tp = 6.283185307179586476925286766559
    out = np.empty(2 * npairs)
    rr = [sqrt(-2.0 * log(a)) for a in u1.tolist()]
    th = (u2 * tp).tolist()
    out[0::2] = [r * cos(t) for r, t in zip(rr, th)]
    out[1::2] = [r * sin(t) for r, t in zip(rr, th)]
    return out[:n]


# ----------------------------------------------------------------------------------
# Model config, parameter layout and init -- include/sgrpo/tinylm.hpp:16-189
# ----------------------------------------------------------------------------------
@dataclass(frozen=True)
class ModelConfig:
    """tinylm.hpp:16-37."""
    vocab_size: int = 16
    d_model: int = 32
    n_layers: int = 2
    n_heads: int = 4
    d_ff: int = 128
    max_seq_len: int = 32
    seed: int = 0

    def validate(self):
        if self.vocab_size < 4:
            raise ValueError("vocab_size must be >= 4 (EOS and PAD included)")
        if min(self.d_model, self.n_layers, self.n_heads, self.d_ff) <= 0:
            raise ValueError("model dims must be positive")
        if self.d_model % self.n_heads:
            raise ValueError("d_model must be divisible by n_heads")
        if self.max_seq_len < 8:
            raise ValueError("max_seq_len must be >= 8")


LAYER_FIELDS = ("ln1_g", "ln1_b", "wq", "wk", "wv", "wo", "ln2_g", "ln2_b", "w1", "w2")


def _layer_specs(d: int, dff: int):
    """tinylm.hpp:67-80 (order ln1_g, ln1_b, wq, wk, wv, wo, ln2_g, ln2_b, w1, w2)."""
    return [("ln1_g", 1, d, "ones"), ("ln1_b", 1, d, "zeros"), ("wq", d, d, "normal"),
            ("wk", d, d, "normal"), ("wv", d, d, "normal"), ("wo", d, d, "normal_residual"),
            ("ln2_g", 1, d, "ones"), ("ln2_b", 1, d, "zeros"), ("w1", d, dff, "normal"),
            ("w2", dff, d, "normal_residual")]


def model_specs(cfg: ModelConfig):
    """tinylm.hpp:133-150."""
    d = cfg.d_model
    s = [("tok_emb", cfg.vocab_size, d, "normal"), ("pos_emb", cfg.max_seq_len, d, "pos_emb")]
    for li in range(cfg.n_layers):
        s += [(f"l{li}.{n}", r, c, i) for n, r, c, i in _layer_specs(d, cfg.d_ff)]
    s += [("lnf_g", 1, d, "ones"), ("lnf_b", 1, d, "zeros"), ("lm_head", d, cfg.vocab_size, "normal")]
    return s


def draft_specs(cfg: ModelConfig, n_layers: int = 1):
    """tinylm.hpp:172-189."""
    d = cfg.d_model
    s = [("w_fuse", 2 * d, d, "normal")]
    for li in range(n_layers):
        s += [(f"l{li}.{n}", r, c, i) for n, r, c, i in _layer_specs(d, cfg.d_ff)]
    s += [("lnf_g", 1, d, "ones"), ("lnf_b", 1, d, "zeros")]
    return s


def _init_flat(specs, seed: int, n_res_layers: int) -> np.ndarray:
    """tinylm.hpp:83-109: one Rng over all tensors in layout order."""
    total = sum(r * c for _, r, c, _ in specs)
    n_norm = sum(r * c for _, r, c, i in specs if i in ("normal", "normal_residual", "pos_emb"))
    z = normal_stream(seed, n_norm)
    res_scale = 0.02 / math.sqrt(2.0 * n_res_layers)
    flat = np.zeros(total, dtype=np.float32)
    off = zo = 0
    for _, r, c, init in specs:
        n = r * c
        if init == "normal":
            flat[off:off + n] = (0.02 * z[zo:zo + n]).astype(np.float32)
            zo += n
        elif init == "normal_residual":
            flat[off:off + n] = (res_scale * z[zo:zo + n]).astype(np.float32)
            zo += n
        elif init == "pos_emb":
            flat[off:off + n] = (0.01 * z[zo:zo + n]).astype(np.float32)
            zo += n
        elif init == "ones":
            flat[off:off + n] = 1.0
        off += n
    return flat


class Params:
    """Flat fp32 storage plus named views (tinylm.hpp:118-131 / 156-170)."""

    def __init__(self, cfg: ModelConfig, specs, flat: np.ndarray, n_layers: int):
        self.config = cfg
        self.specs = specs
        self.flat = flat
        self.n_layers = n_layers
        self._views()

    def _views(self):
        self.t = {}
        off = 0
        for name, r, c, _ in self.specs:
            v = self.flat[off:off + r * c]
            self.t[name] = v.reshape(r, c) if r > 1 else v
            off += r * c

    def layer(self, li: int):
        return {f: self.t[f"l{li}.{f}"] for f in LAYER_FIELDS}

    def copy(self):
        return Params(self.config, self.specs, self.flat.copy(), self.n_layers)

    def offsets(self):
        out, off = {}, 0
        for name, r, c, _ in self.specs:
            out[name] = (off, r, c)
            off += r * c
        return out


def init_model(cfg: ModelConfig) -> Params:
    """tinylm.hpp:133-150."""
    cfg.validate()
    specs = model_specs(cfg)
    return Params(cfg, specs, _init_flat(specs, cfg.seed, cfg.n_layers), cfg.n_layers)


def init_draft(cfg: ModelConfig, n_layers: int = 1) -> Params:
    """tinylm.hpp:172-189 (seed mix_key(seed, 0xd4af7))."""
    cfg.validate()
    if n_layers <= 0:
        raise ValueError("draft n_layers must be positive")
    specs = draft_specs(cfg, n_layers)
    return Params(cfg, specs, _init_flat(specs, mix_key(cfg.seed, 0xD4AF7), n_layers), n_layers)


def model_from_flat(cfg: ModelConfig, flat) -> Params:
    return Params(cfg, model_specs(cfg), np.ascontiguousarray(flat, dtype=np.float32).copy(), cfg.n_layers)


def draft_from_flat(cfg: ModelConfig, flat, n_layers: int = 1) -> Params:
    return Params(cfg, draft_specs(cfg, n_layers), np.ascontiguousarray(flat, dtype=np.float32).copy(), n_layers)


def param_count(cfg: ModelConfig) -> int:
    return sum(r * c for _, r, c, _ in model_specs(cfg))


def draft_param_count(cfg: ModelConfig, n_layers: int = 1) -> int:
    return sum(r * c for _, r, c, _ in draft_specs(cfg, n_layers))


# ----------------------------------------------------------------------------------
# Scalar NN kernels -- include/sgrpo/nn.hpp
# ----------------------------------------------------------------------------------
F32 = np.float32


def layernorm(x: np.ndarray, g, b, eps=F32(1e-5)):
    """nn.hpp:70-98 (population variance, fp32). Returns (y, mean, rstd)."""
    d = x.shape[-1]
    mu = (x.sum(axis=-1, dtype=F32) / F32(d)).astype(F32)
    dv = x - mu[:, None]
    var = ((dv * dv).sum(axis=-1, dtype=F32) / F32(d)).astype(F32)
    rstd = (F32(1) / np.sqrt(var + eps)).astype(F32)
    y = (g * dv * rstd[:, None] + b).astype(F32)
    return y, mu, rstd


def layernorm_bwd(x, g, mu, rstd, dy):
    """nn.hpp:100-125. Returns (dx, dgamma, dbeta)."""
    d = x.shape[-1]
    xhat = (x - mu[:, None]) * rstd[:, None]
    dn = dy * g
    s1 = dn.sum(axis=-1, dtype=F32)
    s2 = (dn * xhat).sum(axis=-1, dtype=F32)
    dx = (dn - s1[:, None] / F32(d) - xhat * s2[:, None] / F32(d)) * rstd[:, None]
    return dx.astype(F32), (dy * xhat).sum(axis=0, dtype=F32), dy.sum(axis=0, dtype=F32)


_GC = F32(0.7978845608028654)


def gelu(x):
    """nn.hpp:128-133 (tanh approximation)."""
    u = _GC * (x + F32(0.044715) * x * x * x)
    return (F32(0.5) * x * (F32(1) + np.tanh(u))).astype(F32)


def gelu_grad(x):
    """nn.hpp:135-144."""
    x3 = x * x * x
    th = np.tanh(_GC * (x + F32(0.044715) * x3))
    sech2 = F32(1) - th * th
    return (F32(0.5) * (F32(1) + th) + F32(0.5) * x * sech2 * _GC * (F32(1) + F32(3) * F32(0.044715) * x * x)).astype(F32)


def softmax_rows(s: np.ndarray) -> np.ndarray:
    """nn.hpp:157-169 over the last axis; -inf entries are masked."""
    mx = s.max(axis=-1, keepdims=True)
    if np.any(mx == -np.inf):
        raise FloatingPointError("softmax over fully masked row")
    e = np.exp(s - mx).astype(F32)
    return (e / e.sum(axis=-1, keepdims=True, dtype=F32)).astype(F32)


def log_softmax_row(row) -> np.ndarray:
    """nn.hpp:172-180 in double; the sum is sequential (np.cumsum) like the reference."""
    r = np.asarray(row, dtype=np.float64)
    mx = r.max()
    s = np.cumsum(np.exp(r - mx))[-1]
    return r - (mx + math.log(s))


# ----------------------------------------------------------------------------------
# KV cache and attention mask -- tinylm.hpp:232-277
# ----------------------------------------------------------------------------------
class KvCache:
    """tinylm.hpp:232-269: per layer [len, d] fp32 K and V."""

    def __init__(self, n_layers: int, d: int):
        self.n_layers, self.d = n_layers, d
        self.k = [np.zeros((0, d), F32) for _ in range(n_layers)]
        self.v = [np.zeros((0, d), F32) for _ in range(n_layers)]

    @property
    def len(self) -> int:
        return self.k[0].shape[0] if self.n_layers else 0

    def copy(self):
        c = KvCache(self.n_layers, self.d)
        c.k = [a.copy() for a in self.k]
        c.v = [a.copy() for a in self.v]
        return c

    def truncate(self, new_len: int):
        """tinylm.hpp:245-250."""
        if new_len > self.len:
            raise ValueError("cache truncate beyond length")
        self.k = [a[:new_len] for a in self.k]
        self.v = [a[:new_len] for a in self.v]

    def gather_tail(self, base_len: int, keep: Sequence[int]):
        """tinylm.hpp:254-268: keep rows base_len+keep[i] at base_len+i, in order."""
        idx = np.concatenate([np.arange(base_len), base_len + np.asarray(keep, dtype=np.int64)])
        self.k = [a[idx] for a in self.k]
        self.v = [a[idx] for a in self.v]


def _decode_blocks(p: Params, x: np.ndarray, mask: Optional[np.ndarray], cache: Optional[KvCache],
                   extra=None, want_kv=False, extend_cache=True):
    """tinylm.hpp:305-413: pre-LN blocks over [cache | ancestor pool | masked new rows].

    ``extra`` = (row_ancestors, pool_k, pool_v); returns x and optional per-layer new K/V."""
    cfg = p.config
    d, H = cfg.d_model, cfg.n_heads
    dh = d // H
    scale = F32(1) / np.sqrt(F32(dh))
    rows = x.shape[0]
    if mask is None:
        mask = np.tril(np.ones((rows, rows), dtype=bool))
    else:
        mask = np.asarray(mask).astype(bool).reshape(rows, rows)
    krows, vrows = [], []
    for li in range(p.n_layers):
        w = p.layer(li)
        xln, _, _ = layernorm(x, w["ln1_g"], w["ln1_b"])
        q = (xln @ w["wq"]).astype(F32)
        kn = (xln @ w["wk"]).astype(F32)
        vn = (xln @ w["wv"]).astype(F32)
        kc = cache.k[li] if cache is not None else np.zeros((0, d), F32)
        vc = cache.v[li] if cache is not None else np.zeros((0, d), F32)
        att = np.zeros_like(q)
        for i in range(rows):
            parts_k, parts_v = [kc], [vc]
            if extra is not None:
                anc = extra[0][i]
                if len(anc):
                    parts_k.append(extra[1][li][anc])
                    parts_v.append(extra[2][li][anc])
            n_fixed = sum(a.shape[0] for a in parts_k)
            K = np.concatenate(parts_k + [kn], 0).reshape(-1, H, dh)
            V = np.concatenate(parts_v + [vn], 0).reshape(-1, H, dh)
            qi = q[i].reshape(H, dh)
            s = (np.einsum("hd,khd->hk", qi, K).astype(F32) * scale).astype(F32)
            allowed = np.concatenate([np.ones(n_fixed, bool), mask[i]])
            s[:, ~allowed] = -np.inf
            pr = softmax_rows(s)
            att[i] = np.einsum("hk,khd->hd", pr, V).reshape(d)
        x = (x + (att @ w["wo"]).astype(F32)).astype(F32)
        xln, _, _ = layernorm(x, w["ln2_g"], w["ln2_b"])
        h = gelu((xln @ w["w1"]).astype(F32))
        x = (x + (h @ w["w2"]).astype(F32)).astype(F32)
        if cache is not None and extend_cache:
            cache.k[li] = np.concatenate([cache.k[li], kn], 0)
            cache.v[li] = np.concatenate([cache.v[li], vn], 0)
        if want_kv:
            krows.append(kn)
            vrows.append(vn)
    return x, krows, vrows


_target_forward_calls = [0]


def target_forward_calls() -> int:
    """tinylm.hpp:288-291."""
    return _target_forward_calls[0]


def forward_target(p: Params, tokens, positions, mask=None, cache: Optional[KvCache] = None):
    """tinylm.hpp:422-463. Returns (logits [rows,V] fp32, hidden [rows,d] fp32)."""
    cfg = p.config
    tokens = np.asarray(tokens, dtype=np.int64)
    positions = np.asarray(positions, dtype=np.int64)
    rows = len(tokens)
    if rows == 0:
        raise ValueError("forward_target: empty input")
    if len(positions) != rows:
        raise ValueError("forward_target: tokens/positions mismatch")
    if mask is not None and np.asarray(mask).size != rows * rows:
        raise ValueError("forward_target: mask shape mismatch")
    if np.any(tokens < 0) or np.any(tokens >= cfg.vocab_size):
        raise ValueError("forward_target: token id out of range")
    if np.any(positions < 0) or np.any(positions >= cfg.max_seq_len):
        raise IndexError("forward_target: position beyond max_seq_len")
    _target_forward_calls[0] += 1
    x = (p.t["tok_emb"][tokens] + p.t["pos_emb"][positions]).astype(F32)
    x, _, _ = _decode_blocks(p, x, mask, cache)
    hidden, _, _ = layernorm(x, p.t["lnf_g"], p.t["lnf_b"])
    logits = (hidden @ p.t["lm_head"]).astype(F32)
    if not np.all(np.isfinite(logits)):
        raise RuntimeError("forward_target: non-finite logits")
    return logits, hidden


def forward_draft_rows(dr: Params, tgt: Params, tokens, prev_features, positions, mask=None,
                       cache: Optional[KvCache] = None, row_ancestors=None, pool_k=None, pool_v=None,
                       want_kv_rows=False, extend_cache=True):
    """tinylm.hpp:502-563. Returns (features, logits, k_rows, v_rows)."""
    cfg = dr.config
    d = cfg.d_model
    tokens = np.asarray(tokens, dtype=np.int64)
    positions = np.asarray(positions, dtype=np.int64)
    rows = len(tokens)
    if rows == 0:
        raise ValueError("forward_draft: empty input")
    prev = np.asarray(prev_features, dtype=F32).reshape(-1)
    if prev.size != rows * d:
        raise ValueError("forward_draft: feature dimension mismatch")
    if np.any(tokens < 0) or np.any(tokens >= cfg.vocab_size):
        raise ValueError("forward_draft: token id out of range")
    if np.any(positions < 0) or np.any(positions >= cfg.max_seq_len):
        raise IndexError("forward_draft: position beyond max_seq_len")
    fused = np.concatenate([tgt.t["tok_emb"][tokens], prev.reshape(rows, d)], 1)
    x = ((fused @ dr.t["w_fuse"]).astype(F32) + tgt.t["pos_emb"][positions]).astype(F32)
    extra = (row_ancestors, pool_k, pool_v) if row_ancestors is not None else None
    x, kr, vr = _decode_blocks(dr, x, mask, cache, extra, want_kv_rows, extend_cache)
    feats, _, _ = layernorm(x, dr.t["lnf_g"], dr.t["lnf_b"])
    logits = (feats @ tgt.t["lm_head"]).astype(F32)
    if not np.all(np.isfinite(logits)):
        raise RuntimeError("forward_draft: non-finite logits")
    return feats, logits, kr, vr


def sample_token(logits, temperature: float, rng_key: int) -> int:
    """tinylm.hpp:591-628: argmax (lowest index) at T=0, fp64 inverse CDF at T>0."""
    l = np.asarray(logits, dtype=np.float64)
    if l.size == 0:
        raise ValueError("sample_token: empty logits")
    if np.any(np.isnan(l)):
        raise ArithmeticError("sample_token: NaN logit")
    mx = l.max()
    if mx == -np.inf:
        raise ArithmeticError("sample_token: all logits are -inf")
    if temperature < 0:
        raise ValueError("sample_token: negative temperature")
    if temperature == 0:
        return int(np.argmax(l))
    cdf = np.cumsum(np.exp((l - mx) / temperature))
    u = Rng(rng_key).uniform() * cdf[-1]
    i = int(np.searchsorted(cdf, u, side="right"))
    return min(i, l.size - 1)


# ----------------------------------------------------------------------------------
# Draft tree -- include/sgrpo/drafttree.hpp, src/drafttree.cpp
# ----------------------------------------------------------------------------------
@dataclass
class DraftNode:
    """drafttree.hpp:11-17."""
    token: int
    parent: int
    depth: int
    log_prob: float = 0.0
    confidence: float = 1.0


def max_candidates(k: int, l: int) -> int:
    """drafttree.cpp:11-15."""
    if k < 0 or l < 0:
        raise ValueError("max_candidates: negative argument")
    return 1 + k + max(0, l - 1) * k * k


def topk_tokens(lps, k: int) -> List[int]:
    """drafttree.cpp:20-30: top-k by (value desc, index asc)."""
    lps = np.asarray(lps, dtype=np.float64)
    kk = min(k, lps.size)
    order = np.lexsort((np.arange(lps.size), -lps))
    return [int(i) for i in order[:kk]]


def expand_tree_with(root_token: int, k_draft: int, l_draft: int, fn: Callable) -> List[DraftNode]:
    """drafttree.cpp:34-70 (EAGLE-2: level 1 expands the root, later levels the top-k by
    (confidence desc, token asc, index asc) of the previous level)."""
    if k_draft < 0 or l_draft < 0:
        raise ValueError("expand_tree: negative k_draft or l_draft")
    t = [DraftNode(root_token, -1, 0, 0.0, 1.0)]
    if k_draft == 0 or l_draft == 0:
        return t
    frontier = [0]
    for level in range(1, l_draft + 1):
        created = []
        for ni in frontier:
            lps = np.asarray(fn(t, ni), dtype=np.float64)
            for tok in topk_tokens(lps, k_draft):
                lp = float(lps[tok])
                created.append(len(t))
                t.append(DraftNode(tok, ni, level, lp, t[ni].confidence * math.exp(lp)))
        if level == l_draft or not created:
            break
        created.sort(key=lambda a: (-t[a].confidence, t[a].token, a))
        frontier = sorted(created[:k_draft])
    return t


def rerank_candidates(tree: List[DraftNode], n_verify: int):
    """drafttree.cpp:126-143: top-n_verify by (confidence desc, index asc), ascending."""
    if n_verify < 1:
        raise ValueError("rerank_candidates: n_verify must be >= 1")
    order = sorted(range(len(tree)), key=lambda a: (-tree[a].confidence, a))[:n_verify]
    sel = sorted(order)
    return sel, build_tree_mask(tree, sel)


def build_tree_mask(tree: List[DraftNode], selected: Sequence[int]) -> np.ndarray:
    """drafttree.cpp:145-168: mask[i][j] = selected j is i or an ancestor of i."""
    n = len(selected)
    if n == 0 or selected[0] != 0:
        raise ValueError("build_tree_mask: selection must include the root first")
    pos = {}
    for i, s in enumerate(selected):
        if i > 0 and s <= selected[i - 1]:
            raise ValueError("build_tree_mask: selection must be ascending")
        pos[s] = i
    m = np.zeros((n, n), dtype=np.uint8)
    for i, s in enumerate(selected):
        node = s
        while node != -1:
            if node not in pos:
                raise ValueError("build_tree_mask: closure violation")
            m[i, pos[node]] = 1
            node = tree[node].parent
    return m


@dataclass
class VerifyResult:
    """drafttree.hpp:53-61."""
    accepted_tokens: List[int]
    accepted_len: int
    bonus_token: int
    accepted_rows: List[int]
    new_hidden: Optional[np.ndarray]
    emitted: List[int] = field(default_factory=list)


def verify(tree: List[DraftNode], selected: Sequence[int], logits, hidden=None, vocab: int = 0,
           temperature: float = 0.0, seq_seed: int = 0, root_pos: int = 0) -> VerifyResult:
    """drafttree.cpp:170-222: target emission per selected node keyed by
    mix_key(seq_seed, root_pos+depth+1); longest matching root walk plus bonus."""
    n = len(selected)
    logits = np.asarray(logits, dtype=F32).reshape(-1)
    if vocab <= 0:
        raise ValueError("verify: vocab must be positive")
    if logits.size != n * vocab:
        raise ValueError("verify: logits row count mismatch")
    L = logits.reshape(n, vocab)
    emitted = []
    for i, s in enumerate(selected):
        key = mix_key(seq_seed, root_pos + tree[s].depth + 1)
        emitted.append(sample_token(L[i], temperature, key))
    acc_tokens, rows, cur = [], [0], 0
    while True:
        cur_node, want, nxt = selected[cur], emitted[cur], -1
        for i in range(cur + 1, n):
            nd = tree[selected[i]]
            if nd.parent == cur_node and nd.token == want:
                nxt = i
                break
        if nxt < 0:
            break
        acc_tokens.append(want)
        rows.append(nxt)
        cur = nxt
    bonus = emitted[cur]
    acc_tokens.append(bonus)
    nh = None
    if hidden is not None and np.asarray(hidden).size:
        nh = np.asarray(hidden, dtype=F32).reshape(n, -1)[rows]
    return VerifyResult(acc_tokens, len(acc_tokens), bonus, rows, nh, emitted)


# ----------------------------------------------------------------------------------
# Concurrency-aware controller -- src/scheduler.cpp:14-54
# ----------------------------------------------------------------------------------
def compute_n_verify(c_peak: int, b: int) -> int:
    """scheduler.cpp:26-29 (Eq. 1)."""
    if c_peak < 1 or b < 1:
        raise ValueError("compute_n_verify: c_peak, b >= 1")
    return max(1, c_peak // b)


def compute_k_draft(n_verify: int, k_max: int) -> int:
    """scheduler.cpp:31-34 (Eq. 2)."""
    if n_verify < 1:
        raise ValueError("compute_k_draft: n_verify >= 1")
    return max(0, min(n_verify - 1, k_max))


def compute_l_draft(n_verify: int, alpha: float, l_max: int, k_draft: int) -> int:
    """scheduler.cpp:36-41 (Eq. 3)."""
    if alpha <= 0:
        raise ValueError("compute_l_draft: alpha must be positive")
    if k_draft == 0:
        return 0
    raw = int(math.floor(math.log2(float(n_verify) / alpha)))
    return max(1, min(raw, l_max))


@dataclass
class SpecConfig:
    """scheduler.hpp:14-24."""
    n_verify: int = 1
    k_draft: int = 0
    l_draft: int = 0
    alpha: float = 2.0
    k_max: int = 10
    l_max: int = 6
    c_peak: int = 1

    def validate(self):
        """scheduler.cpp:14-24."""
        if self.n_verify < 1:
            raise ValueError("spec config: n_verify must be >= 1")
        if self.k_draft < 0 or self.l_draft < 0:
            raise ValueError("spec config: k_draft/l_draft must be >= 0")
        if self.k_draft > max(0, self.n_verify - 1):
            raise ValueError("spec config: k_draft must be <= n_verify - 1")
        if self.k_draft > self.k_max:
            raise ValueError("spec config: k_draft exceeds k_max")
        if self.l_draft > self.l_max:
            raise ValueError("spec config: l_draft exceeds l_max")
        if self.alpha <= 0:
            raise ValueError("spec config: alpha must be positive")
        if self.c_peak < 1:
            raise ValueError("spec config: c_peak must be >= 1")


def plan_step(c_peak: int, b_cur: int, alpha: float = 2.0, k_max: int = 10, l_max: int = 6) -> SpecConfig:
    """scheduler.cpp:43-54."""
    n = compute_n_verify(c_peak, b_cur)
    k = compute_k_draft(n, k_max)
    l = compute_l_draft(n, alpha, l_max, k)
    c = SpecConfig(n, k, l, alpha, k_max, l_max, c_peak)
    c.validate()
    return c


# ----------------------------------------------------------------------------------
# Rollout engine -- src/scheduler.cpp:79-354
# ----------------------------------------------------------------------------------
@dataclass
class SeqResult:
    """scheduler.hpp:60-66."""
    id: int
    tokens: List[int]
    prompt_len: int
    hit_eos: bool
    features: np.ndarray  # [(len-1), d]


@dataclass
class GenResult:
    seqs: List[SeqResult]
    steps: List[tuple]  # (step, b_cur, n_verify, k_draft, l_draft, accepted_total)
    events: List[tuple]  # (step, seq, accepted)
    total_accepted: int
    total_verify_slots: int

    def tau(self) -> float:
        """scheduler.cpp:72-75."""
        if self.total_verify_slots == 0:
            raise ArithmeticError("tau: no verification steps logged")
        return self.total_accepted / self.total_verify_slots


class _Seq:
    def __init__(self):
        self.finished = False
        self.hit_eos = False


def _commit_tokens(s: _Seq, accepted: Sequence[int]) -> int:
    """scheduler.cpp:97-118."""
    appended = 0
    for tok in accepted:
        s.tokens.append(int(tok))
        appended += 1
        if tok == EOS_TOKEN:
            s.finished = s.hit_eos = True
            break
        if len(s.tokens) >= s.len_cap:
            s.finished = True
            break
    new_p = len(s.tokens) - 1
    if s.tgt_cache.len > new_p:
        s.tgt_cache.truncate(new_p)
    if s.feats.shape[0] > new_p:
        s.feats = s.feats[:new_p]
    return appended


def _run_step(s: _Seq, tgt: Params, dr: Params, cfg: SpecConfig, temperature: float, trace=None) -> int:
    """scheduler.cpp:122-232 (one decode step of one sequence)."""
    mc = tgt.config
    d = mc.d_model
    p = len(s.tokens) - 1
    l_eff = min(cfg.l_draft, s.len_cap - 1 - p)
    k_eff = min(cfg.k_draft, mc.vocab_size) if l_eff >= 1 else 0
    if k_eff == 0:
        l_eff = 0
    if k_eff == 0:
        tree = expand_tree_with(s.tokens[p], 0, 0, None)
    else:
        j0 = s.dft_cache.len + 1
        js = list(range(j0, p + 1))
        feats_c, logits_c, _, _ = forward_draft_rows(
            dr, tgt, [s.tokens[j] for j in js], s.feats[[j - 1 for j in js]], js, cache=s.dft_cache)
        root_feat = feats_c[-1]
        root_logits = logits_c[-1].astype(np.float64)
        node_feat = {0: root_feat}
        pool_of_node = {0: -1}
        pool_k = [np.zeros((0, d), F32) for _ in range(dr.n_layers)]
        pool_v = [np.zeros((0, d), F32) for _ in range(dr.n_layers)]

        def fn(t, node):
            nonlocal pool_k, pool_v
            if node == 0:
                return log_softmax_row(root_logits)
            nd = t[node]
            anc, a = [], nd.parent
            while a != -1:
                if pool_of_node[a] >= 0:
                    anc.append(pool_of_node[a])
                a = t[a].parent
            anc.reverse()
            f, lg, kr, vr = forward_draft_rows(
                dr, tgt, [nd.token], node_feat[nd.parent], [p + nd.depth], cache=s.dft_cache,
                row_ancestors=[anc], pool_k=pool_k, pool_v=pool_v, want_kv_rows=True,
                extend_cache=False)
            node_feat[node] = f[0]
            pool_of_node[node] = pool_k[0].shape[0]
            pool_k = [np.concatenate([pk, k], 0) for pk, k in zip(pool_k, kr)]
            pool_v = [np.concatenate([pv, v], 0) for pv, v in zip(pool_v, vr)]
            return log_softmax_row(lg[0].astype(np.float64))

        tree = expand_tree_with(s.tokens[p], k_eff, l_eff, fn)
    sel, mask = rerank_candidates(tree, cfg.n_verify)
    toks = [tree[i].token for i in sel]
    poss = [p + tree[i].depth for i in sel]
    base_len = s.tgt_cache.len
    logits, hidden = forward_target(tgt, toks, poss, mask, s.tgt_cache)
    vr = verify(tree, sel, logits, hidden, mc.vocab_size, temperature, s.seed, p)
    if trace is not None:
        trace.append(dict(seq=s.id, p=p, tree=tree, sel=sel, logits=logits, emitted=vr.emitted,
                          accepted_rows=vr.accepted_rows, accepted_tokens=vr.accepted_tokens))
    s.tgt_cache.gather_tail(base_len, vr.accepted_rows)
    s.feats = np.concatenate([s.feats, vr.new_hidden], 0)
    return _commit_tokens(s, vr.accepted_tokens)


def generate_dynamic_batch(tgt: Params, dr: Params, prompts: Sequence[Sequence[int]], g: int,
                           c_peak: int, alpha: float = 2.0, k_max: int = 10, l_max: int = 6,
                           mode: str = "vanilla", early_term: bool = True, temperature: float = 0.0,
                           seed: int = 0, max_new_tokens: int = 0, fixed: Optional[SpecConfig] = None,
                           seq_max_new: Optional[Sequence[int]] = None, trace=None,
                           sid_offset: int = 0) -> GenResult:
    """scheduler.cpp:236-354.

    ``seq_max_new`` (per-sequence caps, indexed by global sid) is the c3 variable-length
    extension; it is not in the reference (parity unpinned)."""
    mc = tgt.config
    if not len(prompts):
        raise ValueError("generate: prompts must be non-empty")
    if g < 1:
        raise ValueError("generate: g must be >= 1")
    if c_peak < 1:
        raise ValueError("generate: c_peak must be >= 1")
    for pr in prompts:
        if len(pr) == 0:
            raise ValueError("generate: zero-length prompt")
        if len(pr) > mc.max_seq_len - 1:
            raise ValueError("generate: prompt longer than max_seq_len - 1")
    if mode == "fixed_spec":
        fixed.validate()
    n_seqs = len(prompts) * g
    seqs: List[_Seq] = [None] * n_seqs
    for pi, prompt in enumerate(prompts):
        q = len(prompt)
        cache = KvCache(mc.n_layers, mc.d_model)
        logits, hidden = forward_target(tgt, prompt, list(range(q)), None, cache)
        for r in range(g):
            sid = pi * g + r
            s = _Seq()
            s.id = sid
            s.seed = mix_key(seed, sid + sid_offset + 1)  # global sid under data-parallel sharding
            s.tokens = [int(t) for t in prompt]
            s.prompt_len = q
            mn = seq_max_new[sid] if seq_max_new is not None else max_new_tokens
            s.len_cap = min(mc.max_seq_len, q + mn) if mn > 0 else mc.max_seq_len
            s.feats = hidden.copy()
            s.tgt_cache = cache.copy()
            s.dft_cache = KvCache(dr.n_layers, mc.d_model)
            tok = sample_token(logits[q - 1], temperature, mix_key(s.seed, q))
            s.tokens.append(tok)
            if tok == EOS_TOKEN:
                s.finished = s.hit_eos = True
            if len(s.tokens) >= s.len_cap:
                s.finished = True
            seqs[sid] = s
    steps, events, tot_acc, tot_slots, step = [], [], 0, 0, 0
    while True:
        b_cur = sum(1 for s in seqs if not s.finished)
        if b_cur == 0:
            break
        eff_b = b_cur if early_term else n_seqs
        if mode == "vanilla":
            cfg = SpecConfig(1, 0, 0, c_peak=c_peak)
        elif mode == "fixed_spec":
            cfg = fixed
        else:
            cfg = plan_step(c_peak, eff_b, alpha, k_max, l_max)
        acc_total = 0
        for s in seqs:
            if s.finished:
                continue
            a = _run_step(s, tgt, dr, cfg, temperature, trace)
            acc_total += a
            events.append((step, s.id, a))
        steps.append((step, b_cur, cfg.n_verify, cfg.k_draft, cfg.l_draft, acc_total))
        tot_acc += acc_total
        tot_slots += b_cur
        step += 1
    out = [SeqResult(s.id, s.tokens, s.prompt_len, s.hit_eos, s.feats) for s in seqs]
    return GenResult(out, steps, events, tot_acc, tot_slots)


# ----------------------------------------------------------------------------------
# Online draft learning -- tinylm.hpp:653-800, 881-953; grpo.hpp:278-344; grpo.cpp:142-186
# ----------------------------------------------------------------------------------
def _train_blocks_fwd(p: Params, x: np.ndarray):
    """tinylm.hpp:653-718: causal forward, saved activations."""
    cfg = p.config
    d, H = cfg.d_model, cfg.n_heads
    dh = d // H
    scale = F32(1) / np.sqrt(F32(dh))
    rows = x.shape[0]
    causal = np.tril(np.ones((rows, rows), dtype=bool))
    acts = []
    for li in range(p.n_layers):
        w = p.layer(li)
        a = {"x_in": x}
        a["ln1_y"], a["ln1_mu"], a["ln1_rs"] = layernorm(x, w["ln1_g"], w["ln1_b"])
        q = (a["ln1_y"] @ w["wq"]).astype(F32)
        k = (a["ln1_y"] @ w["wk"]).astype(F32)
        v = (a["ln1_y"] @ w["wv"]).astype(F32)
        qh, kh, vh = (t.reshape(rows, H, dh).transpose(1, 0, 2) for t in (q, k, v))
        s = (np.matmul(qh, kh.transpose(0, 2, 1)).astype(F32) * scale).astype(F32)
        s = np.where(causal[None], s, -np.inf)
        P = softmax_rows(s)
        ctx = np.matmul(P, vh).transpose(1, 0, 2).reshape(rows, d).astype(F32)
        a.update(q=q, k=k, v=v, P=P, ctx=ctx)
        a["att_res"] = (ctx @ w["wo"]).astype(F32)
        x = (a["x_in"] + a["att_res"]).astype(F32)
        a["x_mid"] = x
        a["ln2_y"], a["ln2_mu"], a["ln2_rs"] = layernorm(x, w["ln2_g"], w["ln2_b"])
        a["fch"] = (a["ln2_y"] @ w["w1"]).astype(F32)
        a["fgelu"] = gelu(a["fch"])
        x = (x + (a["fgelu"] @ w["w2"]).astype(F32)).astype(F32)
        acts.append(a)
    return x, acts


def _train_blocks_bwd(p: Params, acts, dx: np.ndarray, grads: dict, prefix=""):
    """tinylm.hpp:720-800."""
    cfg = p.config
    d, H = cfg.d_model, cfg.n_heads
    dh = d // H
    scale = F32(1) / np.sqrt(F32(dh))
    for li in range(p.n_layers - 1, -1, -1):
        w, a = p.layer(li), acts[li]
        rows = dx.shape[0]
        g = lambda n: grads[f"l{li}.{n}"]
        g("w2")[...] += (a["fgelu"].T @ dx).astype(F32)
        d_fgelu = (dx @ w["w2"].T).astype(F32)
        d_fch = (d_fgelu * gelu_grad(a["fch"])).astype(F32)
        g("w1")[...] += (a["ln2_y"].T @ d_fch).astype(F32)
        d_ln2 = (d_fch @ w["w1"].T).astype(F32)
        d_xmid, dg, db = layernorm_bwd(a["x_mid"], w["ln2_g"], a["ln2_mu"], a["ln2_rs"], d_ln2)
        g("ln2_g")[...] += dg
        g("ln2_b")[...] += db
        d_xmid = (d_xmid + dx).astype(F32)
        g("wo")[...] += (a["ctx"].T @ d_xmid).astype(F32)
        d_ctx = (d_xmid @ w["wo"].T).astype(F32)
        P = a["P"]
        dch = d_ctx.reshape(rows, H, dh).transpose(1, 0, 2)
        qh, kh, vh = (a[t].reshape(rows, H, dh).transpose(1, 0, 2) for t in ("q", "k", "v"))
        dP = np.matmul(dch, vh.transpose(0, 2, 1)).astype(F32)
        dv = np.matmul(P.transpose(0, 2, 1), dch).astype(F32)
        dot = (dP * P).sum(-1, keepdims=True, dtype=F32)
        dS = (P * (dP - dot) * scale).astype(F32)
        dq = np.matmul(dS, kh).astype(F32)
        dk = np.matmul(dS.transpose(0, 2, 1), qh).astype(F32)
        d_q, d_k, d_v = (t.transpose(1, 0, 2).reshape(rows, d) for t in (dq, dk, dv))
        y1 = a["ln1_y"]
        g("wq")[...] += (y1.T @ d_q).astype(F32)
        g("wk")[...] += (y1.T @ d_k).astype(F32)
        g("wv")[...] += (y1.T @ d_v).astype(F32)
        d_ln1 = (d_q @ w["wq"].T + d_k @ w["wk"].T + d_v @ w["wv"].T).astype(F32)
        d_xin, dg, db = layernorm_bwd(a["x_in"], w["ln1_g"], a["ln1_mu"], a["ln1_rs"], d_ln1)
        g("ln1_g")[...] += dg
        g("ln1_b")[...] += db
        dx = (d_xin + d_xmid).astype(F32)
    return dx


def draft_train_forward(dr: Params, tgt: Params, tokens, prev_features, positions):
    """tinylm.hpp:881-921. Returns (features, logits, acts)."""
    d = dr.config.d_model
    tokens = np.asarray(tokens, dtype=np.int64)
    rows = len(tokens)
    if rows == 0:
        raise ValueError("draft_train_forward: empty input")
    fused = np.concatenate([tgt.t["tok_emb"][tokens], np.asarray(prev_features, F32).reshape(rows, d)], 1)
    x0 = ((fused @ dr.t["w_fuse"]).astype(F32) + tgt.t["pos_emb"][np.asarray(positions)]).astype(F32)
    xf, acts = _train_blocks_fwd(dr, x0)
    feats, mu, rs = layernorm(xf, dr.t["lnf_g"], dr.t["lnf_b"])
    logits = (feats @ tgt.t["lm_head"]).astype(F32)
    return feats, logits, dict(fused=fused, layers=acts, x_final=xf, lnf_mu=mu, lnf_rs=rs)


def draft_train_backward(dr: Params, tgt: Params, acts, dfeatures, dlogits, grad_flat: np.ndarray):
    """tinylm.hpp:923-953 (LM head frozen; d_lnf += dlogits . lm_head^T)."""
    grads = Params(dr.config, dr.specs, grad_flat, dr.n_layers).t
    d_lnf = np.asarray(dfeatures, F32).copy()
    if dlogits is not None:
        d_lnf = (d_lnf + dlogits @ tgt.t["lm_head"].T).astype(F32)
    dx, dg, db = layernorm_bwd(acts["x_final"], dr.t["lnf_g"], acts["lnf_mu"], acts["lnf_rs"], d_lnf)
    grads["lnf_g"][...] += dg
    grads["lnf_b"][...] += db
    dx = _train_blocks_bwd(dr, acts["layers"], dx, grads)
    grads["w_fuse"][...] += (acts["fused"].T @ dx).astype(F32)


def draft_loss_grad(dr: Params, tgt: Params, seqs: Sequence[SeqResult], w_feat=1.0, w_tok=0.1,
                    grad_flat: Optional[np.ndarray] = None, rows_total: Optional[int] = None):
    """grpo.hpp:278-344: SmoothL1(beta=1) on features / (rows*d) * w_feat plus
    CE(next token) / rows * w_tok, teacher-forced pairs (t_j, f_{j-1}), j=1..n-2.

    ``rows_total`` overrides the normaliser (data-parallel shard with a global row count,
    SURVEY.md §8e). Returns (feature_loss, token_loss, total, rows)."""
    d, V = dr.config.d_model, dr.config.vocab_size
    if grad_flat is None:
        grad_flat = np.zeros(dr.flat.size, F32)
    rows_all = sum(max(0, len(s.tokens) - 2) for s in seqs)
    if rows_all == 0 and rows_total is None:
        return 0.0, 0.0, 0.0, 0
    norm = rows_total if rows_total is not None else rows_all
    inv_r = 1.0 / norm
    inv_rd = inv_r / d
    fl = tl = 0.0
    for s in seqs:
        n = len(s.tokens)
        rows = n - 2
        if rows <= 0:
            continue
        toks = np.asarray(s.tokens[1:rows + 1])
        feats = np.asarray(s.features, F32)
        f, lg, acts = draft_train_forward(dr, tgt, toks, feats[:rows], np.arange(1, rows + 1))
        err = f.astype(np.float64) - feats[1:rows + 1].astype(np.float64)
        ae = np.abs(err)
        small = ae <= 1.0
        fl += float(np.sum(np.where(small, w_feat * inv_rd * 0.5 * err * err, w_feat * inv_rd * (ae - 0.5))))
        dfeat = np.where(small, w_feat * inv_rd * err, w_feat * inv_rd * np.sign(err)).astype(F32)
        tgts = np.asarray(s.tokens[2:rows + 2])
        lgd = lg.astype(np.float64)
        mx = lgd.max(1, keepdims=True)
        e = np.exp(lgd - mx)
        sm = e.sum(1, keepdims=True)
        tl += float(np.sum(-w_tok * inv_r * (lgd[np.arange(rows), tgts] - mx[:, 0] - np.log(sm[:, 0]))))
        dlog = (w_tok * inv_r * (e / sm)).astype(F32)
        dlog[np.arange(rows), tgts] -= F32(w_tok * inv_r)
        draft_train_backward(dr, tgt, acts, dfeat, dlog, grad_flat)
    return fl, tl, fl + tl, rows_all


class AdamW:
    """grpo.hpp:97-103, grpo.cpp:142-161 (m, v stored fp32; math in fp64)."""

    def __init__(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
        self.lr, self.beta1, self.beta2, self.eps, self.wd = lr, beta1, beta2, eps, weight_decay
        self.m = self.v = None
        self.t = 0

    def step(self, params: np.ndarray, grad: np.ndarray):
        if params.size != grad.size:
            raise ValueError("adamw: size mismatch")
        if self.m is None or self.m.size != params.size:
            self.m = np.zeros(params.size, F32)
            self.v = np.zeros(params.size, F32)
            self.t = 0
        self.t += 1
        bc1 = 1.0 - self.beta1 ** self.t
        bc2 = 1.0 - self.beta2 ** self.t
        g = grad.astype(np.float64)
        self.m[:] = (self.beta1 * self.m.astype(np.float64) + (1.0 - self.beta1) * g).astype(F32)
        self.v[:] = (self.beta2 * self.v.astype(np.float64) + (1.0 - self.beta2) * g * g).astype(F32)
        mhat = self.m.astype(np.float64) / bc1
        vhat = self.v.astype(np.float64) / bc2
        p = params.astype(np.float64)
        params[:] = (p - self.lr * (mhat / (np.sqrt(vhat) + self.eps) + self.wd * p)).astype(F32)


def draft_update(dr: Params, tgt: Params, seqs: Sequence[SeqResult], opt: AdamW, w_feat=1.0, w_tok=0.1):
    """grpo.cpp:177-186."""
    if not len(seqs):
        return 0.0, 0.0, 0.0, 0
    grad = np.zeros(dr.flat.size, F32)
    terms = draft_loss_grad(dr, tgt, seqs, w_feat, w_tok, grad)
    if terms[3] == 0:
        return terms
    opt.step(dr.flat, grad)
    return terms


# ----------------------------------------------------------------------------------
# Checkpoints -- src/tinylm.cpp:14-105 (SGRPOCK1 + u32 header length + JSON + fp32 LE)
# ----------------------------------------------------------------------------------
def save_checkpoint(path: str, p: Params, kind: str = "target"):
    c = p.config
    hdr = {"kind": kind, "config": {"vocab_size": c.vocab_size, "d_model": c.d_model,
                                     "n_layers": c.n_layers, "n_heads": c.n_heads, "d_ff": c.d_ff,
                                     "max_seq_len": c.max_seq_len, "seed": c.seed}}
    if kind == "draft":
        hdr["draft_layers"] = p.n_layers
    hdr["param_count"] = int(p.flat.size)
    hs = json.dumps(hdr, separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(b"SGRPOCK1" + struct.pack("<I", len(hs)) + hs)
        f.write(np.ascontiguousarray(p.flat, "<f4").tobytes())


def load_checkpoint(path: str):
    """Returns (kind, Params)."""
    with open(path, "rb") as f:
        if f.read(8) != b"SGRPOCK1":
            raise RuntimeError("bad checkpoint magic: " + path)
        (hl,) = struct.unpack("<I", f.read(4))
        hdr = json.loads(f.read(hl))
        n = int(hdr["param_count"])
        flat = np.frombuffer(f.read(4 * n), "<f4").astype(F32)
    if flat.size != n:
        raise RuntimeError("truncated checkpoint: " + path)
    cfg = ModelConfig(**hdr["config"])
    if hdr["kind"] == "draft":
        return "draft", draft_from_flat(cfg, flat, int(hdr["draft_layers"]))
    return "target", model_from_flat(cfg, flat)


# ----------------------------------------------------------------------------------
# Hardware profile: C_peak calibration -- src/roofline.cpp:39-108 (Alg. 2)
# ----------------------------------------------------------------------------------
def detect_knee(curve):
    """roofline.cpp:39-76: normalise both axes to the unit box; the knee is the point
    farthest from the chord first->last; confidence = distance / (sqrt(2)/2), clamped."""
    n = len(curve)
    if n < 4:
        raise ValueError("detect_knee: need at least 4 points")
    xs = [float(b) for b, _ in curve]
    ys = [float(s) for _, s in curve]
    xmin, xmax, ymin, ymax = min(xs), max(xs), min(ys), max(ys)
    xspan = xmax - xmin if xmax > xmin else 1.0
    yspan = ymax - ymin if ymax > ymin else 1.0
    nx = [(x - xmin) / xspan for x in xs]
    ny = [(y - ymin) / yspan for y in ys]
    x0, y0, x1, y1 = nx[0], ny[0], nx[-1], ny[-1]
    cx, cy = x1 - x0, y1 - y0
    clen = math.sqrt(cx * cx + cy * cy)
    best, idx = -1.0, 0
    for i in range(n):
        if clen == 0:
            dist = math.sqrt((nx[i] - x0) ** 2 + (ny[i] - y0) ** 2)
        else:
            dist = abs(cx * (ny[i] - y0) - cy * (nx[i] - x0)) / clen
        if dist > best:
            best, idx = dist, i
    return idx, min(max(best / 0.7071067811865476, 0.0), 1.0)


def measure_c_peak(latency_fn, b_max: int, warmup: int = 1, reps: int = 3):
    """roofline.cpp:78-108: median of `reps` latencies per b = 1..b_max; a >2% drop marks
    low confidence; confidence < 0.05 falls back to c_peak = b_max."""
    if b_max < 4:
        raise ValueError("measure_c_peak: b_max must be >= 4")
    if reps < 1:
        raise ValueError("measure_c_peak: reps must be >= 1")
    curve = []
    for b in range(1, b_max + 1):
        for _ in range(warmup):
            latency_fn(b)
        samples = sorted(latency_fn(b) for _ in range(reps))
        curve.append((b, samples[reps // 2]))
    low = any(curve[i][1] < curve[i - 1][1] * (1.0 - 0.02) for i in range(1, len(curve)))
    idx, conf = detect_knee(curve)
    if conf < 0.05:
        return dict(c_peak=b_max, confidence=conf, low_confidence=True, curve=curve)
    return dict(c_peak=curve[idx][0], confidence=conf, low_confidence=low, curve=curve)


# ----------------------------------------------------------------------------- GRPO rewards
# Task token ids (include/sgrpo/grpo.hpp:19-21) and EOS (tinylm.hpp:41).
K_DIGIT_BASE, K_PLUS, K_EQ, K_EOS = 2, 12, 13, 1


def compute_reward(a: int, b: int, response: Sequence[int]) -> float:
    """compute_reward (src/grpo.cpp:99-116): 1.0 iff the digits after the LAST '=' spell a+b
    (an EOS is allowed only as the very last token), 0.0 for anything malformed."""
    last_eq = -1
    for i, t in enumerate(response):
        if t == K_EQ:
            last_eq = i
    if last_eq < 0:
        return 0.0
    value, digits = 0, 0
    for i in range(last_eq + 1, len(response)):
        t = response[i]
        if t == K_EOS and i + 1 == len(response):
            break
        if t < K_DIGIT_BASE or t >= K_DIGIT_BASE + 10:
            return 0.0
        value = value * 10 + (t - K_DIGIT_BASE)
        digits += 1
        if digits > 15:
            return 0.0
    if digits == 0:
        return 0.0
    return 1.0 if value == a + b else 0.0


def _fma(a: float, b: float, c: float) -> float:
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))  # one rounding


def standardize_advantages(rewards: Sequence[float], eps_var: float):
    """standardize_advantages (src/grpo.cpp:121-136): population-standardized rewards, or None
    (the group is filtered) when sd < eps_var. Sequential fp64 sums as in the reference -- as
    COMPILED (oracle/Makefile, g++ -O3 -march=x86-64-v3): the deviation loop is vectorised
    two/four wide with exact products added in order, and the odd tail element is fused into
    one vfmadd231sd (objdump of grpo.o); pinned bit for bit by tests/golden/rewards.json."""
    g = len(rewards)
    if g < 2:
        raise ValueError("standardize_advantages: need G >= 2")
    mean = 0.0
    for r in rewards:
        mean += float(r)
    mean /= float(g)
    var = 0.0
    for i, r in enumerate(rewards):
        dv = float(r) - mean
        var = _fma(dv, dv, var) if (g % 2 == 1 and i == g - 1) else var + dv * dv
    var /= float(g)
    sd = math.sqrt(var)
    if sd < eps_var:
        return None
    return [(float(r) - mean) / sd for r in rewards]
