"""Shared helpers for the -m gpu parity tests (CUDA path vs the numpy oracle)."""
import numpy as np
import pytest

from oracle import oracle as O

# head dim 64 (the CUDA attention supports dh in {64,128,256}); small enough for the oracle.
SMALL = O.ModelConfig(vocab_size=256, d_model=128, n_layers=2, n_heads=2, d_ff=256, max_seq_len=96, seed=5)
C1 = O.ModelConfig(vocab_size=512, d_model=256, n_layers=2, n_heads=4, d_ff=1024, max_seq_len=192, seed=1)


def capi():
    try:
        from paper_2509_21792_b200 import capi as c
    except ImportError as e:  # the product must never silently fall back
        pytest.fail(f"CUDA library missing: {e}")
    if c.device_count() < 1:
        pytest.fail("no CUDA device visible")
    return c


def make_engine(cfg, max_seqs=16, max_rows=512, k_max=10, l_max=6, seed_models=True):
    c = capi()
    e = c.Engine(cfg, 1, 0, max_seqs, max_rows, k_max, l_max)
    m, d = O.init_model(cfg), O.init_draft(cfg, 1)
    if seed_models:
        e.upload_target(m.flat)
        e.upload_draft(d.flat)
    return e, m, d


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
