"""B200-native GRPO-rollout hot path of arXiv 2509.21792 (FastGRPO).

The product is libsgrpo_b200.so (hand-written sm_100a kernels + the C++ engine behind
the C-ABI in include/sgrpo_b200.h). This package only builds it and binds it.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libsgrpo_b200.so")


def load():
    """Import the ctypes binding; raises ImportError if the CUDA library is missing."""
    from . import capi  # noqa: F401
    return capi
