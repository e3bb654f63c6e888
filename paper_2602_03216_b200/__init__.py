"""B200-native Token Sparse Attention prefill path (arXiv 2602.03216).

The compute path is ``libtsa_b200.so`` (hand-written sm_100a CUDA behind the C
ABI in include/tsa_b200.h); this package binds it and mirrors the reference's
operator API (``ops``) and its multi-GPU head sharding (``dist``).
"""
from .ops import *  # noqa: F401,F403
from .ops import __all__ as _ops_all

__all__ = list(_ops_all)
__version__ = "0.1.0"
