"""B200-native re-forwarding training (arXiv 1808.00079).

Host planner (C++, bit-exact with the reference planner) + a re-forward
training executor whose hot path is hand-written sm_100a CUDA, exposed through
the C-ABI in include/reforward_b200.h.
"""
from ._lib import LIB_PATH, load_library  # noqa: F401

__all__ = ["LIB_PATH", "load_library"]
