"""Loader for the in-tree native library (libreforward_b200.so).

The product path has no fallback: if the library is missing the import of any
compute entry point fails loudly (build it with ``python -m
paper_1808_00079_b200.build`` or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# RF_LIB_PATH: another build of the same library (A/B timing experiments)
LIB_PATH = os.environ.get("RF_LIB_PATH") or os.path.join(PKG_DIR, "libreforward_b200.so")
_lib = None


def load_library() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"native library missing: {LIB_PATH} (run paper_1808_00079_b200.build)")
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib
