"""ctypes binding of the rfx_* kernel entry points (include/reforward_b200_exec.h).

Device memory comes from torch (plumbing only); every compute call goes
through libreforward_b200.so.  There is no CPU or torch fallback: a missing
library raises ImportError, a failing launch raises RuntimeError.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from ._lib import load_library

KMAJOR, MNMAJOR, IM2COL_K, IM2COL_MN = 0, 1, 2, 3


class ConvGeom(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("N", "H", "W", "C", "P", "Q", "R", "S", "pad_h", "pad_w", "stride_h", "stride_w")]


class GemmArgs(C.Structure):
    _fields_ = [("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
                ("a_kind", C.c_int32), ("a", C.c_void_p), ("a_ld", C.c_int64), ("a_geom", ConvGeom),
                ("b_kind", C.c_int32), ("b", C.c_void_p), ("b_ld", C.c_int64), ("b_geom", ConvGeom),
                ("out", C.c_void_p), ("ldc", C.c_int64), ("out_f32", C.c_int32), ("accumulate_out", C.c_int32),
                ("bias", C.c_void_p), ("stats", C.c_void_p), ("splits", C.c_int32), ("split_stride", C.c_int64),
                ("remap", C.c_int32), ("rP", C.c_int32), ("rQ", C.c_int32), ("rH", C.c_int32), ("rW", C.c_int32),
                ("rsh", C.c_int32), ("rsw", C.c_int32), ("block_n", C.c_int32), ("b_extent", C.c_int64),
                ("b_taps", C.c_int32), ("b_cpad", C.c_int32), ("b_rows", C.c_int32), ("band", C.c_int32),
                ("b_tap_map", C.c_int32), ("b_tap_base", C.c_int32), ("b_tap_dr", C.c_int32),
                ("b_tap_ds", C.c_int32), ("stats_bwd", C.c_int32), ("replay", C.c_int32), ("bs_y", C.c_void_p),
                ("bs_ldy", C.c_int64), ("bs_mean", C.c_void_p), ("bs_scale", C.c_void_p), ("bs_shift", C.c_void_p),
                ("pair", C.c_int32)]


def conv_geom(N, H, W, Cin, R, S, pad, stride) -> ConvGeom:
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    return ConvGeom(N, H, W, Cin, P, Q, R, S, pad, pad, stride, stride)


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = load_library()
        _lib.rfx_gemm.restype = C.c_int
        _lib.rfx_gemm.argtypes = [C.POINTER(GemmArgs), C.c_void_p]
        _lib.rfx_im2col.restype = C.c_int
        _lib.rfx_im2col.argtypes = [C.c_void_p] + [C.c_int] * 12 + [C.c_void_p, C.c_void_p]
        _lib.rfx_maxpool_bwd.restype = C.c_int
        _lib.rfx_maxpool_bwd.argtypes = [C.c_void_p, C.c_void_p] + [C.c_int] * 7 + [C.c_void_p, C.c_int, C.c_void_p,
                                                                                     C.c_void_p]
        _lib.rf_last_error.restype = C.c_char_p
    return _lib


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def gemm(args: GemmArgs, stream=None) -> None:
    L = lib()
    rc = L.rfx_gemm(C.byref(args), stream_handle(stream))
    if rc != 0:
        raise RuntimeError(L.rf_last_error().decode())


def im2col(x: torch.Tensor, C_real: int, R: int, S: int, stride: int, pad: int, kpad: int, out: torch.Tensor = None,
           stream=None) -> torch.Tensor:
    """Explicit im2col of an NHWC bf16 input with C_real of its x.shape[3]
    channels: [N*P*Q][kpad], K order (r, s, c), zero padded."""
    N, H, W, Cs = x.shape
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    if out is None:
        out = torch.empty(N * P * Q, kpad, dtype=torch.bfloat16, device=x.device)
    L = lib()
    rc = L.rfx_im2col(x.data_ptr(), N, H, W, C_real, Cs, P, Q, R, S, stride, pad, kpad, out.data_ptr(),
                      stream_handle(stream))
    if rc != 0:
        raise RuntimeError(L.rf_last_error().decode())
    return out


def maxpool_bwd(x: torch.Tensor, dy: torch.Tensor, k: int, stride: int, pad: int, dx: torch.Tensor = None,
                accumulate: bool = False, stream=None) -> torch.Tensor:
    """Max-pool backward of an NHWC bf16 input (first-argmax ties, fixed-order sums)."""
    N, H, W, Cc = x.shape
    if dx is None:
        dx = torch.zeros_like(x)
    ws = torch.empty(dy.numel(), dtype=torch.uint8, device=x.device)
    L = lib()
    rc = L.rfx_maxpool_bwd(x.data_ptr(), dy.data_ptr(), N, H, W, Cc, k, stride, pad, dx.data_ptr(),
                           1 if accumulate else 0, ws.data_ptr(), stream_handle(stream))
    if rc != 0:
        raise RuntimeError(L.rf_last_error().decode())
    return dx
