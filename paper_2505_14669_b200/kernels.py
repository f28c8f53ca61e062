"""A ``kernels`` backend for the reference's operator-plugin seam, running on the B200.

The reference selects its kernel module at import time (mx4train/_backend/__init__.py:13-35) and
calls it through a duck-typed interface: ``NAME``, ``quantize_rtn``, ``quantize_sr``,
``quantize_quest``, ``fwht``, ``gemm_nt`` and the ``*_values`` helpers the diagnostics use, with numpy in
and numpy out (_native.pyx:104-396).  This module implements that interface on top of
libquartet_b200.so so a maintainer can register it as a third backend:

    quantize_rtn(x f64[R,C], g)                       -> (codes u8[R,C], scales u8[R,ceil(C/g)])
    quantize_sr(x, g, seed, counter_start)            -> (codes, scales)
    quantize_quest(x, g, ratio_lo)                    -> (codes, scales, mask u8[R,C])
    rtn_values / sr_values / quest_values             -> f64 values (+ mask for QuEST)
    fwht(x f32|f64 [R,n], g)                          -> same dtype [R,n], any power-of-two g dividing n
    gemm_nt(a, b)                                     -> a @ b.T in a's dtype, ascending-k per output

Every entry point runs on the exact seam kernels (csrc/seam.cu: scalar f64 / f32 replays of
_native.pyx, one thread per group / block / output), so results are bit-identical to the reference's
compiled backend for EVERY input it accepts -- f64 values, any group size and clip ratio, ragged
trailing groups, f32 and f64 FWHT at any block size, and the GEMM's fixed summation order at any K.
Inputs follow the reference's typed memoryviews: quantizers take float64 (other float dtypes are
converted exactly first), fwht / gemm_nt keep float32 or float64.  The layer path (qlinear.py) does not
go through this module: it uses the tiled tcgen05 / TMA kernels on bf16 / fp32 device tensors.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .mxfp4 import seam_fwht, seam_gemm_nt, seam_quantize

NAME = "b200"


def _f64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x)
    if x.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    return np.ascontiguousarray(x, dtype=np.float64)


def _dev(x: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _check_group(group_size: int) -> int:
    g = int(group_size)
    if g < 1:
        raise ValueError(f"group_size must be positive, got {group_size}")
    return g


def _quantize(x, group_size, rounding, *, seed=0, counter_start=0, ratio_lo=1.0 / 16.0, values=False):
    g = _check_group(group_size)
    x = _f64(x)
    rows, cols = x.shape
    if x.size == 0:  # the reference returns empty arrays of the right shapes without touching a kernel
        ng = -(-cols // g)
        if values:
            v = np.empty((rows, cols), np.float64)
            return (v, np.empty((rows, cols), np.uint8)) if rounding == _lib.QT_ROUND_QUEST else v
        c, s = np.empty((rows, cols), np.uint8), np.empty((rows, ng), np.uint8)
        return (c, s, np.empty((rows, cols), np.uint8)) if rounding == _lib.QT_ROUND_QUEST else (c, s)
    out = seam_quantize(_dev(x), g, rounding, seed=seed, counter_start=counter_start, ratio_lo=ratio_lo,
                        values=values)
    if isinstance(out, tuple):
        return tuple(t.cpu().numpy() for t in out)
    return out.cpu().numpy()


def quantize_rtn(x: np.ndarray, group_size: int):
    """_native.pyx:104-131"""
    return _quantize(x, group_size, _lib.QT_ROUND_RTN)


def quantize_sr(x: np.ndarray, group_size: int, seed: int, counter_start: int):
    """_native.pyx:134-168 (stream position counter_start + i*cols + j)"""
    return _quantize(x, group_size, _lib.QT_ROUND_SR, seed=seed, counter_start=counter_start)


def quantize_quest(x: np.ndarray, group_size: int, ratio_lo: float):
    """_native.pyx:171-245"""
    return _quantize(x, group_size, _lib.QT_ROUND_QUEST, ratio_lo=ratio_lo)


def rtn_values(x: np.ndarray, group_size: int) -> np.ndarray:
    """_native.pyx:248-271"""
    return _quantize(x, group_size, _lib.QT_ROUND_RTN, values=True)


def sr_values(x: np.ndarray, group_size: int, seed: int, counter_start: int) -> np.ndarray:
    """_native.pyx:274-301"""
    return _quantize(x, group_size, _lib.QT_ROUND_SR, seed=seed, counter_start=counter_start, values=True)


def quest_values(x: np.ndarray, group_size: int, ratio_lo: float):
    """_native.pyx:304-350 -> (values, mask)"""
    return _quantize(x, group_size, _lib.QT_ROUND_QUEST, ratio_lo=ratio_lo, values=True)


def fwht(x: np.ndarray, g: int) -> np.ndarray:
    """_native.pyx:353-379: blockwise orthonormal FWHT of a float32 / float64 matrix, block g."""
    x = np.asarray(x)
    if x.dtype not in (np.float32, np.float64):
        raise TypeError(f"fwht takes float32 or float64 (the reference's fused `real` type), got {x.dtype}")
    if x.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    g = int(g)
    if g < 1 or (g & (g - 1)) != 0:
        raise ValueError(f"block size must be a power of two, got {g}")
    if x.size == 0:
        return np.empty_like(x)
    if x.shape[1] % g:
        raise ValueError(f"axis length {x.shape[1]} not divisible by block size {g}")
    return seam_fwht(_dev(x), g).cpu().numpy()


def gemm_nt(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """_native.pyx:382-396: a @ b.T with c = c + a*b over ascending k per output, in a's dtype."""
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype != b.dtype or a.dtype not in (np.float32, np.float64):
        raise TypeError("gemm_nt takes two float32 or two float64 matrices (the reference's fused `real` type)")
    if a.ndim != 2 or b.ndim != 2:
        raise ValueError("expected 2-D matrices")
    if a.shape[1] != b.shape[1]:
        raise ValueError(f"contraction mismatch: {a.shape[1]} vs {b.shape[1]}")
    m, n = a.shape[0], b.shape[0]
    if m == 0 or n == 0 or a.shape[1] == 0:  # empty output, or an empty contraction: zeros like the reference
        return np.zeros((m, n), a.dtype)
    return seam_gemm_nt(_dev(a), _dev(b)).cpu().numpy()
