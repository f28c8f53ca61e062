"""A ``kernels`` backend for the reference's operator-plugin seam, running on the B200.

The reference selects its kernel module at import time (mx4train/_backend/__init__.py:13-35) and
calls it through a duck-typed interface: ``NAME``, ``quantize_rtn``, ``quantize_sr``,
``quantize_quest``, ``fwht``, ``gemm_nt`` (+ the ``*_values`` diagnostics helpers), with numpy in and
numpy out (_native.pyx:104-396).  This module implements that interface on top of
libquartet_b200.so so a maintainer can register it as a third backend:

    quantize_rtn(x f64[R,C], g=32)                    -> (codes u8[R,C], scales u8[R,ceil(C/32)])
    quantize_sr(x, g=32, seed, counter_start)         -> (codes, scales)
    quantize_quest(x, g=32, ratio_lo=1/16)            -> (codes, scales, mask u8[R,C])
    fwht(x f32[R,n], g=32)                            -> f32[R,n]
    gemm_nt(a, b)                                     -> a @ b.T for MXFP4-valued operands

Results are bit-identical to the reference for every input the layer path produces (fp32-valued
matrices).  Restrictions (each raises instead of silently diverging):
  * inputs must be exactly representable in fp32 (the layer path always passes fp32 values);
  * group size 32, ratio_lo 1/16, FWHT block 32 in fp32 (the Quartet configuration);
  * gemm_nt only accepts operands whose rows are MXFP4 grids (dequantized codes, as in
    qlinear.gemm_lp) -- the product then runs on the tcgen05 MXFP4 GEMM.
Ragged trailing groups (C % 32 != 0) are supported by zero padding, which changes no result.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .mxfp4 import GROUP, fwht32, gemm, quant_rows

NAME = "b200"


def _to_f32_exact(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x)
    if x.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    if x.dtype == np.float32:
        return x
    x32 = x.astype(np.float32)
    if not np.array_equal(x32.astype(x.dtype), x, equal_nan=True):
        raise ValueError("b200 backend: input is not exactly representable in fp32")
    return x32


def _check_group(group_size: int) -> None:
    if group_size != GROUP:
        raise NotImplementedError("b200 backend implements group_size = 32 (MXFP4)")


def _pad(x32: np.ndarray):
    rows, cols = x32.shape
    pc = -(-cols // GROUP) * GROUP
    if pc != cols:
        x32 = np.concatenate([x32, np.zeros((rows, pc - cols), np.float32)], axis=1)
    return torch.from_numpy(np.ascontiguousarray(x32)).cuda(), rows, cols


def _finish(op, rows, cols, want_mask=False):
    codes = op.unpacked_codes()[:, :cols].cpu().numpy().astype(np.uint8)
    scales = op.scales_rowmajor()[:, : -(-cols // GROUP)].cpu().numpy().astype(np.uint8)
    if want_mask:
        return codes, scales, op.mask_bool()[:, :cols].cpu().numpy().astype(np.uint8)
    return codes, scales


def quantize_rtn(x: np.ndarray, group_size: int):
    """_native.pyx:104-131"""
    _check_group(group_size)
    if x.size == 0:
        return np.empty(x.shape, np.uint8), np.empty((x.shape[0], -(-x.shape[1] // GROUP)), np.uint8)
    xd, rows, cols = _pad(_to_f32_exact(x))
    return _finish(quant_rows(xd, _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN), rows, cols)


def quantize_sr(x: np.ndarray, group_size: int, seed: int, counter_start: int):
    """_native.pyx:134-168 (stream position counter_start + i*cols + j, original cols)"""
    _check_group(group_size)
    if x.size == 0:
        return np.empty(x.shape, np.uint8), np.empty((x.shape[0], -(-x.shape[1] // GROUP)), np.uint8)
    xd, rows, cols = _pad(_to_f32_exact(x))
    op = quant_rows(xd, _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_SR, sr_seed=seed, counter_start=counter_start,
                    counter_ld=cols)
    return _finish(op, rows, cols)


def quantize_quest(x: np.ndarray, group_size: int, ratio_lo: float):
    """_native.pyx:206-245"""
    _check_group(group_size)
    if ratio_lo != 1.0 / 16.0:
        raise NotImplementedError("b200 backend implements the QuEST clip range (1/16, 1)")
    if x.size == 0:
        return (np.empty(x.shape, np.uint8), np.empty((x.shape[0], -(-x.shape[1] // GROUP)), np.uint8),
                np.empty(x.shape, np.uint8))
    xd, rows, cols = _pad(_to_f32_exact(x))
    return _finish(quant_rows(xd, _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_QUEST, want_mask=True), rows, cols, True)


def fwht(x: np.ndarray, g: int) -> np.ndarray:
    """_native.pyx:353-379 for the Quartet block (g = 32, fp32)."""
    if g != 32 or x.dtype != np.float32:
        raise NotImplementedError("b200 backend implements the fp32 FWHT-32 used by the Quartet layer")
    if x.size == 0:
        return np.empty_like(x)
    if x.shape[1] % 32:
        raise ValueError(f"axis length {x.shape[1]} not divisible by block size 32")
    return fwht32(torch.from_numpy(np.ascontiguousarray(x)).cuda(), _lib.QT_TRANSFORM_HADAMARD).cpu().numpy()


def gemm_nt(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """a @ b.T (gemm_lp's product, qlinear.py:96-111) for MXFP4-valued rows, on tcgen05."""
    a32, b32 = _to_f32_exact(a), _to_f32_exact(b)
    if a32.shape[1] != b32.shape[1]:
        raise ValueError(f"contraction mismatch: {a32.shape[1]} vs {b32.shape[1]}")
    np_out = np.float64 if a.dtype == np.float64 else np.float32
    if a32.size == 0 or b32.size == 0:  # empty rows, columns or contraction: the reference returns zeros
        return np.zeros((a32.shape[0], b32.shape[0]), np_out)
    ad, m, k = _pad(a32)
    n = b32.shape[0]
    if n % GROUP:  # the GEMM epilogue works on 32-column chunks: pad B with zero rows
        b32 = np.concatenate([b32, np.zeros((GROUP - n % GROUP, b32.shape[1]), np.float32)], axis=0)
    bd, _, _ = _pad(b32)
    A = quant_rows(ad, _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    B = quant_rows(bd, _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    if not (torch.equal(A.dequantize(torch.float32), ad) and torch.equal(B.dequantize(torch.float32), bd)):
        raise ValueError("b200 backend gemm_nt: operands are not MXFP4 grids (dequantize-then-matmul inputs)")
    return gemm(A, B, out_dtype=torch.float32)[:, :n].cpu().numpy().astype(np_out)


def _values_from(codes, scales, cols):
    grid = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])
    dec = np.concatenate([grid, -grid])
    s = np.ldexp(1.0, scales.astype(np.int32) - 127)
    return dec[codes] * np.repeat(s, GROUP, axis=1)[:, :cols]


def rtn_values(x: np.ndarray, group_size: int) -> np.ndarray:
    """_native.pyx:248-271"""
    c, s = quantize_rtn(x, group_size)
    return _values_from(c, s, x.shape[1])


def sr_values(x: np.ndarray, group_size: int, seed: int, counter_start: int) -> np.ndarray:
    """_native.pyx:274-301"""
    c, s = quantize_sr(x, group_size, seed, counter_start)
    return _values_from(c, s, x.shape[1])


def quest_values(x: np.ndarray, group_size: int, ratio_lo: float):
    """_native.pyx:304-350"""
    c, s, m = quantize_quest(x, group_size, ratio_lo)
    return _values_from(c, s, x.shape[1]), m
