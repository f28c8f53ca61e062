"""ctypes binding of libquartet_b200.so (the C ABI in include/quartet_b200.h).

There is no fallback: if the library is missing or cannot be loaded, every op raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# QT_LIB_PATH: load another build of the library (A/B experiments with tools/; never set in production)
LIB_PATH = os.environ.get("QT_LIB_PATH") or os.path.join(HERE, "_build", "libquartet_b200.so")

QT_IN_BF16, QT_IN_F32, QT_IN_MXFP4 = 0, 1, 2
QT_TRANSFORM_NONE, QT_TRANSFORM_HADAMARD, QT_TRANSFORM_RANDOMIZED = 0, 1, 2
QT_ROUND_QUEST, QT_ROUND_RTN, QT_ROUND_SR, QT_ROUND_SR_FAST = 0, 1, 2, 3
QT_EPI_STORE, QT_EPI_MASK_H, QT_EPI_MASK = 0, 1, 2
QT_EPI_ACCUMULATE = 0x10
QT_OUT_F32, QT_OUT_BF16 = 0, 1
QT_ERR_SHAPE, QT_ERR_ALIGN, QT_ERR_ARG, QT_ERR_TMA = 2001, 2002, 2003, 2004

# name -> (restype, argtypes)
_vp, _i32, _i64, _u64, _f32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
SIGNATURES = {
    "qt_abi_version": (_i32, []),
    "qt_error_string": (ctypes.c_char_p, [_i32]),
    "qt_codes_ld": (_i64, [_i64]),
    "qt_sf_katoms": (_i64, [_i64]),
    "qt_sf_bytes": (_i64, [_i64, _i64]),
    "qt_mix64": (_u64, [_u64]),
    "qt_derive_seed": (_u64, [_vp, _i32]),
    "qt_sign_bits": (_i32, [_vp, _i64, _u64, _vp]),
    "qt_sign_bits_at": (_i32, [_vp, _i64, _i64, _u64, _vp]),
    "qt_sign_bits_pair": (_i32, [_vp, _i64, _i64, _vp, _i64, _i64, _u64, _vp]),
    "qt_sign_bits_pair_dev": (_i32, [_vp, _i64, _i64, _vp, _i64, _i64, _vp, _vp]),
    "qt_layer_seeds": (_i32, [_vp, _vp, _i32, _u64, _vp, _i32, _vp]),
    "qt_debug_set_gemm": (None, [_i32]),
    "qt_debug_set_grid": (None, [_i32]),
    "qt_debug_set_quant": (None, [_i32, _vp]),
    "qt_rope": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp, _i32, _i64, _i64, _i64, _vp]),
    "qt_swiglu": (_i32, [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _vp]),
    "qt_cross_entropy": (_i32, [_vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _f32, _i32, _vp]),
    "qt_rmsnorm": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _f32, _i32, _vp]),
    "qt_rmsnorm_res": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i32, _f32, _i32, _vp]),
    "qt_seam_quantize": (_i32, [_vp, _i64, _i64, _i64, _i32, _i32, _u64, _u64, ctypes.c_double, _vp, _vp, _vp, _vp,
                                _vp]),
    "qt_seam_fwht": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp]),
    "qt_seam_gemm_nt": (_i32, [_vp, _vp, _vp, _i32, _i64, _i64, _i64, _vp]),
    "qt_seam_row_sums": (_i32, [_vp, _vp, _i32, _i64, _i64, _vp, _vp]),
    "qt_fwht32": (_i32, [_vp, _vp, _i64, _i64, _i32, _vp, _f32, _vp]),
    "qt_quant_rows": (_i32, [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _f32, _i32, _u64, _u64, _i64,
                             _vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp]),
    "qt_quant_cols": (_i32, [_vp, _i32, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i32, _vp, _f32, _i32,
                             _u64, _u64, _i64, _vp, _i64, _vp, _i64, _vp, _vp]),
    "qt_quant_dual": (_i32, [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _f32, _i32, _u64, _u64, _u64, _u64,
                             _i64, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp]),
    "qt_quant_fused": (_i32, [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _f32, _i32, _u64, _u64, _i64, _vp, _i64, _vp,
                              _i64, _vp, _i32, _vp, _f32, _i32, _u64, _u64, _i64, _vp, _i64, _vp, _i64, _vp, _vp,
                              _vp]),
    "qt_quant_fwd_quest": (_i32, [_vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp]),
    "qt_quant_bwd_rows": (_i32, [_vp, _i32, _i64, _i64, _vp, _i32, _u64, _vp, _vp, _vp, _vp]),
    "qt_quant_bwd_cols": (_i32, [_vp, _i32, _i64, _i64, _vp, _i32, _u64, _vp, _vp, _vp, _vp]),
    "qt_requant_t": (_i32, [_vp, _vp, _i64, _i64, _vp, _i32, _u64, _vp, _vp, _vp, _vp]),
    "qt_gemm_mxf4": (_i32, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _i32, _i64, _i32, _vp, _f32, _vp]),
}

_lib = None


class QuartetError(RuntimeError):
    pass


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise QuartetError(
                f"{LIB_PATH} not built: run `python -m paper_2505_14669_b200.build` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.qt_abi_version() != 1:
            raise QuartetError("libquartet_b200 ABI mismatch")
        _lib = L
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().qt_error_string(rc).decode()
        if rc in (QT_ERR_SHAPE,):
            raise ValueError(f"{what}: {msg}")
        raise QuartetError(f"{what} failed ({rc}): {msg}")
