"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/*.h declares, and
its host-only helpers agree with the oracle.  No compute kernels are launched (no GPU here)."""

import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.build import build

    build()
    return _lib.load()


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        names |= set(re.findall(r"QT_API\s+[\w\s\*]+?\b(qt_\w+)\s*\(", open(h).read()))
    return names


def test_header_declares_entry_points():
    names = _declared()
    for must in ("qt_quant_fwd_quest", "qt_quant_bwd_rows", "qt_quant_bwd_cols", "qt_requant_t", "qt_gemm_mxf4",
                 "qt_quant_rows", "qt_quant_cols", "qt_sign_bits"):
        assert must in names


def test_every_declared_symbol_exported(lib):
    from paper_2505_14669_b200._lib import SIGNATURES

    for name in _declared():
        assert hasattr(lib, name), name
        assert name in SIGNATURES, f"{name} has no ctypes signature"


def test_host_helpers(lib, oracle):
    assert lib.qt_abi_version() == 1
    assert lib.qt_error_string(2001).decode().startswith("shape")
    assert lib.qt_codes_ld(1024) == 512
    assert lib.qt_sf_katoms(640) == 6
    assert lib.qt_sf_bytes(300, 1024) == 2 * 2 * 8 * 512
    arr = (ctypes.c_uint64 * 2)(7, 21)
    assert lib.qt_derive_seed(ctypes.cast(arr, ctypes.c_void_p), 2) == oracle.derive_seed(7, 21)
    assert lib.qt_mix64(12345) == oracle.mix64(12345)


def test_argument_errors_without_gpu(lib):
    # shape / enum validation happens before any CUDA call
    assert lib.qt_quant_rows(None, 0, 33, 4, 33, 0, None, 1.0, 0, 0, 0, 0, None, 16, None, 2, None, None, None,
                             None) == 2001
    assert lib.qt_gemm_mxf4(None, None, None, None, 32, 32, 48, None, 0, 32, 0, None, 1.0, None) == 2001
    assert lib.qt_gemm_mxf4(None, None, None, None, 32, 32, 64, None, 7, 32, 0, None, 1.0, None) == 2003
    assert lib.qt_gemm_mxf4(None, None, None, None, 32, 32, 64, None, 0, 32, 0x13, None, 1.0, None) == 2003  # ACCUMULATE | 3
    assert lib.qt_gemm_mxf4(None, None, None, None, 32, 32, 64, None, 0, 32, 0x11, None, 1.0, None) == 2003  # mask missing


def test_glue_entry_points_reject_bad_shapes(lib):
    """The Llama-loop glue entries validate shapes before touching the device (QT_ERR_SHAPE = 2001)."""
    assert lib.qt_rope(None, None, 64, 2, 10, 64, None, None, 0, 0, 0, 0, None) == 2001      # head_dim % 16
    assert lib.qt_rope(None, None, 65, 2, 16, 64, None, None, 0, 0, 0, 0, None) == 2001      # rows % seq
    assert lib.qt_swiglu(None, None, None, None, None, 7, 0, None) == 2001                   # n % 8
    assert lib.qt_rmsnorm(None, None, None, None, None, None, 8, 100, 1e-6, 0, None) == 2001  # d % 8
    assert lib.qt_rmsnorm(None, None, None, None, None, None, 8, 10240, 1e-6, 0, None) == 2001
    assert lib.qt_cross_entropy(None, None, 8, 7, None, None, None, None, 1.0, 0, None) == 2001


def test_empty_dimensions_are_no_ops(lib):
    """An empty row / column / token dimension is valid (the reference accepts batch = 0): the entry points
    return 0 before reading any pointer -- the sign vector of an empty dimension is legitimately null."""
    assert lib.qt_quant_rows(None, 0, 32, 0, 32, 2, None, 1.0, 0, 0, 0, 0, None, 16, None, 2, None, None, None,
                             None) == 0
    assert lib.qt_fwht32(None, None, 0, 64, 2, None, 1.0, None) == 0
    assert lib.qt_gemm_mxf4(None, None, None, None, 0, 32, 64, None, 0, 32, 1, None, 1.0, None) == 0   # M = 0
    assert lib.qt_gemm_mxf4(None, None, None, None, 32, 32, 0, None, 0, 32, 0x11, None, 1.0, None) == 0  # D += 0
    assert lib.qt_gemm_mxf4(None, None, None, None, -32, 32, 64, None, 0, 32, 0, None, 1.0, None) == 2001


def test_layer_rejects_unsupported_output_dtypes():
    """The GEMM epilogues store bf16 / fp32 only: other dtypes raise before any device work (no
    out-of-bounds write into a 2-byte fp16 buffer)."""
    import torch

    import paper_2505_14669_b200 as qt

    x = torch.zeros(32, 32)
    with pytest.raises(ValueError, match="out_dtype"):
        qt.forward(x, x, out_dtype=torch.float16)
    with pytest.raises(ValueError, match="out_dtype"):
        qt.forward(x, x, out_dtype=torch.float64)
    ctx = qt.LayerContext(x_q=None, w_q=None, scheme=qt.QUEST, policy=qt.DEFAULT_POLICY, hadamard=True, batch=32,
                          d_in=32, d_out=32)
    with pytest.raises(ValueError, match="dx_dtype"):
        qt.backward(x, ctx, xi=1, dx_dtype=torch.float16)
    with pytest.raises(ValueError, match="dw_dtype"):
        qt.backward(x, ctx, xi=1, dw_dtype=torch.float16)
