"""The named hot-path entry points of the C ABI (include/quartet_b200.h: qt_quant_fwd_quest, qt_quant_bwd_rows,
qt_quant_bwd_cols, qt_requant_t, qt_gemm_mxf4) called through RAW ctypes -- the 9-call layer path of
INTEGRATION.md section 3, with caller-allocated buffers and no package wrapper -- against the oracle:
operands bit-exact, y / dx / dw within 1e-5 of the oracle's layer (qlinear.py:114-252)."""

import ctypes

import numpy as np
import pytest
import torch

from gpu_util import bf16_values, rel_err

pytestmark = pytest.mark.gpu

V, I64, I32, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64


@pytest.fixture(scope="module")
def L():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200._lib import LIB_PATH

    qt.load()
    lib = ctypes.CDLL(LIB_PATH)   # a second, plain handle: exactly what a foreign caller does
    lib.qt_quant_fwd_quest.argtypes = [V, I32, I64, I64, I32, V, V, V, V, V]
    lib.qt_quant_bwd_rows.argtypes = [V, I32, I64, I64, V, I32, U64, V, V, V, V]
    lib.qt_quant_bwd_cols.argtypes = [V, I32, I64, I64, V, I32, U64, V, V, V, V]
    lib.qt_requant_t.argtypes = [V, V, I64, I64, V, I32, U64, V, V, V, V]
    lib.qt_gemm_mxf4.argtypes = [V, V, V, V, I64, I64, I64, V, I32, I64, I32, V, ctypes.c_float, V]
    lib.qt_sign_bits.argtypes = [V, I64, U64, V]
    lib.qt_sf_bytes.argtypes = [I64, I64]
    lib.qt_sf_bytes.restype = I64
    for f in ("qt_quant_fwd_quest", "qt_quant_bwd_rows", "qt_quant_bwd_cols", "qt_requant_t", "qt_gemm_mxf4",
              "qt_sign_bits"):
        getattr(lib, f).restype = I32
    return lib


class Op:
    """caller-owned MXFP4 buffers of one [rows, k] operand (codes k/2 bytes per row, zeroed scale atoms)"""

    def __init__(self, L, rows, k, mask=False):
        self.rows, self.k = rows, k
        self.codes = torch.empty((rows, k // 2), dtype=torch.uint8, device="cuda")
        self.sf = torch.zeros(int(L.qt_sf_bytes(rows, k)), dtype=torch.uint8, device="cuda")
        self.mask = torch.empty((rows, k // 32), dtype=torch.int32, device="cuda") if mask else None

    def unpacked(self):
        c = self.codes
        return torch.stack([c & 15, c >> 4], -1).reshape(self.rows, self.k).cpu().numpy()

    def scales(self):
        r = torch.arange(self.rows, device="cuda").view(-1, 1)
        g = torch.arange(self.k // 32, device="cuda").view(1, -1)
        katoms = 2 * ((self.k + 255) // 256)
        off = ((r >> 7) * katoms + (g >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (g & 3)
        return self.sf[off].cpu().numpy()


def _p(t):
    return t.data_ptr() if t is not None else None


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
def test_nine_call_layer_through_raw_ctypes(L, oracle, rounding):
    T, d_in, d_out, xi = 256, 384, 128, 5
    r = np.random.default_rng(17)
    x = bf16_values(r.normal(size=(T, d_in)).astype(np.float32))
    w = (r.normal(size=(d_out, d_in)) / 16).astype(np.float32)
    dy = bf16_values(r.normal(size=(T, d_out)).astype(np.float32))
    xd = torch.from_numpy(x).cuda().to(torch.bfloat16)
    wd = torch.from_numpy(w).cuda()
    dyd = torch.from_numpy(dy).cuda().to(torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    rc = 1 if rounding == "rtn" else 2
    err = torch.zeros(1, dtype=torch.int32, device="cuda")

    # forward: X_q, W_q (+ masks), y = X_q W_q^T
    xq, wq = Op(L, T, d_in, mask=True), Op(L, d_out, d_in, mask=True)
    assert L.qt_quant_fwd_quest(_p(xd), 0, T, d_in, 1, _p(xq.codes), _p(xq.sf), _p(xq.mask), _p(err), st) == 0
    assert L.qt_quant_fwd_quest(_p(wd), 1, d_out, d_in, 1, _p(wq.codes), _p(wq.sf), _p(wq.mask), _p(err), st) == 0
    y = torch.empty((T, d_out), dtype=torch.float32, device="cuda")
    assert L.qt_gemm_mxf4(_p(xq.codes), _p(xq.sf), _p(wq.codes), _p(wq.sf), T, d_out, d_in, _p(y), 0, d_out, 0, None,
                          1.0, st) == 0
    # backward: signs along d_out and tokens; G (rows), G_t (cols), W_t, X_t (requant-transpose)
    s_out = torch.empty(((d_out + 31) // 32,), dtype=torch.int32, device="cuda")
    s_tok = torch.empty(((T + 31) // 32,), dtype=torch.int32, device="cuda")
    assert L.qt_sign_bits(_p(s_out), d_out, xi, st) == 0 and L.qt_sign_bits(_p(s_tok), T, xi, st) == 0
    seeds = {tag: oracle.derive_seed(xi, tag) if rounding == "sr" else 0 for tag in (21, 22, 23, 24)}
    g, gt = Op(L, T, d_out), Op(L, d_out, T)
    wt, xt = Op(L, d_in, d_out), Op(L, d_in, T)
    assert L.qt_quant_bwd_rows(_p(dyd), 0, T, d_out, _p(s_out), rc, seeds[21], _p(g.codes), _p(g.sf), _p(err), st) == 0
    assert L.qt_requant_t(_p(wq.codes), _p(wq.sf), d_out, d_in, _p(s_out), rc, seeds[22], _p(wt.codes), _p(wt.sf),
                          _p(err), st) == 0
    assert L.qt_quant_bwd_cols(_p(dyd), 0, T, d_out, _p(s_tok), rc, seeds[23], _p(gt.codes), _p(gt.sf), _p(err),
                               st) == 0
    assert L.qt_requant_t(_p(xq.codes), _p(xq.sf), T, d_in, _p(s_tok), rc, seeds[24], _p(xt.codes), _p(xt.sf),
                          _p(err), st) == 0
    post = float(np.float32(16.0 / 9.0))
    dx = torch.empty((T, d_in), dtype=torch.float32, device="cuda")
    dw = torch.empty((d_out, d_in), dtype=torch.float32, device="cuda")
    assert L.qt_gemm_mxf4(_p(g.codes), _p(g.sf), _p(wt.codes), _p(wt.sf), T, d_in, d_out, _p(dx), 0, d_in, 1,
                          _p(xq.mask), post, st) == 0
    assert L.qt_gemm_mxf4(_p(gt.codes), _p(gt.sf), _p(xt.codes), _p(xt.sf), d_out, d_in, T, _p(dw), 0, d_in, 1,
                          _p(wq.mask), post, st) == 0
    torch.cuda.synchronize()
    assert int(err.item()) == 0

    y_ref, ctx = oracle.forward(x, w)
    dx_ref, dw_ref = oracle.backward(dy, ctx, xi=xi, rounding=rounding)
    ops = {"g": ctx.inter["gq"], "gt": ctx.inter["gtq"], "wt": ctx.inter["wtq"], "xt": ctx.inter["xtq"]}
    np.testing.assert_array_equal(xq.unpacked(), ctx.x_codes)
    np.testing.assert_array_equal(xq.scales(), ctx.x_scales)
    np.testing.assert_array_equal(wq.unpacked(), ctx.w_codes)
    for op, key in ((g, "g"), (gt, "gt"), (wt, "wt"), (xt, "xt")):
        np.testing.assert_array_equal(op.unpacked(), ops[key][0], err_msg=key)
        np.testing.assert_array_equal(op.scales(), ops[key][1], err_msg=key)
    for got, ref, name in ((y, y_ref, "y"), (dx, dx_ref, "dx"), (dw, dw_ref, "dw")):
        assert rel_err(got.cpu().numpy(), ref) <= 1e-5, name
