"""Oracle parity on the persistent multi-tile paths the bench runs.

At the shapes of the other parity tests every CTA of the persistent kernels gets at most one tile, so
the code that only runs when a CTA walks several tiles -- the double-buffered k_quant loop and its
barrier structure, the k_tcq_dual stage / TMEM-buffer reuse across tiles, the GEMMs' TMEM accumulator
hand-off and operand-ring phases -- would never be compared with the oracle.  qt_debug_set_grid(n) caps
every persistent grid at n CTAs (the 2-CTA GEMM at n/2 pairs, at least one), so with n in {1, 3, 7} each
CTA walks tens to hundreds of tiles.  Everything is checked against the oracle (pinned to the
reference in test_oracle_golden.py): operands bit-exact, GEMM outputs within the stated tolerances.
"""

import os

import numpy as np
import pytest
import torch

from gpu_util import assert_operand_equal, bf16_values, rel_err, to_dev

pytestmark = pytest.mark.gpu
TOL = 1e-5
CAPS = [1, 3, 7]


@pytest.fixture(scope="module")
def qt():
    import paper_2505_14669_b200 as qt

    qt.load()
    return qt


@pytest.fixture(params=CAPS, ids=[f"grid{n}" for n in CAPS])
def grid(qt, request):
    L = qt._lib.load()
    L.qt_debug_set_grid(request.param)
    yield request.param
    torch.cuda.synchronize()
    L.qt_debug_set_grid(0)


_C1 = {}


def _config1(oracle, rounding):
    """BASELINE config 1 (2048 tokens, 1024 x 1024) through the oracle, cached per rounding."""
    if rounding not in _C1:
        T, d_in, d_out, xi = 2048, 1024, 1024, 7
        x = bf16_values(oracle.gaussians(1, oracle.DOMAIN_GAUSS, 0, T * d_in).reshape(T, d_in).astype(np.float32))
        w = bf16_values((oracle.gaussians(2, oracle.DOMAIN_GAUSS, 0, d_out * d_in) / 32.0)
                        .reshape(d_out, d_in).astype(np.float32))
        dy = bf16_values(oracle.gaussians(3, oracle.DOMAIN_GAUSS, 0, T * d_out).reshape(T, d_out)
                         .astype(np.float32))
        oracle.set_threads(os.cpu_count() or 1)
        try:
            y, octx = oracle.forward(x, w)
            dx, dw = oracle.backward(dy, octx, xi=xi, rounding=rounding)
        finally:
            oracle.set_threads(1)
        _C1[rounding] = (x, w, dy, xi, y, octx, dx, dw)
    return _C1[rounding]


@pytest.mark.parametrize("eager", [False, True], ids=["lazy", "eager"])
@pytest.mark.parametrize("rounding", ["rtn", "sr"])
def test_config1_multitile(qt, oracle, grid, rounding, eager):
    x, w, dy, xi, y_ref, octx, dx_ref, dw_ref = _config1(oracle, rounding)
    kw = dict(bwd_xi=xi, bwd_rounding=rounding) if eager else {}
    y, ctx = qt.forward(to_dev(x, torch.bfloat16), to_dev(w, torch.bfloat16), **kw)
    assert_operand_equal(ctx.x_q, octx.x_codes, octx.x_scales, "X_q")
    assert_operand_equal(ctx.w_q, octx.w_codes, octx.w_scales, "W_q")
    assert np.array_equal(ctx.m_x.cpu().numpy(), octx.m_x)
    assert np.array_equal(ctx.m_w.cpu().numpy(), octx.m_w)
    dx, dw, ops = qt.backward(to_dev(dy, torch.bfloat16), ctx, xi=xi, rounding=rounding, return_operands=True)
    for name, key in (("g_q", "gq"), ("wt_q", "wtq"), ("gt_q", "gtq"), ("xt_q", "xtq")):
        c, s = octx.inter[key]
        assert_operand_equal(ops[name], c, s, name)
    for got, ref, what in ((y, y_ref, "y"), (dx, dx_ref, "dx"), (dw, dw_ref, "dw")):
        e = rel_err(got.cpu().numpy(), ref)
        assert e <= TOL, (what, e)


def _mat(seed, shape, kind="t4"):
    r = np.random.default_rng(seed)
    x = r.standard_t(df=4, size=shape) if kind == "t4" else r.normal(size=shape)
    x = x * np.exp2(r.integers(-8, 8, size=(shape[0], 1)))   # per-row magnitudes: varied scales per tile
    return x.astype(np.float32)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_forward_fused_multitile(qt, oracle, grid, dtype):
    """qt_quant_fused (X_q + M_x + X_t from one read; the CUDA-core k_quant double-buffered loop without the
    trailing barrier) vs the oracle's QuEST(H32 x) and Q(H32(deq(X_q)^T (.) s) * 0.75), RTN and SR."""
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_fused, sign_bits

    R, C = 1024, 768
    x = _mat(R + C, (R, C))
    if dtype == torch.bfloat16:
        x = bf16_values(x)
    xi = 21
    signs = sign_bits(xi, R, "cuda", start=64)
    xc, xs, m = oracle.quantize_quest(oracle.fwht(x, 32).astype(np.float64), 32, 1.0 / 16.0)
    xval = oracle.dequantize(xc, xs, 32, np.float32)
    xt = oracle.fwht(np.ascontiguousarray(xval.T) * oracle.signs(xi, 64, R), 32) * np.float32(0.75)
    for cr, name in ((_lib.QT_ROUND_RTN, "rtn"), (_lib.QT_ROUND_SR, "sr")):
        row, col = quant_fused(to_dev(x, dtype), _lib.QT_ROUND_QUEST, cr, transform=_lib.QT_TRANSFORM_HADAMARD,
                               col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=signs, col_prescale=0.75,
                               col_seed=99, col_counter_start=64, col_counter_ld=R + 64)
        assert_operand_equal(row, xc, xs, f"X_q {name}")
        assert np.array_equal(row.mask_bool().cpu().numpy(), m.astype(bool))
        if name == "rtn":
            c, s = oracle.quantize_rtn(xt.astype(np.float64), 32)
        else:  # shard stream: row c of X_t draws positions 64 + c * (R + 64) + j (a slice of a larger matrix)
            c = np.empty(xt.shape, np.uint8)
            s = np.empty((xt.shape[0], xt.shape[1] // 32), np.uint8)
            for i in range(xt.shape[0]):
                c[i:i + 1], s[i:i + 1] = oracle.quantize_sr(xt[i:i + 1].astype(np.float64), 32, 99, 64 + i * (R + 64))
        assert_operand_equal(col, c, s, f"X_t {name}")


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
@pytest.mark.parametrize("mode", [0, 1], ids=["tensor_core", "cuda_core"])
def test_dual_multitile(qt, oracle, grid, rounding, mode):
    """G_q and G_t from one read of dy: the k_tcq_dual stage/TMEM reuse (mode 0, RTN) and the CUDA-core
    k_quant dual loop (mode 1, and SR) against the oracle."""
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_dual, sign_bits

    T, d_out, xi = 1024, 640, 5
    dy = bf16_values(_mat(11, (T, d_out), "normal"))
    rs, cs = sign_bits(xi, d_out, "cuda"), sign_bits(xi, T, "cuda")
    rc = _lib.QT_ROUND_RTN if rounding == "rtn" else _lib.QT_ROUND_SR
    s_r, s_c = oracle.derive_seed(xi, 21), oracle.derive_seed(xi, 23)
    L = _lib.load()
    L.qt_debug_set_quant(mode, None)
    try:
        g_op, gt_op = quant_dual(to_dev(dy, torch.bfloat16), rc, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs,
                                 col_signs=cs, prescale=0.75, seed_rows=s_r, seed_cols=s_c)
        torch.cuda.synchronize()
    finally:
        L.qt_debug_set_quant(0, None)
    gh = oracle.fwht(dy * oracle.signs(xi, 0, d_out), 32) * np.float32(0.75)
    gt = oracle.fwht(np.ascontiguousarray(dy.T) * oracle.signs(xi, 0, T), 32) * np.float32(0.75)
    if rounding == "rtn":
        (c1, s1), (c2, s2) = oracle.quantize_rtn(gh.astype(np.float64), 32), oracle.quantize_rtn(gt.astype(np.float64), 32)
    else:
        c1, s1 = oracle.quantize_sr(gh.astype(np.float64), 32, s_r, 0)
        c2, s2 = oracle.quantize_sr(gt.astype(np.float64), 32, s_c, 0)
    assert_operand_equal(g_op, c1, s1, "G")
    assert_operand_equal(gt_op, c2, s2, "G_t")


def test_requant_multitile(qt, oracle, grid):
    """Lazy requantization of a saved MXFP4 operand (k_quant<MXFP4>, codes-sourced col pass)."""
    from paper_2505_14669_b200 import _lib

    T, d_in, xi = 1024, 512, 3
    x = bf16_values(_mat(5, (T, d_in)))
    xq = qt.quant_rows(to_dev(x, torch.bfloat16), _lib.QT_TRANSFORM_HADAMARD, _lib.QT_ROUND_QUEST, want_mask=True)
    signs = qt.sign_bits(xi, T, "cuda")
    op = qt.quant_cols(xq, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=signs, prescale=0.75)
    xc, xs, _ = oracle.quantize_quest(oracle.fwht(x, 32).astype(np.float64), 32, 1.0 / 16.0)
    xt = oracle.fwht(np.ascontiguousarray(oracle.dequantize(xc, xs, 32, np.float32).T) * oracle.signs(xi, 0, T),
                     32) * np.float32(0.75)
    c, s = oracle.quantize_rtn(xt.astype(np.float64), 32)
    assert_operand_equal(op, c, s, "X_t (lazy)")


@pytest.mark.parametrize("mnk,epi", [((1024, 1024, 2048), "store"), ((1024, 768, 1024), "mask_h"),
                                     ((768, 640, 1536), "mask_h"), ((512, 1024, 4096), "store")])
def test_gemm_multitile(qt, oracle, grid, mnk, epi):
    """Each CTA (pair) walks many output tiles: TMEM accumulator hand-off, operand-ring phases and scale-set
    rotation across tiles.  N = 640 takes the 1-CTA kernel, the others the 2-CTA pair kernel.  Tolerance:
    relative Frobenius error vs the float64 product <= max(4 x the reference fp32 loop's, 1e-6)."""
    from paper_2505_14669_b200 import _lib

    M, N, K = mnk
    a = bf16_values(_mat(M + K, (M, K), "normal"))
    b = bf16_values(_mat(N + K, (N, K)))
    A = qt.quant_rows(to_dev(a), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(to_dev(b), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    ac, as_ = oracle.quantize_rtn(a.astype(np.float64), 32)
    bc, bs = oracle.quantize_rtn(b.astype(np.float64), 32)
    ad, bd = oracle.dequantize(ac, as_, 32), oracle.dequantize(bc, bs, 32)
    prod = ad @ bd.T
    ref32 = oracle.gemm_nt(ad.astype(np.float32), bd.astype(np.float32))
    if epi == "store":
        got = qt.gemm(A, B).cpu().numpy()
        exact = prod
        e_ref = rel_err(ref32, exact)
    else:  # qlinear.py:229-230: H32(D (.) mask) * 16/9
        mask = torch.randint(0, 2**31 - 1, (M, N // 32), dtype=torch.int32, device="cuda") | 0x0F0F0F0F
        mbits = ((mask.cpu().numpy().view(np.uint32)[:, :, None] >> np.arange(32)) & 1).reshape(M, N).astype(bool)
        scale = np.float32(16.0 / 9.0)
        got = qt.gemm(A, B, mask=mask, hadamard=True, scale=float(scale)).cpu().numpy()
        exact = oracle.fwht(prod * mbits, 32).astype(np.float64) * float(scale)
        e_ref = rel_err(oracle.fwht((ref32 * mbits).astype(np.float32), 32) * scale, exact)
    e = rel_err(got, exact)
    assert e <= max(4 * e_ref, 1e-6), (e, e_ref)


_C3 = {}


def _config3_slice(oracle, T, d_in, d_out, rounding):
    """A T-token slice of a BASELINE configs[2] shape (SURVEY 8d inputs: x, dy ~ N(0,1) bf16, W ~ N(0, 1/d_in))
    through the oracle on all host threads, cached."""
    key = (T, d_in, d_out, rounding)
    if key not in _C3:
        r = np.random.default_rng(d_in * 7 + d_out)
        x = bf16_values(r.standard_normal((T, d_in), dtype=np.float32))
        w = bf16_values((r.standard_normal((d_out, d_in), dtype=np.float32) / np.float32(np.sqrt(d_in))))
        dy = bf16_values(r.standard_normal((T, d_out), dtype=np.float32))
        xi = 1000 + d_out
        oracle.set_threads(os.cpu_count() or 1)
        try:
            y, octx = oracle.forward(x, w)
            dx, dw = oracle.backward(dy, octx, xi=xi, rounding=rounding)
        finally:
            oracle.set_threads(1)
        _C3[key] = (x, w, dy, xi, y, octx, dx, dw)
    return _C3[key]


@pytest.mark.parametrize("eager", [False, True], ids=["lazy", "eager"])
@pytest.mark.parametrize("rounding", ["rtn", "sr"])
@pytest.mark.parametrize("shape", [(4096, 4096), (4096, 11008), (11008, 4096)], ids=["4096x4096", "4096x11008",
                                                                                   "11008x4096"])
@pytest.mark.parametrize("T", [256, 512])
def test_config3_slices_against_oracle(qt, oracle, T, shape, rounding, eager):
    """configs[2] (Llama-7B widths) at 256- and 512-token slices, production grid: the bench's kernels at the
    bench's widths against the oracle -- every operand bit-exact, y / dx / dw <= 1e-5."""
    if T == 512 and (rounding, eager) != ("rtn", True):
        pytest.skip("512-token slice: the bench's own mode (RTN, eager) only")
    d_in, d_out = shape
    x, w, dy, xi, y_ref, octx, dx_ref, dw_ref = _config3_slice(oracle, T, d_in, d_out, rounding)
    kw = dict(bwd_xi=xi, bwd_rounding=rounding) if eager else {}
    y, ctx = qt.forward(to_dev(x, torch.bfloat16), to_dev(w, torch.bfloat16), **kw)
    assert_operand_equal(ctx.x_q, octx.x_codes, octx.x_scales, "X_q")
    assert_operand_equal(ctx.w_q, octx.w_codes, octx.w_scales, "W_q")
    assert np.array_equal(ctx.m_x.cpu().numpy(), octx.m_x)
    assert np.array_equal(ctx.m_w.cpu().numpy(), octx.m_w)
    dx, dw, ops = qt.backward(to_dev(dy, torch.bfloat16), ctx, xi=xi, rounding=rounding, return_operands=True)
    for name, key in (("g_q", "gq"), ("wt_q", "wtq"), ("gt_q", "gtq"), ("xt_q", "xtq")):
        c, s = octx.inter[key]
        assert_operand_equal(ops[name], c, s, name)
    for got, ref, what in ((y, y_ref, "y"), (dx, dx_ref, "dx"), (dw, dw_ref, "dw")):
        e = rel_err(got.cpu().numpy(), ref)
        assert e <= TOL, (what, e)
