"""GPU quantizers vs the CPU oracle: bit-exact FP4 codes, E8M0 scales and trust masks.

The oracle (oracle/, pinned to the reference by test_oracle_golden.py) restates
mx4train/_backend/_native.pyx; the GPU kernels are called through the C ABI
(libquartet_b200.so) via paper_2505_14669_b200.mxfp4.
"""

import os

import numpy as np
import pytest
import torch

from gpu_util import assert_operand_equal, bf16_values, op_codes, op_scales, to_dev

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def qt():
    import paper_2505_14669_b200 as qt

    qt.load()
    return qt


def _fp32_inputs():
    z = np.load(os.path.join(GOLDEN, "kernels.npz"))
    out = []
    for i in range(int(z["n"])):
        x = z[f"x{i}"]
        if x.shape[1] % 32:
            x = x[:, : (x.shape[1] // 32) * 32]
        if x.shape[1] == 0:
            continue
        out.append((i, x.astype(np.float32)))
    return out


def _edge_matrix():
    """Grid midpoints, exact grid points, signed zeros, huge/tiny ranges, +-6 saturation."""
    r = np.random.default_rng(5)
    rows = []
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, 6.0, 7.0, 0.0, -0.0, 0.5, 1.0, 1.5, 2.0, 3.0])
    for s in (1.0, 2.0**-3, 2.0**7, 2.0**-120, 2.0**100):
        rows.append(np.concatenate([mids, -mids]) * s)
        rows.append(np.concatenate([np.nextafter(mids, 10), np.nextafter(mids, -10)]) * s)
    rows.append(np.ldexp(1.0, np.arange(-60, 4, 2)))
    rows.append(r.standard_t(df=1.2, size=32) * 1e3)
    rows.append(np.full(32, 1.5 * 2.0**-3))
    rows.append(np.zeros(32))
    m = np.stack(rows).astype(np.float32)
    return m


@pytest.mark.parametrize("rounding", ["quest", "rtn", "sr"])
def test_quantizers_golden_inputs(qt, oracle, rounding):
    L = qt._lib
    inputs = _fp32_inputs() + [("edge", _edge_matrix())]
    for i, x in inputs:
        xd = to_dev(x)
        if rounding == "quest":
            op = qt.quant_rows(xd, L.QT_TRANSFORM_NONE, L.QT_ROUND_QUEST, want_mask=True)
            c, s, m = oracle.quantize_quest(x.astype(np.float64), 32, 1.0 / 16.0)
            assert np.array_equal(op.mask_bool().cpu().numpy(), m.astype(bool)), i
        elif rounding == "rtn":
            op = qt.quant_rows(xd, L.QT_TRANSFORM_NONE, L.QT_ROUND_RTN)
            c, s = oracle.quantize_rtn(x.astype(np.float64), 32)
        else:
            op = qt.quant_rows(xd, L.QT_TRANSFORM_NONE, L.QT_ROUND_SR, sr_seed=1234, counter_start=17)
            c, s = oracle.quantize_sr(x.astype(np.float64), 32, 1234, 17)
        assert_operand_equal(op, c, s, f"{rounding} input {i}")


def test_packed_bytes_equal_reference_layout(qt, oracle):
    """codes bytes == reference pack_nibbles(codes) (element 2k in the low nibble)."""
    L = qt._lib
    x = bf16_values(np.random.default_rng(0).normal(size=(64, 256)).astype(np.float32))
    op = qt.quant_rows(to_dev(x), L.QT_TRANSFORM_NONE, L.QT_ROUND_RTN)
    c, _ = oracle.quantize_rtn(x.astype(np.float64), 32)
    assert np.array_equal(op.codes.cpu().numpy(), oracle.pack_nibbles(c))


@pytest.mark.parametrize("shape", [(2048, 1024), (96, 640), (32, 32)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_forward_quantizer_h32_quest(qt, oracle, shape, dtype):
    """x_h = FWHT32(x) (fp32 butterfly), QuEST: qlinear.py:139-141, 156."""
    r = np.random.default_rng(shape[0] + shape[1])
    x = r.standard_t(df=4, size=shape).astype(np.float32)
    if dtype == torch.bfloat16:
        x = bf16_values(x)
    xd = to_dev(x, dtype)
    fb = torch.zeros(1, dtype=torch.int32, device="cuda")
    op = qt.quant_rows(xd, qt._lib.QT_TRANSFORM_HADAMARD, qt._lib.QT_ROUND_QUEST, want_mask=True, fallbacks=fb)
    xh = oracle.fwht(x, 32)
    c, s, m = oracle.quantize_quest(xh.astype(np.float64), 32, 1.0 / 16.0)
    assert_operand_equal(op, c, s, "fwd quest")
    assert np.array_equal(op.mask_bool().cpu().numpy(), m.astype(bool))
    print("quest exact-search fallbacks:", int(fb.item()), "of", shape[0] * shape[1] // 32)


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
def test_backward_row_quantizer(qt, oracle, rounding):
    """G_q = Q(FWHT(dy * s_xi) * 0.75) (qlinear.py:214, 219, 225)."""
    T, d_out, xi = 256, 384, 7
    dy = bf16_values(np.random.default_rng(1).normal(size=(T, d_out)).astype(np.float32))
    signs = qt.sign_bits(xi, max(T, d_out), "cuda")
    rc = qt._lib.QT_ROUND_RTN if rounding == "rtn" else qt._lib.QT_ROUND_SR
    seed = oracle.derive_seed(xi, 21)
    op = qt.quant_rows(to_dev(dy, torch.bfloat16), qt._lib.QT_TRANSFORM_RANDOMIZED, rc, signs=signs, prescale=0.75,
                       sr_seed=seed)
    gh = oracle.fwht(dy * oracle.signs(xi, 0, d_out), 32) * np.float32(0.75)
    if rounding == "rtn":
        c, s = oracle.quantize_rtn(gh.astype(np.float64), 32)
    else:
        c, s = oracle.quantize_sr(gh.astype(np.float64), 32, seed, 0)
    assert_operand_equal(op, c, s, "bwd rows")


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
@pytest.mark.parametrize("shape", [(256, 384), (160, 96)])
def test_backward_col_quantizer(qt, oracle, rounding, shape):
    """Gt_q = Q(FWHT(dy^T * s_xi) * 0.75) (qlinear.py:234, 239, 245)."""
    T, d_out = shape
    xi = 9
    dy = bf16_values(np.random.default_rng(2).normal(size=(T, d_out)).astype(np.float32))
    signs = qt.sign_bits(xi, max(T, d_out), "cuda")
    rc = qt._lib.QT_ROUND_RTN if rounding == "rtn" else qt._lib.QT_ROUND_SR
    seed = oracle.derive_seed(xi, 23)
    op = qt.quant_cols(to_dev(dy, torch.bfloat16), rc, transform=qt._lib.QT_TRANSFORM_RANDOMIZED, signs=signs,
                       prescale=0.75, sr_seed=seed)
    gt = oracle.fwht(np.ascontiguousarray(dy.T) * oracle.signs(xi, 0, T), 32) * np.float32(0.75)
    if rounding == "rtn":
        c, s = oracle.quantize_rtn(gt.astype(np.float64), 32)
    else:
        c, s = oracle.quantize_sr(gt.astype(np.float64), 32, seed, 0)
    assert_operand_equal(op, c, s, "bwd cols")


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
def test_requant_transpose(qt, oracle, rounding):
    """Xt_q = Q(FWHT(deq(X_q)^T * s_xi) * 0.75) (qlinear.py:207, 235, 240, 246)."""
    T, d_in, xi = 384, 256, 11
    x = bf16_values(np.random.default_rng(3).normal(size=(T, d_in)).astype(np.float32))
    xq = qt.quant_rows(to_dev(x, torch.bfloat16), qt._lib.QT_TRANSFORM_HADAMARD, qt._lib.QT_ROUND_QUEST,
                       want_mask=True)
    signs = qt.sign_bits(xi, T, "cuda")
    rc = qt._lib.QT_ROUND_RTN if rounding == "rtn" else qt._lib.QT_ROUND_SR
    seed = oracle.derive_seed(xi, 24)
    op = qt.quant_cols(xq, rc, transform=qt._lib.QT_TRANSFORM_RANDOMIZED, signs=signs, prescale=0.75, sr_seed=seed)
    xc, xs, _ = oracle.quantize_quest(oracle.fwht(x, 32).astype(np.float64), 32, 1.0 / 16.0)
    xval = oracle.dequantize(xc, xs, 32, np.float32)
    xt = oracle.fwht(np.ascontiguousarray(xval.T) * oracle.signs(xi, 0, T), 32) * np.float32(0.75)
    if rounding == "rtn":
        c, s = oracle.quantize_rtn(xt.astype(np.float64), 32)
    else:
        c, s = oracle.quantize_sr(xt.astype(np.float64), 32, seed, 0)
    assert_operand_equal(op, c, s, "requant-transpose")


def test_sign_bits_match_rng(qt, oracle):
    for xi, n in ((7, 4096), (2**64 - 1, 333), (0, 32)):
        bits = qt.sign_bits(xi, n, "cuda").cpu().numpy().view(np.uint32)
        flips = ((bits[np.arange(n) // 32] >> (np.arange(n) % 32)) & 1).astype(bool)
        assert np.array_equal(flips, oracle.signs(xi, 0, n) < 0)


def test_derive_seed_matches(qt, oracle):
    for parts in ((7, 21), (2**64 - 1, 24), (3, 4, 5)):
        assert qt.derive_seed(*parts) == oracle.derive_seed(*parts)


def test_nonfinite_flag(qt):
    x = torch.zeros(32, 64, device="cuda")
    x[3, 5] = float("nan")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    qt.quant_rows(x, qt._lib.QT_TRANSFORM_HADAMARD, qt._lib.QT_ROUND_QUEST, want_mask=True, err=err)
    assert int(err.item()) == 1
    with pytest.raises(ValueError):
        qt.forward(x, torch.ones(32, 64, device="cuda"))


def test_sr_unbiased_known_answer(qt):
    """test_quantizers.py:43-56: 2.4 at scale 1 rounds to 3 with P = 0.4."""
    n = 200_000
    x = torch.zeros(n, 32, device="cuda")
    x[:, 0] = 6.0
    x[:, 1] = 2.4
    op = qt.quant_rows(x, qt._lib.QT_TRANSFORM_NONE, qt._lib.QT_ROUND_SR, sr_seed=5)
    vals = op.dequantize(torch.float64)[:, 1].cpu().numpy()
    assert set(np.unique(vals)) <= {2.0, 3.0}
    assert abs((vals == 3.0).mean() - 0.4) < 0.005


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
@pytest.mark.parametrize("shape,dtype", [((256, 384), torch.bfloat16), ((160, 96), torch.bfloat16),
                                         ((96, 224), torch.float32)])
def test_dual_dy_quantizer(qt, oracle, rounding, shape, dtype):
    """G_q and G_t from one read of dy (qlinear.py:214-245), both bit-exact."""
    T, d_out = shape
    xi = 13
    dy = r = np.random.default_rng(7).normal(size=(T, d_out)).astype(np.float32)
    if dtype == torch.bfloat16:
        dy = bf16_values(dy)
    signs = qt.sign_bits(xi, max(T, d_out), "cuda")
    rc = qt._lib.QT_ROUND_RTN if rounding == "rtn" else qt._lib.QT_ROUND_SR
    s_r, s_c = oracle.derive_seed(xi, 21), oracle.derive_seed(xi, 23)
    g_op, gt_op = qt.quant_dual(to_dev(dy, dtype), rc, transform=qt._lib.QT_TRANSFORM_RANDOMIZED, signs=signs,
                                prescale=0.75, seed_rows=s_r, seed_cols=s_c)
    gh = oracle.fwht(dy * oracle.signs(xi, 0, d_out), 32) * np.float32(0.75)
    gt = oracle.fwht(np.ascontiguousarray(dy.T) * oracle.signs(xi, 0, T), 32) * np.float32(0.75)
    if rounding == "rtn":
        (c1, s1), (c2, s2) = oracle.quantize_rtn(gh.astype(np.float64), 32), oracle.quantize_rtn(gt.astype(np.float64), 32)
    else:
        (c1, s1) = oracle.quantize_sr(gh.astype(np.float64), 32, s_r, 0)
        (c2, s2) = oracle.quantize_sr(gt.astype(np.float64), 32, s_c, 0)
    assert_operand_equal(g_op, c1, s1, "dual rows")
    assert_operand_equal(gt_op, c2, s2, "dual cols")


@pytest.mark.parametrize("prescale", [1.0, 0.75])
def test_fwht32_bit_exact(qt, oracle, prescale):
    """The packed f32x2 butterfly equals the reference's scalar fp32 butterfly bit for bit."""
    r = np.random.default_rng(17)
    x = (r.standard_t(df=3, size=(4096, 256)) * np.exp(r.normal(size=(4096, 1)))).astype(np.float32)
    signs = qt.sign_bits(5, 256, "cuda")
    got = qt.mxfp4.fwht32(to_dev(x), qt._lib.QT_TRANSFORM_RANDOMIZED, signs, prescale).cpu().numpy()
    ref = oracle.fwht(x * oracle.signs(5, 0, 256), 32) * np.float32(prescale)
    bad = np.argwhere(got.view(np.uint32) != ref.view(np.uint32))
    assert bad.size == 0, (len(bad), bad[:3], got[tuple(bad[0])], ref[tuple(bad[0])])


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("shape", [(96, 160), (320, 96), (256, 384)])
@pytest.mark.parametrize("col_round", ["rtn", "sr"])
@pytest.mark.parametrize("row_round", ["quest", "rtn"])
def test_fused_forward_equals_rows_then_requant(qt, shape, dtype, col_round, row_round):
    """qt_quant_fused (one read of x) == qt_quant_rows followed by qt_quant_cols on the saved operand,
    including partial tiles (rows / cols not multiples of the 128 / 64-row tile)."""
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_cols, quant_fused, quant_rows, sign_bits

    g = torch.Generator(device="cuda").manual_seed(shape[0] + shape[1])
    x = (torch.randn(*shape, device="cuda", generator=g) * 3).to(dtype)
    x[5, :32] = 0  # a zero group
    rr = {"quest": _lib.QT_ROUND_QUEST, "rtn": _lib.QT_ROUND_RTN}[row_round]
    cr = {"rtn": _lib.QT_ROUND_RTN, "sr": _lib.QT_ROUND_SR}[col_round]
    signs = sign_bits(11, shape[0], "cuda", start=64)
    ref_row = quant_rows(x, _lib.QT_TRANSFORM_HADAMARD, rr, want_mask=True)
    ref_col = quant_cols(ref_row, cr, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=signs, prescale=0.75,
                         sr_seed=99, counter_start=64, counter_ld=shape[0] + 64)
    row, col = quant_fused(x, rr, cr, transform=_lib.QT_TRANSFORM_HADAMARD,
                           col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=signs, col_prescale=0.75,
                           col_seed=99, col_counter_start=64, col_counter_ld=shape[0] + 64)
    torch.cuda.synchronize()
    assert torch.equal(row.codes, ref_row.codes)
    assert torch.equal(row.scales_rowmajor(), ref_row.scales_rowmajor())
    assert torch.equal(row.mask, ref_row.mask)
    assert torch.equal(col.codes, ref_col.codes)
    assert torch.equal(col.scales_rowmajor(), ref_col.scales_rowmajor())


def _dual_inputs():
    g = torch.Generator(device="cuda").manual_seed(3)
    yield "gauss", torch.randn(512, 384, device="cuda", generator=g)
    yield "ragged", torch.randn(96, 160, device="cuda", generator=g) * 1e-3
    t = torch.distributions.StudentT(1.0).sample((256, 256)).cuda()
    yield "t1", t
    x = torch.randn(256, 128, device="cuda", generator=g)
    x[:, ::7] *= 1e6
    x[3] = 0
    x[5, :64] = 0.25
    yield "outliers", x
    yield "grid", (torch.randint(-12, 13, (128, 256), device="cuda", generator=g).float() * 0.25)
    yield "wide", torch.randn(128, 128, device="cuda", generator=g) * torch.exp2(
        torch.randint(-60, 60, (128, 128), device="cuda", generator=g).float())
    yield "large", torch.randn(4096, 1024, device="cuda", generator=g)


@pytest.mark.parametrize("case", ["gauss", "ragged", "t1", "outliers", "grid", "wide", "large"])
def test_tensor_core_dual_equals_exact_path(qt, oracle, case):
    """The tcgen05 Hadamard quantizer (checked RTN + exact per-group fallback) is bit-identical to the
    CUDA-core path (itself pinned to the oracle) -- and, for the small cases, to the oracle directly."""
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_dual, sign_bits

    x = dict(_dual_inputs())[case].to(torch.bfloat16)
    R, C = x.shape
    rs, cs = sign_bits(5, C, "cuda"), sign_bits(9, R, "cuda", start=32)
    L = _lib.load()
    fb = torch.zeros(1, dtype=torch.int32, device="cuda")
    outs = []
    for mode in (0, 1):
        L.qt_debug_set_quant(mode, fb.data_ptr())
        try:
            outs.append(quant_dual(x, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs,
                                   col_signs=cs, prescale=0.75))
        finally:
            L.qt_debug_set_quant(0, None)
    torch.cuda.synchronize()
    (g0, gt0), (g1, gt1) = outs
    for a, b in ((g0, g1), (gt0, gt1)):
        assert torch.equal(a.codes, b.codes)
        assert torch.equal(a.scales_rowmajor(), b.scales_rowmajor())
    groups = 2 * R * C // 32
    print(f"{case}: {int(fb.item())} of {groups} groups re-decided exactly")
    if R * C <= 512 * 384:
        xf = x.float().cpu().numpy()
        s_c = np.array(oracle.signs(5, 0, C), np.float32)
        s_r = np.array(oracle.signs(9, 32, R), np.float32)
        gh = oracle.fwht(xf * s_c[None, :], 32) * np.float32(0.75)
        c, s = oracle.quantize_rtn(gh.astype(np.float64), 32)
        assert_operand_equal(g0, c, s, "G")
        gth = oracle.fwht(np.ascontiguousarray(xf.T) * s_r[None, :], 32) * np.float32(0.75)
        c, s = oracle.quantize_rtn(gth.astype(np.float64), 32)
        assert_operand_equal(gt0, c, s, "G_t")


def test_mxf4_export_of_gpu_operand_matches_oracle(qt, oracle):
    """Forward operand quantized on the GPU, exported as the reference's MXF4 container: byte-identical
    to serializing the oracle's QuantizedTensor (codec.py:214-216)."""
    import struct

    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.formats import from_mxf4, to_mxf4, to_msk1
    from paper_2505_14669_b200.mxfp4 import quant_rows

    x = bf16_values(np.random.default_rng(9).normal(size=(256, 192)).astype(np.float32))
    op = quant_rows(to_dev(x, torch.bfloat16), _lib.QT_TRANSFORM_HADAMARD, _lib.QT_ROUND_QUEST, want_mask=True)
    c, s, m = oracle.quantize_quest(oracle.fwht(x, 32).astype(np.float64), 32, 1 / 16)
    packed = (c[:, 0::2] | (c[:, 1::2] << 4)).astype(np.uint8)
    assert to_mxf4(op) == struct.pack("<4sHIIHH", b"MXF4", 1, 256, 192, 32, 0) + packed.tobytes() + s.tobytes()
    assert to_msk1(op)[12:] == np.packbits(m.astype(bool), axis=1, bitorder="little").tobytes()
    back = from_mxf4(to_mxf4(op))
    assert torch.equal(back.codes, op.codes) and torch.equal(back.scales_rowmajor(), op.scales_rowmajor())


@pytest.mark.parametrize("case", ["gauss", "ragged", "t1", "outliers", "grid", "wide", "large"])
def test_tensor_core_quest_forward_equals_exact_path(qt, case):
    """qt_quant_fused with X_q's QuEST search AND X_t's requantization on the tensor cores (checked
    decisions, exact per-group fallback; qt_debug_set_quant mode 3) is bit-identical to the CUDA-core
    fused kernel on adversarial bf16 inputs."""
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_fused, sign_bits

    x = dict(_dual_inputs())[case].to(torch.bfloat16)
    R, C = x.shape
    signs = sign_bits(13, R, "cuda", start=96)
    L = _lib.load()
    fb = torch.zeros(3, dtype=torch.int32, device="cuda")
    outs = []
    for mode in (3, 1):
        L.qt_debug_set_quant(mode, fb.data_ptr())
        try:
            outs.append(quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_HADAMARD,
                                    col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=signs, col_prescale=0.75))
        finally:
            L.qt_debug_set_quant(0, None)
    torch.cuda.synchronize()
    (r0, c0), (r1, c1) = outs
    assert torch.equal(r0.scales_rowmajor(), r1.scales_rowmajor())
    assert torch.equal(r0.codes, r1.codes) and torch.equal(r0.mask, r1.mask)
    assert torch.equal(c0.codes, c1.codes)
    assert torch.equal(c0.scales_rowmajor(), c1.scales_rowmajor())
    print(f"{case}: X_q / X_t groups re-decided exactly {fb.tolist()} of {R * C // 32}")


def test_sign_bits_pair_equals_two_calls(qt):
    from paper_2505_14669_b200.mxfp4 import sign_bits, sign_bits_pair

    for n_a, n_b, s_b in [(4096, 16384, 0), (96, 160, 64), (11008, 2048, 8192), (0, 33, 5)]:
        a, b = sign_bits_pair(12345, n_a, n_b, "cuda", start_b=s_b)
        assert torch.equal(a, sign_bits(12345, n_a, "cuda")) if n_a else a.numel() == 0
        assert torch.equal(b, sign_bits(12345, n_b, "cuda", start=s_b))

