"""tcgen05 MXFP4 GEMM vs the reference's dequantize-then-matmul (gemm_lp, qlinear.py:96-111).

Tolerance (stated): the GPU accumulates the exact FP4 x FP4 x E8M0 products in fp32 in a different
order than the reference's sequential fp32 loop, so results are compared with a relative Frobenius
error against the float64 product of the dequantized operands:
    err(GPU) <= max(4 * err(reference fp32 loop), 1e-6).
"""

import numpy as np
import pytest
import torch

from gpu_util import bf16_values, rel_err, to_dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qt():
    import paper_2505_14669_b200 as qt

    qt.load()
    return qt


def _operand(qt, x: np.ndarray):
    return qt.quant_rows(to_dev(x), qt._lib.QT_TRANSFORM_NONE, qt._lib.QT_ROUND_RTN)


def _check(qt, oracle, a, b, out_dtype=torch.float32):
    A, B = _operand(qt, a), _operand(qt, b)
    got = qt.gemm(A, B, out_dtype=out_dtype).float().cpu().numpy()
    ac, as_ = oracle.quantize_rtn(a.astype(np.float64), 32)
    bc, bs = oracle.quantize_rtn(b.astype(np.float64), 32)
    ad, bd = oracle.dequantize(ac, as_, 32), oracle.dequantize(bc, bs, 32)
    exact = ad @ bd.T
    ref32 = oracle.gemm_nt(ad.astype(np.float32), bd.astype(np.float32))
    e_gpu, e_ref = rel_err(got, exact), rel_err(ref32, exact)
    tol = max(4 * e_ref, 1e-6) if out_dtype == torch.float32 else 4e-3
    assert e_gpu <= tol, (e_gpu, e_ref, a.shape, b.shape)
    return e_gpu, e_ref


def test_gemm_identity_like(qt):
    """test_qlinear.py:146-149: quantize(6 I) squared is 36 I exactly."""
    q6 = qt.quant_rows(torch.eye(32, device="cuda") * 6.0, qt._lib.QT_TRANSFORM_NONE, qt._lib.QT_ROUND_RTN)
    out = qt.gemm(q6, q6).cpu().numpy()
    assert np.array_equal(out, 36.0 * np.eye(32))


def test_gemm_structured_scales(qt):
    """Per-row / per-column / per-group scales land in the right place (SF layout check)."""
    M, N, K = 256, 256, 512
    a = np.zeros((M, K), np.float32)
    b = np.zeros((N, K), np.float32)
    r = np.random.default_rng(0)
    # group-constant powers of two: exact in MXFP4, every partial sum exact in fp32 (< 2^17 span)
    a[:] = np.ldexp(1.0, (np.arange(M)[:, None] % 3) - 1 + (np.arange(K)[None, :] // 32) % 2)
    b[:] = np.ldexp(1.0, (np.arange(N)[:, None] % 3) - 1 + (np.arange(K)[None, :] // 32) % 3)
    a *= r.choice([-1.0, 1.0], size=a.shape)
    b *= r.choice([-1.0, 1.0], size=b.shape)
    A, B = _operand(qt, a), _operand(qt, b)
    got = qt.gemm(A, B).cpu().numpy()
    exact = a.astype(np.float64) @ b.astype(np.float64).T   # powers of two are exact in MXFP4
    assert np.array_equal(got, exact)


@pytest.mark.parametrize("mnk", [(128, 256, 256), (256, 512, 1024), (2048, 1024, 1024), (96, 160, 640),
                                 (300, 96, 96), (1024, 1152, 2048),
                                 # 2-CTA pair kernel: M not a multiple of 256 (clipped rows of the second CTA's
                                 # TMA-stored boxes), K not a multiple of 256 (zero-filled last K tile), one pair
                                 (288, 512, 640), (640, 768, 1184), (256, 256, 32)])
def test_gemm_random(qt, oracle, mnk):
    M, N, K = mnk
    r = np.random.default_rng(M + N + K)
    a = bf16_values(r.normal(size=(M, K)).astype(np.float32))
    b = bf16_values(r.standard_t(df=3, size=(N, K)).astype(np.float32))
    e_gpu, e_ref = _check(qt, oracle, a, b)
    print(f"gemm {mnk}: rel err gpu {e_gpu:.3e} ref-fp32 {e_ref:.3e}")


@pytest.mark.parametrize("mn", [(288, 512), (1024, 768)])
def test_gemm_masked_epilogue_fp32_and_bf16_paths_agree(qt, mn):
    """The staged (TMA-store) epilogue writes the same values in fp32 and bf16 (bf16 = RNE of the fp32)
    for the masked FWHT . 16/9 epilogue, including clipped edge rows."""
    M, N = mn
    K = 512
    g = torch.Generator(device="cuda").manual_seed(M)
    from paper_2505_14669_b200 import _lib

    A = qt.quant_rows(torch.randn(M, K, device="cuda", generator=g), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(torch.randn(N, K, device="cuda", generator=g), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    mask = torch.randint(-2**31, 2**31 - 1, (M, N // 32), device="cuda", dtype=torch.int32, generator=g)
    f32 = qt.gemm(A, B, mask=mask, hadamard=True, scale=16 / 9)
    b16 = qt.gemm(A, B, mask=mask, hadamard=True, scale=16 / 9, out_dtype=torch.bfloat16)
    assert torch.equal(f32.to(torch.bfloat16), b16)


def test_gemm_bf16_out(qt, oracle):
    r = np.random.default_rng(3)
    _check(qt, oracle, r.normal(size=(256, 512)).astype(np.float32), r.normal(size=(256, 512)).astype(np.float32),
           out_dtype=torch.bfloat16)


def test_gemm_mask_hadamard_epilogue(qt, oracle):
    """dx = FWHT(dx_q * m) * fp32(16/9) fused in the epilogue (qlinear.py:229-230)."""
    M, N, K = 256, 512, 256
    r = np.random.default_rng(4)
    a = r.normal(size=(M, K)).astype(np.float32)
    b = r.normal(size=(N, K)).astype(np.float32)
    A, B = _operand(qt, a), _operand(qt, b)
    m = r.random((M, N)) < 0.9
    words = np.zeros((M, N // 32), np.uint32)
    for j in range(32):
        words |= m[:, j::32].astype(np.uint32) << j
    mask = torch.from_numpy(words.view(np.int32)).cuda()
    post = np.float32(16.0 / 9.0)
    got = qt.gemm(A, B, mask=mask, scale=float(post)).cpu().numpy()
    plain = qt.gemm(A, B).cpu().numpy()
    ref = oracle.fwht((plain * m).astype(np.float32), 32) * post
    assert np.array_equal(got, ref)   # same fp32 accumulator -> epilogue must be bit-exact
    got_nh = qt.gemm(A, B, mask=mask, hadamard=False, scale=float(post)).cpu().numpy()
    assert np.array_equal(got_nh, (plain * m).astype(np.float32) * post)


@pytest.mark.parametrize("mnk", [(256, 256, 256), (512, 768, 1024), (2048, 1024, 2304)])
def test_gemm_1cta_kernel(qt, oracle, mnk):
    """The 1-CTA kernel (128 x 256 tiles; the 2-CTA pair kernel is the default where N % 256 == 0) matches
    the oracle like the default path."""
    from paper_2505_14669_b200 import _lib

    L = _lib.load()
    L.qt_debug_set_gemm(0x40000)
    try:
        test_gemm_random(qt, oracle, mnk)
    finally:
        L.qt_debug_set_gemm(0)


@pytest.mark.parametrize("mnk", [(2048, 1024, 1024), (1024, 1152, 2048), (640, 768, 1184)])
def test_gemm_cluster8_multicast_kernel(qt, oracle, mnk):
    """The opt-in cluster-of-8 variant (2 x 2 pair tiles, A and B boxes multicast between pairs, partial
    super-tiles at the edges) matches the oracle like the default path."""
    from paper_2505_14669_b200 import _lib

    L = _lib.load()
    L.qt_debug_set_gemm(0x80000)
    try:
        test_gemm_random(qt, oracle, mnk)
    finally:
        L.qt_debug_set_gemm(0)


@pytest.mark.parametrize("mn", [(512, 768), (288, 512), (256, 96), (640, 1184)])
@pytest.mark.parametrize("odt", [torch.bfloat16, torch.float32])
def test_gemm_accumulate_equals_add(qt, mn, odt):
    """QT_EPI_ACCUMULATE: the epilogue adds its (dtype-rounded) result into out -- TMA reduce-add on the
    2-CTA kernel (N % 256 == 0), read-add-write on the 1-CTA kernel -- bit-identical to out.add_(gemm)."""
    M, N = mn
    K = 256
    g = torch.Generator(device="cuda").manual_seed(M * N)
    from paper_2505_14669_b200 import _lib

    A = qt.quant_rows(torch.randn(M, K, device="cuda", generator=g), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(torch.randn(N, K, device="cuda", generator=g), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    mask = torch.randint(-2**31, 2**31 - 1, (M, N // 32), device="cuda", dtype=torch.int32, generator=g)
    base = (torch.randn(M, N, device="cuda", generator=g) * 3).to(odt)
    for kw in ({}, {"mask": mask, "hadamard": True, "scale": 16 / 9}):
        want = base.clone().add_(qt.gemm(A, B, out_dtype=odt, **kw))
        got = base.clone()
        qt.gemm(A, B, out=got, accumulate=True, **kw)
        assert torch.equal(got, want), (mn, odt, kw)


@pytest.mark.parametrize("shape", [(256, 256, 8192), (1280, 1280, 4096), (768, 512, 2048), (4096, 4096, 2048),
                                   (4096, 11008, 2048)])
@pytest.mark.parametrize("epi", ["store", "maskH"])
def test_split_k_for_underfilled_fp32_gemms(qt, oracle, shape, epi):
    """fp32 GEMMs split K in two for the tiles of their last, partial wave (all tiles of an under-filled GEMM, e.g.
    the Llama-200M 1280 x 1280 attention dW; the last 34 of 256 tiles at 4096 x 4096): two K-half work units per
    such tile, added into zeroed output blocks by the epilogue's TMA reduce-add.  Deterministic (two addends per
    element), within the stated tolerance of the f64 product, and within fp32 rounding of the unsplit kernel
    (qt_debug_set_gemm bit 20)."""
    import ctypes

    M, N, K = shape
    r = np.random.default_rng(M + N + K)
    a = r.normal(size=(M, K)).astype(np.float32)
    b = r.normal(size=(N, K)).astype(np.float32)
    if epi == "store" and M * N * K <= 2 ** 31:
        _check(qt, oracle, a, b)
    A, B = _operand(qt, a), _operand(qt, b)
    kw = {}
    if epi == "maskH":
        kw = dict(mask=torch.randint(-2**31, 2**31 - 1, (M, N // 32), device="cuda", dtype=torch.int32),
                  hadamard=True, scale=16 / 9)
    s1 = qt.gemm(A, B, **kw)
    s2 = qt.gemm(A, B, **kw)
    assert torch.equal(s1, s2)
    L = qt._lib.load()
    L.qt_debug_set_gemm.argtypes = [ctypes.c_int]
    L.qt_debug_set_gemm(0x100000)
    try:
        u = qt.gemm(A, B, **kw)
    finally:
        L.qt_debug_set_gemm(0)
    assert float((s1 - u).norm() / u.norm()) < 1e-6


@pytest.mark.parametrize("mnk", [(640, 640, 4096), (512, 384, 4096), (1024, 128, 4352), (768, 640, 8192)])
def test_gemm_2cta_half_column_tile(qt, oracle, mnk):
    """N % 256 == 128 with K >= 4096 runs on the 2-CTA pair kernel: the last column tile's second-CTA B box lies
    wholly past N (TMA zero fill; its scale atoms in the zeroed 256-row padding) and its columns are clipped by the
    store map.
    Matches the oracle like every other path (the fp32 shapes also take the split-K tail)."""
    test_gemm_random(qt, oracle, mnk)


@pytest.mark.parametrize("odt", [torch.bfloat16, torch.float32])
def test_gemm_2cta_half_column_tile_epilogues(qt, odt):
    """Masked FWHT . 16/9 epilogue and accumulate on a N % 256 == 128 shape: the 2-CTA result equals the 1-CTA
    kernel's within fp32 rounding, and accumulate equals out + gemm."""
    from paper_2505_14669_b200 import _lib

    M, N, K = 768, 640, 4096
    g = torch.Generator(device="cuda").manual_seed(7)
    A = qt.quant_rows(torch.randn(M, K, device="cuda", generator=g), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(torch.randn(N, K, device="cuda", generator=g), _lib.QT_TRANSFORM_NONE, _lib.QT_ROUND_RTN)
    mask = torch.randint(-2**31, 2**31 - 1, (M, N // 32), device="cuda", dtype=torch.int32, generator=g)
    two = qt.gemm(A, B, mask=mask, hadamard=True, scale=16 / 9, out_dtype=odt)
    L = _lib.load()
    L.qt_debug_set_gemm(0x40000)
    try:
        one = qt.gemm(A, B, mask=mask, hadamard=True, scale=16 / 9, out_dtype=odt)
    finally:
        L.qt_debug_set_gemm(0)
    tol = 1e-5 if odt == torch.float32 else 1e-2
    assert torch.allclose(two.float(), one.float(), rtol=tol, atol=tol * float(one.float().abs().max()))
    base = torch.randn(M, N, device="cuda", generator=g).to(odt)
    out = base.clone()
    qt.gemm(A, B, out=out, accumulate=True)
    assert torch.equal(out, base + qt.gemm(A, B, out_dtype=odt))
