"""GPU quantizer diagnostics against the reference itself.

* Exact: gaussian_mse for every scheme and misalignment_suite reproduce the reference's estimates BIT FOR BIT
  (value, stderr, excluded) -- tests/golden/diag.npz was produced by mx4train.diagnostics
  (make_seam_golden.py); same sample streams, same per-sample arithmetic, same reductions.
* The reductions are numpy's pairwise add.reduce (seam_row_sums vs np.sum on ragged lengths).
* SR unbiasedness of the PRODUCTION stochastic-rounding kernel (the tiled quantizer the backward pass uses),
  with the reference's own multiple-comparison z-score criterion (selftest.py:125-153: 100 inputs x 32
  elements, 1e5 draws each; at most 1 % of |z| beyond 3 and every |z| <= 6).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def diag():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200 import diagnostics

    qt.load()
    return diagnostics


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "diag.npz"))


@pytest.mark.parametrize("kind", ["exact", "rtn_absmax", "sr_absmax", "quest"])
def test_gaussian_mse_bit_exact(diag, gold, kind):
    est = diag.gaussian_mse(kind, dim=256, samples=48, seed=5, batch=20)
    ref = gold[f"mse_{kind}"]
    assert (est.value, est.stderr, est.samples) == (ref[0], ref[1], int(ref[2]))


def test_misalignment_suite_bit_exact(diag, gold):
    kinds = ("exact", "rtn_absmax", "sr_absmax", "quest")
    got = diag.misalignment_suite(kinds, dim=128, samples=300, seed=3, batch=128)
    for kind in kinds:
        ref = gold[f"mis_{kind}"]
        est = got[kind]
        assert (est.value, est.stderr, est.samples, est.excluded) == (ref[0], ref[1], int(ref[2]), int(ref[3])), kind


def test_row_sums_are_numpy_pairwise():
    import torch

    from paper_2505_14669_b200.mxfp4 import seam_row_sums

    r = np.random.default_rng(3)
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 2048, 4096):
        a = r.normal(size=(6, n)) * np.exp(r.normal(size=(6, n)) * 4)
        b = r.normal(size=(6, n))
        ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        assert np.array_equal(seam_row_sums(ta, tb, 0).cpu().numpy(), ((a - b) ** 2).sum(axis=1)), n
        assert np.array_equal(seam_row_sums(ta, tb, 1).cpu().numpy(), (a * b).sum(axis=1)), n
        assert np.array_equal(seam_row_sums(ta, None, 1).cpu().numpy(), (a * a).sum(axis=1)), n


@pytest.mark.parametrize("mode", ["sr", "sr_fast"])
def test_production_sr_unbiased_zscores(diag, mode):
    """selftest.py:125-153 (c04) on the tiled SR kernel: 100 fp32 inputs of 32 elements at scales
    2^-4 .. 2^4, 1e5 draws each (distinct stream positions), z of the mean against the input.  "sr" is the
    reference's splitmix64 stream, "sr_fast" the hash-uniform mode (QT_ROUND_SR_FAST)."""
    import torch

    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import derive_seed, quant_rows

    draws, width, seed = 100_000, 32, 0
    zs = []
    for i in range(100):
        base = diag.gaussians(derive_seed(seed, 4, i), 0x4755, 0, width) * 2.0 ** ((i % 9) - 4)
        b32 = torch.from_numpy(base.astype(np.float32)).cuda()
        x = b32.view(1, width).expand(draws, width).contiguous()
        rc = _lib.QT_ROUND_SR if mode == "sr" else _lib.QT_ROUND_SR_FAST
        op = quant_rows(x, _lib.QT_TRANSFORM_NONE, rc, sr_seed=derive_seed(seed, 4, i, 1))
        d = op.dequantize(torch.float64)
        mean = d.mean(dim=0)
        se = d.std(dim=0) / draws ** 0.5
        se[se == 0] = float("inf")   # exact grid points round deterministically
        zs.append(((mean - b32.double()) / se).abs().cpu().numpy())
    zs = np.concatenate(zs)
    frac3, zmax = float((zs > 3.0).mean()), float(zs.max())
    assert frac3 <= 0.01 and zmax <= 6.0, (frac3, zmax)


def test_sr_fast_rounds_to_the_same_neighbours():
    """QT_ROUND_SR_FAST draws differ from the reference's stream, but every code is one of the two grid
    neighbours the exact SR picks from and the E8M0 scales are identical."""
    import torch

    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_rows

    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn(512, 1024, device="cuda", generator=g) * torch.exp2(torch.randint(-8, 8, (512, 1), device="cuda",
                                                                                        generator=g).float())
    a = quant_rows(x, _lib.QT_TRANSFORM_HADAMARD, _lib.QT_ROUND_SR, sr_seed=77)
    b = quant_rows(x, _lib.QT_TRANSFORM_HADAMARD, _lib.QT_ROUND_SR_FAST, sr_seed=77)
    assert torch.equal(a.scales_rowmajor(), b.scales_rowmajor())
    da, db = a.dequantize(torch.float64), b.dequantize(torch.float64)
    step = torch.exp2(a.scales_rowmajor().double() - 127).repeat_interleave(32, dim=1) * 2.0   # widest grid gap
    assert bool(((da - db).abs() <= step).all())
    assert not torch.equal(a.codes, b.codes)       # a different (hash) stream
    c = quant_rows(x, _lib.QT_TRANSFORM_HADAMARD, _lib.QT_ROUND_SR_FAST, sr_seed=77)
    assert torch.equal(b.codes, c.codes)           # deterministic given the seed


@pytest.mark.parametrize("grid", [0, 3])
@pytest.mark.parametrize("path", ["dual", "fused"])
def test_tensor_core_sr_fast_matches_cuda_core_sr_fast(path, grid):
    """QT_ROUND_SR_FAST on the tensor-core quantizers (k_tcq_dual, k_tcq_xq's X_t) draws the same hash uniforms
    at the same stream positions as the CUDA-core path, for values within the tensor-core error bound of the
    reference's: the codes agree except where a uniform falls within ~1e-6 of p, and every difference is
    between the two SR neighbours; the E8M0 scales are identical."""
    import torch

    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_dual, quant_fused, sign_bits

    g = torch.Generator(device="cuda").manual_seed(12)
    x = (torch.randn(2048, 1024, device="cuda", generator=g) * 3).to(torch.bfloat16)
    rs, cs = sign_bits(5, 1024, "cuda"), sign_bits(9, 2048, "cuda", start=64)
    L = _lib.load()
    outs = []
    L.qt_debug_set_grid(grid)       # 3 CTAs: every CTA walks many tiles (stage / TMEM reuse)
    try:
        for mode in (0, 1):
            L.qt_debug_set_quant(mode, None)
            try:
                if path == "dual":
                    outs.append(quant_dual(x, _lib.QT_ROUND_SR_FAST, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs,
                                           col_signs=cs, prescale=0.75, seed_rows=3, seed_cols=4, row_counter_start=99,
                                           col_counter_start=64, col_counter_ld=4096))
                else:
                    outs.append(quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_SR_FAST,
                                            transform=_lib.QT_TRANSFORM_HADAMARD,
                                            col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=cs, col_prescale=0.75,
                                            col_seed=4, col_counter_start=64, col_counter_ld=4096))
            finally:
                L.qt_debug_set_quant(0, None)
    finally:
        L.qt_debug_set_grid(0)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a.scales_rowmajor(), b.scales_rowmajor())
        ca, cb = a.unpacked_codes(), b.unpacked_codes()
        diff = ca != cb
        assert float(diff.float().mean()) < 1e-4, float(diff.float().mean())
        da, db = a.dequantize(torch.float64), b.dequantize(torch.float64)
        step = torch.exp2(a.scales_rowmajor().double() - 127).repeat_interleave(32, dim=1) * 2.0
        assert bool(((da - db).abs() <= step).all())
