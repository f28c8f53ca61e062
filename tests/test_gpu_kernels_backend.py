"""The b200 `kernels` backend (paper_2505_14669_b200.kernels) against the oracle, in the style of the
reference's own backend-equivalence test (mx4train tests/test_backends.py:18-88): same adversarial
inputs (cast to fp32, the values the layer path produces), bit-identical outputs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    from paper_2505_14669_b200 import kernels

    return kernels


def _random_inputs():
    r = np.random.default_rng(0)
    yield r.normal(size=(7, 97)).astype(np.float32)                       # ragged trailing group
    yield (r.normal(size=(3, 32)) * 1e-6).astype(np.float32)
    yield (r.normal(size=(2, 64)) * 1e6).astype(np.float32)
    yield r.standard_t(df=2, size=(5, 160)).astype(np.float32)
    x = np.zeros((2, 40), np.float32)
    x[0, 0] = 6.0
    yield x
    yield np.array([[0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, -0.75, -2.5, -0.0] + [6.0] * 22], np.float32)


def test_quantize_rtn_identical(kb, oracle):
    for x in _random_inputs():
        c1, s1 = kb.quantize_rtn(x.astype(np.float64), 32)
        c2, s2 = oracle.quantize_rtn(x, 32)
        assert np.array_equal(c1, c2) and np.array_equal(s1, s2)


def test_quantize_sr_identical(kb, oracle):
    for i, x in enumerate(_random_inputs()):
        c1, s1 = kb.quantize_sr(x.astype(np.float64), 32, 1234 + i, 17)
        c2, s2 = oracle.quantize_sr(x, 32, 1234 + i, 17)
        assert np.array_equal(c1, c2) and np.array_equal(s1, s2), i


def test_quantize_quest_identical(kb, oracle):
    for x in _random_inputs():
        got = kb.quantize_quest(x.astype(np.float64), 32, 1.0 / 16.0)
        ref = oracle.quantize_quest(x, 32, 1.0 / 16.0)
        for a, b in zip(got, ref):
            assert np.array_equal(a, b)


def test_fwht_identical(kb, oracle):
    x = np.random.default_rng(32).normal(size=(5, 64)).astype(np.float32)
    assert np.array_equal(kb.fwht(x, 32), oracle.fwht(x, 32))


def test_sr_stream_position_invariance(kb):
    """test_backends.py:77-88: the draw depends only on (seed, counter_start + index)."""
    x = np.random.default_rng(2).normal(size=(4, 64)).astype(np.float32)
    c_full, _ = kb.quantize_sr(x, 32, 7, 0)
    c_rows = np.vstack([kb.quantize_sr(x[i:i + 1], 32, 7, i * 64)[0] for i in range(4)])
    assert np.array_equal(c_full, c_rows)


def test_gemm_nt_on_mxfp4_operands(kb, oracle):
    r = np.random.default_rng(4)
    ac, as_ = oracle.quantize_rtn(r.normal(size=(64, 96)), 32)
    bc, bs = oracle.quantize_rtn(r.normal(size=(40, 96)), 32)
    a = oracle.dequantize(ac, as_, 32, np.float32)
    b = oracle.dequantize(bc, bs, 32, np.float32)
    got = kb.gemm_nt(a, b)
    assert np.array_equal(got, oracle.gemm_nt(a, b))  # exact products, sums exact in fp32 here


def test_rejects_non_fp32_inputs(kb):
    with pytest.raises(ValueError):
        kb.quantize_rtn(np.array([[0.1] * 32]), 32)


@pytest.mark.parametrize("shape", [(0, 64), (3, 0), (0, 0)])
def test_empty_inputs_match_reference(kb, oracle, shape):
    """Empty rows / columns: the reference's kernels return empty (or, for gemm_nt with an empty
    contraction, all-zero) arrays of the right shapes and dtypes without touching a kernel."""
    x = np.zeros(shape, np.float32)
    for got, want in ((kb.quantize_rtn(x.astype(np.float64), 32), oracle.quantize_rtn(x, 32)),
                      (kb.quantize_sr(x.astype(np.float64), 32, 5, 0), oracle.quantize_sr(x, 32, 5, 0)),
                      (kb.quantize_quest(x.astype(np.float64), 32, 1 / 16), oracle.quantize_quest(x, 32, 1 / 16))):
        for g, w in zip(got, want):
            assert g.shape == w.shape and g.dtype == w.dtype
    assert kb.fwht(x, 32).shape == shape
    b = np.zeros((2, shape[1]), np.float32)
    g, w = kb.gemm_nt(x, b), oracle.gemm_nt(x, b)
    assert g.shape == w.shape and np.array_equal(g, w)
