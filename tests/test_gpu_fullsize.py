"""BASELINE config 3 at full size (16384 tokens, the Llama-7B projection shapes): size-independent
properties of the production kernels, checked on the bench's own operand sizes.

* the fused forward (X -> X_q, M_x, X_t in one read) equals rows-then-requantize bit for bit;
* the tensor-core dual backward quantizer equals the CUDA-core path bit for bit;
* the 2-CTA GEMM's dW for two token shards sums to the full-batch dW (the data-parallel identity, fp32
  order tolerance) and the layer's y equals deq(X_q) deq(W_q)^T computed blockwise in fp64 on a sample.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu

T = 16384


@pytest.fixture(scope="module")
def qt():
    import paper_2505_14669_b200 as qt

    qt.load()
    return qt


@pytest.mark.parametrize("d_in", [4096, 11008])
def test_fused_forward_equals_rows_then_requant_full_size(qt, d_in):
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_cols, quant_fused, quant_rows, sign_bits

    g = torch.Generator(device="cuda").manual_seed(d_in)
    x = torch.randn(T, d_in, device="cuda", generator=g).to(torch.bfloat16)
    s = sign_bits(77, T, "cuda")
    H, RH, Q, R = _lib.QT_TRANSFORM_HADAMARD, _lib.QT_TRANSFORM_RANDOMIZED, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN
    xq, xt = quant_fused(x, Q, R, transform=H, col_transform=RH, col_signs=s, col_prescale=0.75)
    xq2 = quant_rows(x, H, Q, want_mask=True)
    xt2 = quant_cols(xq2, R, transform=RH, signs=s, prescale=0.75)
    assert torch.equal(xq.codes, xq2.codes) and torch.equal(xq.mask, xq2.mask)
    assert torch.equal(xq.scales_rowmajor(), xq2.scales_rowmajor())
    assert torch.equal(xt.codes, xt2.codes) and torch.equal(xt.scales_rowmajor(), xt2.scales_rowmajor())


@pytest.mark.parametrize("d_out", [4096, 11008])
def test_tensor_core_dual_equals_cuda_core_full_size(qt, d_out):
    from paper_2505_14669_b200 import _lib
    from paper_2505_14669_b200.mxfp4 import quant_dual, sign_bits

    g = torch.Generator(device="cuda").manual_seed(d_out + 1)
    dy = torch.randn(T, d_out, device="cuda", generator=g).to(torch.bfloat16)
    rs, cs = sign_bits(5, d_out, "cuda"), sign_bits(9, T, "cuda")
    L = _lib.load()
    outs = []
    for mode in (0, 1):
        L.qt_debug_set_quant(mode, None)
        try:
            outs.append(quant_dual(dy, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs,
                                   col_signs=cs, prescale=0.75))
        finally:
            L.qt_debug_set_quant(0, None)
    (a0, b0), (a1, b1) = outs
    assert torch.equal(a0.codes, a1.codes) and torch.equal(a0.scales_rowmajor(), a1.scales_rowmajor())
    assert torch.equal(b0.codes, b1.codes) and torch.equal(b0.scales_rowmajor(), b1.scales_rowmajor())


def test_layer_full_size_shards_and_sampled_gemm(qt):
    """4096 -> 11008 layer at 16384 tokens: two 8192-token shards (global sign / SR offsets) give the same
    y and dx rows and a dW that sums to the full-batch dW; y matches an fp64 product on sampled rows."""
    d_in, d_out, xi = 4096, 11008, 31
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(T, d_in, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(d_out, d_in, device="cuda", generator=g) / 64
    dy = torch.randn(T, d_out, device="cuda", generator=g).to(torch.bfloat16)
    y, ctx = qt.forward(x, w, check_finite=False, bwd_xi=xi)
    dx, dw = qt.backward(dy, ctx, xi=xi, check_finite=False)
    h = T // 2
    dw_sum = torch.zeros_like(dw)
    for r in range(2):
        sl = slice(r * h, (r + 1) * h)
        yr, cr = qt.forward(x[sl], w, check_finite=False, bwd_xi=xi, token_offset=r * h, total_tokens=T)
        dxr, dwr = qt.backward(dy[sl].contiguous(), cr, xi=xi, check_finite=False, token_offset=r * h, total_tokens=T)
        assert torch.equal(yr, y[sl]) and torch.equal(dxr, dx[sl])
        dw_sum += dwr
    assert ((dw_sum - dw).norm() / dw.norm()).item() < 1e-6
    rows = torch.arange(0, T, 997, device="cuda")
    ref = ctx.x_q.dequantize(torch.float64)[rows] @ ctx.w_q.dequantize(torch.float64).T
    assert ((y[rows].double() - ref).norm() / ref.norm()).item() < 1e-6
