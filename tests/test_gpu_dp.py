"""Data-parallel token shards on the GPU path (2 shards simulated on one B200): each shard's
operands are bit-exact slices of the single-run operands, dx rows are bit-exact, and the dw partials
sum to the single-run dw within 1e-6 relative Frobenius (fp32 summation order)."""

import numpy as np
import pytest
import torch

from gpu_util import rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
def test_two_shards_match_single(rounding):
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200.dp import token_shard

    T, d_in, d_out, xi, world = 512, 256, 384, 29, 2
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(T, d_in, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(d_out, d_in, device="cuda", generator=g) / 16
    dy = torch.randn(T, d_out, device="cuda", generator=g).to(torch.bfloat16)
    _, ctx = qt.forward(x, w)
    dx, dw, ops = qt.backward(dy, ctx, xi=xi, rounding=rounding, return_operands=True)
    dw_sum = torch.zeros_like(dw, dtype=torch.float64)
    for r in range(world):
        off, n = token_shard(T, r, world)
        _, c = qt.forward(x[off:off + n], w)
        dxr, dwr, o = qt.backward(dy[off:off + n], c, xi=xi, rounding=rounding, return_operands=True,
                                  token_offset=off, total_tokens=T)
        assert torch.equal(dxr, dx[off:off + n])
        for name in ("gt_q", "xt_q"):
            full, part = ops[name], o[name]
            assert torch.equal(part.unpacked_codes(), full.unpacked_codes()[:, off:off + n]), name
            assert torch.equal(part.scales_rowmajor(), full.scales_rowmajor()[:, off // 32:(off + n) // 32]), name
        assert torch.equal(o["g_q"].unpacked_codes(), ops["g_q"].unpacked_codes()[off:off + n])
        dw_sum += dwr.double()
    assert rel_err(dw_sum.cpu().numpy(), dw.double().cpu().numpy()) <= 1e-6


@pytest.mark.parametrize("eager", [False, True])
def test_two_shards_sr_absmax_forward(eager):
    """sr_absmax forward (quantizers.py:79-84) on token shards: each shard's X_q (and, eager, X_t) is the
    exact slice of the single-run operand -- its SR stream positions are the global row * cols + col."""
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200.dp import token_shard

    T, d_in, d_out, seed, xi, world = 256, 128, 96, 17, 5, 2
    g = torch.Generator(device="cuda").manual_seed(8)
    x = torch.randn(T, d_in, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(d_out, d_in, device="cuda", generator=g) / 8
    kw = dict(bwd_xi=xi, total_tokens=T) if eager else {}
    y, ctx = qt.forward(x, w, scheme=qt.SR_ABSMAX, seed=seed, **kw)
    for r in range(world):
        off, n = token_shard(T, r, world)
        kr = dict(bwd_xi=xi, total_tokens=T, token_offset=off) if eager else dict(token_offset=off)
        yr, c = qt.forward(x[off:off + n], w, scheme=qt.SR_ABSMAX, seed=seed, **kr)
        assert torch.equal(c.x_q.unpacked_codes(), ctx.x_q.unpacked_codes()[off:off + n])
        assert torch.equal(c.x_q.scales_rowmajor(), ctx.x_q.scales_rowmajor()[off:off + n])
        assert torch.equal(yr, y[off:off + n])
        if eager:
            assert torch.equal(c.eager.xt_q.unpacked_codes(), ctx.eager.xt_q.unpacked_codes()[:, off:off + n])
