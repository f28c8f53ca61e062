"""End-to-end Quartet linear layer on the GPU vs the reference (golden fixtures) and the oracle.

Bit-exact: every quantized operand (X_q, W_q, masks, G_q, Wt_q, Gt_q, Xt_q).
Tolerance (stated): y, dx, dw relative Frobenius error vs the reference's fp32 outputs
    <= 1e-5  (the only difference is the fp32 accumulation order inside the three GEMMs).
"""

import os

import numpy as np
import pytest
import torch

from gpu_util import assert_operand_equal, bf16_values, rel_err, to_dev

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-5
GOLDEN_CASES = ["quest_rtn", "quest_sr", "quest_rtn_t256", "rtnfwd_rtn", "quest_rtn_noh", "srfwd_sr", "srfwd_rtn_t256",
                "quest_rtn_noh_ragged", "quest_sr_noh_ragged", "rtnfwd_sr_noh_ragged"]


@pytest.fixture(scope="module")
def qt():
    import paper_2505_14669_b200 as qt

    qt.load()
    return qt


def _scheme(qt, kind):
    return {"quest": qt.QUEST, "rtn_absmax": qt.RTN_ABSMAX, "sr_absmax": qt.SR_ABSMAX}[kind]


@pytest.mark.parametrize("eager", [False, True], ids=["lazy", "eager"])
@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_golden_end_to_end(qt, oracle, case, eager):
    """eager: forward(..., bwd_xi=xi) builds X_t / W_t in the forward read (qt_quant_fused).
    srfwd_*: the sr_absmax forward scheme (stochastic rounding of X and W with derive_seed(seed, 11/12),
    qlinear.py:148-154, quantizers.py:79-84)."""
    z = np.load(os.path.join(GOLDEN, f"qlinear_{case}.npz"))
    had = bool(z["hadamard"])
    seed = int(z["seed"]) if "seed" in z.files else None
    kw = dict(bwd_xi=int(z["xi"]), bwd_rounding=str(z["rounding"])) if eager else {}
    y, ctx = qt.forward(to_dev(z["x"], torch.bfloat16), to_dev(z["w"], torch.bfloat16),
                        scheme=_scheme(qt, str(z["scheme"])), hadamard=had, seed=seed, **kw)
    whole = z["x"].shape[0] % 32 == 0 and z["w"].shape[0] % 32 == 0   # ragged shapes take the lazy path
    assert (ctx.eager is not None) == (eager and whole)
    # saved context: bit-exact against the reference's LayerContext
    assert np.array_equal(ctx.x_q.codes.cpu().numpy(), z["x_codes"])
    assert np.array_equal(ctx.x_q.scales_rowmajor().cpu().numpy(), z["x_scales"])
    assert np.array_equal(ctx.w_q.codes.cpu().numpy(), z["w_codes"])
    assert np.array_equal(ctx.w_q.scales_rowmajor().cpu().numpy(), z["w_scales"])
    assert np.array_equal(ctx.m_x.cpu().numpy(), z["m_x"])
    assert np.array_equal(ctx.m_w.cpu().numpy(), z["m_w"])
    assert rel_err(y.cpu().numpy(), z["y"]) <= TOL
    dx, dw, ops = qt.backward(to_dev(z["dy"], torch.bfloat16), ctx, xi=int(z["xi"]), rounding=str(z["rounding"]),
                              return_operands=True)
    assert rel_err(dx.cpu().numpy(), z["dx"]) <= TOL, rel_err(dx.cpu().numpy(), z["dx"])
    assert rel_err(dw.cpu().numpy(), z["dw"]) <= TOL, rel_err(dw.cpu().numpy(), z["dw"])
    # backward operands: bit-exact against the oracle's recomposition (itself pinned to the reference)
    _, octx = oracle.forward(z["x"], z["w"], scheme=str(z["scheme"]), hadamard=had, seed=seed)
    oracle.backward(z["dy"], octx, xi=int(z["xi"]), rounding=str(z["rounding"]))
    for name, key in (("g_q", "gq"), ("wt_q", "wtq"), ("gt_q", "gtq"), ("xt_q", "xtq")):
        c, s = octx.inter[key]
        assert_operand_equal(ops[name], c, s, name)


@pytest.mark.parametrize("shape", [(50, 64, 45), (96, 128, 200), (33, 32, 1)])
def test_ragged_forward_with_hadamard(qt, oracle, shape):
    """The reference's forward takes any batch and d_out (only d_in must be whole blocks, qlinear.py:114-165);
    backward then needs whole blocks of d_out and batch when hadamard=True and raises ValueError otherwise."""
    T, d_in, d_out = shape
    r = np.random.default_rng(T * 1000 + d_out)
    x = bf16_values(r.normal(size=(T, d_in)).astype(np.float32))
    w = bf16_values((r.normal(size=(d_out, d_in)) / np.sqrt(d_in)).astype(np.float32))
    y_ref, octx = oracle.forward(x, w)
    y, ctx = qt.forward(to_dev(x, torch.bfloat16), to_dev(w, torch.bfloat16), bwd_xi=3)
    assert ctx.eager is None
    assert_operand_equal(ctx.x_q, octx.x_codes, octx.x_scales, "X_q")
    assert_operand_equal(ctx.w_q, octx.w_codes, octx.w_scales, "W_q")
    assert tuple(y.shape) == (T, d_out)
    assert rel_err(y.cpu().numpy(), y_ref) <= TOL
    dy = torch.randn(T, d_out, device="cuda", dtype=torch.bfloat16)
    if T % 32 or d_out % 32:
        with pytest.raises(ValueError, match="not divisible"):
            qt.backward(dy, ctx, xi=3)


@pytest.mark.parametrize("eager", [False, True], ids=["lazy", "eager"])
@pytest.mark.parametrize("rounding", ["rtn", "sr"])
def test_config1_against_oracle(qt, oracle, rounding, eager):
    """BASELINE config 1: 1024x1024 weight, 2048 tokens, g = 32 (the CPU reference's own case)."""
    T, d_in, d_out, xi = 2048, 1024, 1024, 7
    x = bf16_values(oracle.gaussians(1, oracle.DOMAIN_GAUSS, 0, T * d_in).reshape(T, d_in).astype(np.float32))
    w = bf16_values((oracle.gaussians(2, oracle.DOMAIN_GAUSS, 0, d_out * d_in) / 32.0)
                    .reshape(d_out, d_in).astype(np.float32))
    dy = bf16_values(oracle.gaussians(3, oracle.DOMAIN_GAUSS, 0, T * d_out).reshape(T, d_out).astype(np.float32))
    oracle.set_threads(os.cpu_count() or 1)
    try:
        y_ref, octx = oracle.forward(x, w)
        dx_ref, dw_ref = oracle.backward(dy, octx, xi=xi, rounding=rounding)
    finally:
        oracle.set_threads(1)
    kw = dict(bwd_xi=xi, bwd_rounding=rounding) if eager else {}
    y, ctx = qt.forward(to_dev(x, torch.bfloat16), to_dev(w, torch.bfloat16), **kw)
    assert (ctx.eager is not None) == eager
    assert_operand_equal(ctx.x_q, octx.x_codes, octx.x_scales, "X_q")
    assert_operand_equal(ctx.w_q, octx.w_codes, octx.w_scales, "W_q")
    assert np.array_equal(ctx.m_x.cpu().numpy(), octx.m_x)
    dx, dw, ops = qt.backward(to_dev(dy, torch.bfloat16), ctx, xi=xi, rounding=rounding, return_operands=True)
    for name, key in (("g_q", "gq"), ("wt_q", "wtq"), ("gt_q", "gtq"), ("xt_q", "xtq")):
        c, s = octx.inter[key]
        assert_operand_equal(ops[name], c, s, name)
    for got, ref, what in ((y, y_ref, "y"), (dx, dx_ref, "dx"), (dw, dw_ref, "dw")):
        e = rel_err(got.cpu().numpy(), ref)
        print(f"config1 {rounding} {what}: rel err {e:.3e}")
        assert e <= TOL, (what, e)


def test_shape_validation(qt):
    """test_qlinear.py:200-211 on the GPU path."""
    dev = "cuda"
    with pytest.raises(ValueError):
        qt.forward(torch.ones(4, 33, device=dev), torch.ones(8, 33, device=dev))
    with pytest.raises(ValueError):
        qt.forward(torch.ones(4, 32, device=dev), torch.ones(8, 64, device=dev))
    _, ctx = qt.forward(torch.ones(32, 32, device=dev), torch.ones(64, 32, device=dev))
    with pytest.raises(ValueError):
        qt.backward(torch.ones(32, 16, device=dev), ctx, xi=0)
    with pytest.raises(ValueError):
        qt.backward(torch.ones(32, 64, device=dev), ctx, xi=0, rounding="nearest")
    with pytest.raises(ValueError):
        qt.forward(torch.ones(32, 32, device=dev), torch.ones(32, 32, device=dev), scheme=qt.SR_ABSMAX)


@pytest.mark.parametrize("bwd_xi", [None, 3])
def test_empty_batch(qt, bwd_xi):
    """batch = 0 passes the reference's checks (0 % 32 == 0): y and dx are empty, dW is all zeros."""
    x, w = torch.zeros(0, 64, device="cuda"), torch.randn(32, 64, device="cuda")
    y, ctx = qt.forward(x, w, bwd_xi=bwd_xi)
    assert tuple(y.shape) == (0, 32)
    dx, dw = qt.backward(torch.zeros(0, 32, device="cuda"), ctx, xi=3)
    assert tuple(dx.shape) == (0, 64) and tuple(dw.shape) == (32, 64) and torch.all(dw == 0)


def test_zero_dy_gives_zero_grads(qt):
    x = torch.randn(64, 64, device="cuda")
    w = torch.randn(32, 64, device="cuda")
    _, ctx = qt.forward(x, w)
    dx, dw = qt.backward(torch.zeros(64, 32, device="cuda"), ctx, xi=1)
    assert torch.all(dx == 0) and torch.all(dw == 0)


def test_determinism_and_seed_sensitivity(qt):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(128, 256, device="cuda", generator=g)
    w = torch.randn(96, 256, device="cuda", generator=g)
    dy = torch.randn(128, 96, device="cuda", generator=g)
    _, ctx = qt.forward(x, w)
    a1 = qt.backward(dy, ctx, xi=5)
    a2 = qt.backward(dy, ctx, xi=5)
    b = qt.backward(dy, ctx, xi=6)
    assert torch.equal(a1[0], a2[0]) and torch.equal(a1[1], a2[1])
    assert not torch.equal(a1[0], b[0])


def test_quantized_gradient_close_to_exact(qt):
    """test_qlinear.py:254-264: cosine > 0.9 against the exact gradients."""
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(256, 512, device="cuda", generator=g)
    w = torch.randn(256, 512, device="cuda", generator=g)
    dy = torch.randn(256, 256, device="cuda", generator=g)
    _, ctx = qt.forward(x, w)
    dx, dw = qt.backward(dy, ctx, xi=3)
    for got, ref in ((dx, dy @ w), (dw, dy.T @ x)):
        cos = torch.nn.functional.cosine_similarity(got.flatten().double(), ref.flatten().double(), dim=0)
        assert cos > 0.9


def test_autograd_function_and_module(qt):
    torch.manual_seed(0)
    layer = qt.QuartetLinear(256, 128, seed=3, layer_id=1).cuda()
    x = torch.randn(4, 64, 256, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    y = layer(x)
    assert y.shape == (4, 64, 128) and y.dtype == torch.bfloat16
    y.float().square().mean().backward()
    assert x.grad is not None and x.grad.shape == x.shape and torch.isfinite(x.grad.float()).all()
    assert layer.weight.grad is not None and layer.weight.grad.dtype == torch.float32
    # the autograd path equals the functional path for the same xi
    x2 = x.detach().reshape(-1, 256)
    y_ref, ctx = qt.forward(x2, layer.weight.detach(), out_dtype=torch.bfloat16)
    xi = qt.derive_seed(qt.derive_seed(3, 4, 0), 1)
    y2 = qt.quartet_linear(x2, layer.weight, xi)
    assert torch.equal(y2, y_ref)


@pytest.mark.parametrize("rounding", ["rtn", "sr", "sr_fast"])
def test_group_of_linears_sharing_x_matches_separate_layers(rounding):
    """quartet_linear_group (one QuEST read of x for q/k/v-style layers) gives bit-identical outputs and
    weight gradients to separate QuartetLinear calls; dx agrees to bf16 rounding of the summed gradient."""
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200.nn import QuartetLinear, quartet_linear_group

    qt.load()
    torch.manual_seed(0)
    mods_a = [QuartetLinear(256, o, seed=3, layer_id=i, rounding=rounding, device="cuda")
              for i, o in enumerate((256, 128, 384))]
    mods_b = [QuartetLinear(256, o, seed=3, layer_id=i, rounding=rounding, device="cuda")
              for i, o in enumerate((256, 128, 384))]
    for a, b in zip(mods_a, mods_b):
        b.weight.data.copy_(a.weight.data)
    x = torch.randn(512, 256, device="cuda").to(torch.bfloat16)
    xa, xb = x.clone().requires_grad_(True), x.clone().requires_grad_(True)
    ya = [m(xa) for m in mods_a]
    yb = quartet_linear_group(xb, mods_b)
    dys = [torch.randn_like(y) for y in ya]
    torch.autograd.backward(ya, dys)
    torch.autograd.backward(list(yb), dys)
    for y1, y2 in zip(ya, yb):
        assert torch.equal(y1, y2)
    for a, b in zip(mods_a, mods_b):
        assert torch.equal(a.weight.grad, b.weight.grad)
    # both sum three bf16 dx in bf16; the summation order may differ -- agreement to bf16 rounding
    scale = xb.grad.float().abs().max()
    assert (xa.grad.float() - xb.grad.float()).abs().max() <= 2 ** -7 * scale
