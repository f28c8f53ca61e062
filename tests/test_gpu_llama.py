"""Llama-style model with every linear in Quartet MXFP4 (BASELINE configs 2/4/5 building blocks)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def llama():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200 import llama

    qt.load()
    return llama


def test_all_linears_are_quartet(llama):
    from paper_2505_14669_b200.nn import QuartetLinear

    cfg = llama.LlamaConfig(n_layer=2, d_model=256, n_head=2, vocab=1024, seq_len=64)
    m = llama.LlamaQuartet(cfg, device="cuda")
    assert not any(isinstance(mod, torch.nn.Linear) for mod in m.modules())
    assert sum(isinstance(mod, QuartetLinear) for mod in m.modules()) == 2 * 7 + 1


def test_training_reduces_loss(llama):
    torch.manual_seed(0)
    cfg = llama.LlamaConfig(n_layer=2, d_model=256, n_head=2, vocab=1024, seq_len=128)
    m = llama.LlamaQuartet(cfg, seed=1, device="cuda")
    tr = llama.Trainer(m, steps=40, lr=3e-3)
    tok, tgt = llama.synthetic_batch(cfg, 16, seed=3, device="cuda")
    losses = [float(tr.step(tok, tgt)) for _ in range(40)]
    assert all(l == l and l < 1e4 for l in losses)  # finite
    assert losses[-1] < losses[0] - 1.0, losses


def test_30m_forward_backward_shapes(llama):
    """BASELINE config 2 architecture (Llama-30M: 6 x 640, 5 heads), one step on a short batch."""
    cfg = llama.PRESETS["30m"]
    m = llama.LlamaQuartet(cfg, device="cuda")
    assert 25e6 < cfg.n_params() < 40e6
    tr = llama.Trainer(m, steps=10, lr=llama.PAPER_LR["30m"])
    tok, tgt = llama.synthetic_batch(cfg, 2, seed=0, device="cuda")
    loss = tr.step(tok, tgt)
    assert torch.isfinite(loss)
    assert all(p.grad is not None and torch.isfinite(p.grad).all() for p in m.parameters())


def test_lr_schedule_matches_reference(llama):
    """train.py:76-85 (warm-up 10 %, cosine to lr_floor)."""
    steps, lr = 100, 1.0
    assert llama.lr_at(0, steps, lr) == pytest.approx(0.1)
    assert llama.lr_at(9, steps, lr) == pytest.approx(1.0)
    assert llama.lr_at(99, steps, lr) == pytest.approx(0.0, abs=1e-12)


def test_fused_rope_matches_fp32_reference(llama):
    """csrc/glue.cu rotary embedding vs a plain fp32 torch reference (forward and the transposed backward);
    tolerance: one bf16 rounding of the fp32 result (2^-8 relative, plus tiny absolute)."""
    B, S, H, dh = 2, 64, 4, 128
    cos, sin = llama._rope(S, dh, 10000.0, "cuda")
    x = torch.randn(B, S, H, dh, device="cuda").to(torch.bfloat16).requires_grad_(True)
    y = llama.rope(x, cos, sin)
    xf = x.detach().float().transpose(1, 2)          # [B, H, S, dh]
    h = dh // 2
    rot = torch.cat((-xf[..., h:], xf[..., :h]), dim=-1)
    ref = (xf * cos.float() + rot * sin.float()).transpose(1, 2)
    torch.testing.assert_close(y.float(), ref, rtol=2 ** -8, atol=1e-6)
    dy = torch.randn_like(y)
    (gx,) = torch.autograd.grad(y, x, dy)
    xr = x.detach().float().requires_grad_(True)
    xrt = xr.transpose(1, 2)
    rr = torch.cat((-xrt[..., h:], xrt[..., :h]), dim=-1)
    yr = (xrt * cos.float() + rr * sin.float()).transpose(1, 2)
    (gr,) = torch.autograd.grad(yr, xr, dy.float())
    torch.testing.assert_close(gx.float(), gr, rtol=2 ** -8, atol=1e-6)


def test_fused_swiglu_matches_fp32_reference(llama):
    g = torch.randn(512, 384, device="cuda").to(torch.bfloat16).requires_grad_(True)
    u = torch.randn(512, 384, device="cuda").to(torch.bfloat16).requires_grad_(True)
    y = llama.swiglu(g, u)
    gf, uf = g.detach().float().requires_grad_(True), u.detach().float().requires_grad_(True)
    yf = torch.nn.functional.silu(gf) * uf
    torch.testing.assert_close(y.float(), yf, rtol=2 ** -7, atol=1e-5)
    dy = torch.randn_like(y)
    dg, du = torch.autograd.grad(y, (g, u), dy)
    dgf, duf = torch.autograd.grad(yf, (gf, uf), dy.float())
    torch.testing.assert_close(dg.float(), dgf, rtol=2 ** -7, atol=1e-4)
    torch.testing.assert_close(du.float(), duf, rtol=2 ** -7, atol=1e-4)


@pytest.mark.parametrize("d", [640, 1280, 1800, 4096])
def test_fused_rmsnorm_matches_fp32_reference(llama, d):
    """csrc/glue.cu RMSNorm (forward, dx, dw; warp-per-row and block-per-row variants) vs an fp32 torch
    reference; tolerance: bf16 rounding of the outputs (2^-7 relative) and fp32 summation order for dw."""
    x = torch.randn(1000, d, device="cuda").to(torch.bfloat16).requires_grad_(True)
    norm = llama.RMSNorm(d, device="cuda")
    with torch.no_grad():
        norm.weight.uniform_(0.5, 1.5)
    y = norm(x)
    xf = x.detach().float().requires_grad_(True)
    wf = norm.weight.detach().clone().requires_grad_(True)
    yf = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + norm.eps) * wf
    torch.testing.assert_close(y.float(), yf, rtol=2 ** -7, atol=1e-5)
    dy = torch.randn_like(y)
    dx, dw = torch.autograd.grad(y, (x, norm.weight), dy)
    dxf, dwf = torch.autograd.grad(yf, (xf, wf), dy.float())
    torch.testing.assert_close(dx.float(), dxf, rtol=2 ** -7, atol=1e-4)
    torch.testing.assert_close(dw, dwf, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("ignore", [False, True])
def test_fused_cross_entropy_matches_fp32_reference(llama, ignore):
    """csrc/glue.cu cross-entropy (loss and dlogits) vs torch's fp32 cross-entropy on the same bf16 logits;
    with ignore, some targets are -100 (torch's ignore_index): no loss, no gradient, not counted."""
    g = torch.Generator(device="cuda").manual_seed(5)
    logits = (torch.randn(300, 4000, device="cuda", generator=g) * 3).to(torch.bfloat16).requires_grad_(True)
    tgt = torch.randint(0, 4000, (300,), device="cuda", generator=g)
    if ignore:
        tgt[::7] = -100
    loss = llama.cross_entropy(logits, tgt)
    lf = logits.detach().float().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(lf, tgt)
    torch.testing.assert_close(loss, ref, rtol=1e-5, atol=1e-5)
    (gl,) = torch.autograd.grad(loss * 2.5, logits)
    (gr,) = torch.autograd.grad(ref * 2.5, lf)
    torch.testing.assert_close(gl.float(), gr, rtol=2 ** -7, atol=1e-6)


def test_fused_rope_strided_input(llama):
    """The rotary kernel reads a non-contiguous [B, S, H, dh] view (attention's transposed gradient layout)
    directly; result equal to rotating the contiguous copy."""
    B, S, H, dh = 2, 64, 4, 128
    cos, sin = llama._rope(S, dh, 10000.0, "cuda")
    base = torch.randn(B, H, S, dh, device="cuda").to(torch.bfloat16)
    xv = base.transpose(1, 2)                    # [B, S, H, dh], non-contiguous
    assert not xv.is_contiguous()
    for bwd in (False, True):
        a = llama._rope_call(xv, cos, sin, bwd)
        b = llama._rope_call(xv.contiguous(), cos, sin, bwd)
        assert torch.equal(a, b)


def _unfused_logits(llama, model, tokens):
    """The Llama forward with separate residual adds and norms (the structure before add_rmsnorm)."""
    import torch.nn.functional as F

    x = F.embedding(tokens, model.embed).to(torch.bfloat16)
    for blk in model.blocks:
        B, S, d = x.shape
        H, dh = blk.n_head, d // blk.n_head
        a = blk.attn_norm(x)
        q, k, v = llama.linear_group(a, (blk.q, blk.k, blk.v))
        q = llama.rope(q.view(B, S, H, dh), model.cos, model.sin).transpose(1, 2)
        k = llama.rope(k.view(B, S, H, dh), model.cos, model.sin).transpose(1, 2)
        v = v.view(B, S, H, dh).transpose(1, 2)
        att = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + blk.o(att.transpose(1, 2).reshape(B, S, d))
        m = blk.mlp_norm(x)
        g, u = llama.linear_group(m, (blk.gate, blk.up))
        x = x + blk.down(llama.swiglu(g, u))
    return model.head(model.norm(x))


@pytest.mark.parametrize("linear", ["quartet", "bf16"])
@pytest.mark.parametrize("d", [256, 4096])
def test_fused_residual_norms_bit_identical(llama, linear, d):
    """add_rmsnorm (residual add fused into the RMSNorm forward, the residual gradient into its backward;
    qt_rmsnorm_res) gives the same loss and the same gradients, bit for bit, as separate adds and norms with
    autograd's accumulation.  RMSNorm weight gradients are compared within fp32 rounding: their cross-block
    atomic sums have no fixed order in either structure."""
    cfg = llama.LlamaConfig(n_layer=2, d_model=d, n_head=d // 128, vocab=1024, seq_len=64, linear=linear)
    model = llama.LlamaQuartet(cfg, seed=3, device="cuda")
    model.eval()   # fixed backward seeds: both passes draw the same signs
    tok, tgt = llama.synthetic_batch(cfg, 2, seed=1, device="cuda")
    grads = []
    for fwd in (lambda: model(tok), lambda: _unfused_logits(llama, model, tok)):
        model.zero_grad(set_to_none=True)
        logits = fwd()
        loss = llama.cross_entropy(logits.reshape(-1, cfg.vocab), tgt.reshape(-1))
        loss.backward()
        grads.append((loss.detach().clone(), {n: p.grad.clone() for n, p in model.named_parameters()}))
    (l0, g0), (l1, g1) = grads
    assert torch.equal(l0, l1)
    for n in g0:
        if n.endswith("norm.weight"):
            torch.testing.assert_close(g0[n], g1[n], rtol=1e-5, atol=1e-6)
        else:
            assert torch.equal(g0[n], g1[n]), n


@pytest.mark.parametrize("d", [640, 1280, 1800, 2048, 6144])
def test_add_rmsnorm_equals_add_then_norm(llama, d):
    """qt_rmsnorm_res at the narrow (one warp per row, every NV) and wide kernel sizes: forward (h, n) equal
    torch's bf16 add and the plain RMSNorm of it, backward dx equals the plain backward plus the residual
    gradient (bf16 add), bit for bit; dw within fp32 rounding (atomic order)."""
    g = torch.Generator(device="cuda").manual_seed(d)
    x = torch.randn(777, d, device="cuda", generator=g).to(torch.bfloat16).requires_grad_(True)
    y = torch.randn(777, d, device="cuda", generator=g).to(torch.bfloat16).requires_grad_(True)
    norm = llama.RMSNorm(d, device="cuda")
    with torch.no_grad():
        norm.weight.uniform_(0.5, 1.5)
    h, n = llama.add_rmsnorm(x, y, norm)
    h_ref = x.detach() + y.detach()
    assert torch.equal(h, h_ref)
    h_ref.requires_grad_(True)
    n_ref = norm(h_ref)
    assert torch.equal(n, n_ref)
    dh, dn = torch.randn_like(h), torch.randn_like(n)
    dx, dy_, dw = torch.autograd.grad((h, n), (x, y, norm.weight), (dh, dn))
    dh_ref, dw_ref = torch.autograd.grad(n_ref, (h_ref, norm.weight), dn)
    assert torch.equal(dx, dh_ref + dh) and torch.equal(dy_, dx)
    # dw: 777-term fp32 sums of O(1) products in different (atomic) orders: |error| <= 777 * 3 * 2^-24 ~ 1.4e-4
    torch.testing.assert_close(dw, dw_ref, rtol=1e-5, atol=5e-4)
