import torch, numpy as np
torch.manual_seed(0)
dev = "cuda"
H = torch.tensor([[(-1) ** bin(i & j).count("1") for j in range(32)] for i in range(32)], dtype=torch.float64)
Hb = H.to(dev).to(torch.bfloat16)
u = 2.0 ** -24
def test(name, x):
    x = x.to(torch.bfloat16)
    y = torch.mm(x, Hb, out_dtype=torch.float32).double()
    ex = x.double() @ H.to(dev)
    S = x.double().abs().sum(1, keepdim=True)
    m = ex.abs().max(1, keepdim=True).values
    e = (y - ex).abs()
    r1 = (e / (u * S.clamp_min(1e-300))).max().item()
    ok = S > 0
    print(f"{name:28s} max err/(u*S) = {r1:8.3f}   frac exact = {(e == 0).double().mean().item():.4f}   max err/(u*max|Hx|) = {(e/(u*m.clamp_min(1e-300))).max().item():9.3f}")
N = 1 << 20
g = torch.randn(N, 32, device=dev)
test("gaussian", g)
test("t(2)", torch.distributions.StudentT(2.0).sample((N, 32)).to(dev))
test("t(1)", torch.distributions.StudentT(1.0).sample((N, 32)).to(dev))
test("wide exp 2^U(-40,40)", g.sign() * torch.exp2(torch.rand(N, 32, device=dev) * 80 - 40))
test("wide exp 2^U(-20,20)", g.sign() * torch.exp2(torch.rand(N, 32, device=dev) * 40 - 20))
test("cancel: big +- plus small", torch.cat([torch.full((N, 1), 1e4, device=dev), g[:, :31]], 1))
x = g.clone(); x[:, ::2] = x[:, 1::2] * (1 + 2 ** -7)
test("near-cancel pairs", x)
test("ones + tiny", torch.ones(N, 32, device=dev) + g * 2 ** -9)
test("subnormal range", g * 2.0 ** -130)
