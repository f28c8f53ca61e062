"""torch.autograd.Function / nn.Module surface of the Quartet linear layer.

``QuartetLinearFn`` is the drop-in autograd form of the reference's functional pair
(qlinear.forward / qlinear.backward, qlinear.py:114-252): its ctx carries the reference's
LayerContext (quantized X/W operands and trust masks), ``xi`` seeds the backward randomized
Hadamard / stochastic rounding, and ``rounding`` selects "rtn" (default) or "sr".

``QuartetLinear`` is a bias-free linear module (the reference's layers are bias-free,
qlinear.py:18) holding an fp32 master weight; it derives a fresh ``xi`` per step the way the
reference's training loop does (train.py:346-348: derive_seed(derive_seed(seed, 4, step), layer)).
"""

from __future__ import annotations

import math

import torch

from . import qlinear
from .mxfp4 import derive_seed


DEVICE_XI = -1   # placeholder xi of layers whose seed is device-resident (matches forward's eager operands)
_NONFINITE: dict = {}


def nonfinite_flag(device) -> torch.Tensor:
    """The per-device flag the autograd path ORs non-finite quantizer inputs into (no host sync per call; the
    reference raises ValueError("non-finite input") at once, codec.py:164-170)."""
    dev = torch.device(device)
    if dev not in _NONFINITE:
        _NONFINITE[dev] = torch.zeros(1, dtype=torch.int32, device=dev)
    return _NONFINITE[dev]


def raise_if_nonfinite(device=None) -> None:
    """One host sync: raise ValueError if any Quartet layer on `device` (default: all) quantized a non-finite
    value since the last call, and clear the flag.  The training loop calls it once per step, after backward
    (the reference's loop stops on a non-finite loss, train.py:341-343)."""
    devs = [torch.device(device)] if device is not None else list(_NONFINITE)
    bad = False
    for d in devs:
        f = _NONFINITE.get(d)
        if f is not None and int(f.item()) != 0:
            f.zero_()
            bad = True
    if bad:
        raise ValueError("non-finite input")


class QuartetLinearFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, xi: int, rounding: str = "rtn", hadamard: bool = True,
                scheme: qlinear.QuantScheme = qlinear.QUEST, shard: tuple = (0, None), xi_dev=None):
        lead = x.shape[:-1]
        x2 = x.reshape(-1, x.shape[-1])
        if x2.dtype not in (torch.bfloat16, torch.float32):
            x2 = x2.float()
        ctx.shard = shard
        # xi is known now, so X_t / W_t come out of the same read of x / w (qt_quant_fused)
        y, lctx = qlinear.forward(x2, w.detach(), scheme=scheme, hadamard=hadamard, seed=xi,
                                  out_dtype=x.dtype if x.dtype in (torch.bfloat16, torch.float32) else torch.float32,
                                  check_finite=nonfinite_flag(x.device), bwd_xi=int(xi), bwd_rounding=rounding,
                                  token_offset=shard[0], total_tokens=shard[1], bwd_xi_dev=xi_dev)
        ctx.lctx = lctx
        ctx.xi = int(xi)
        ctx.rounding = rounding
        ctx.x_shape = x.shape
        ctx.x_dtype = x.dtype
        ctx.w_dtype = w.dtype
        return y.reshape(*lead, w.shape[0])

    @staticmethod
    def backward(ctx, dy):
        dy2 = dy.reshape(-1, dy.shape[-1])
        if dy2.dtype not in (torch.bfloat16, torch.float32):
            dy2 = dy2.float()
        dx, dw = qlinear.backward(dy2, ctx.lctx, ctx.xi, ctx.rounding, dx_dtype=ctx.x_dtype
                                  if ctx.x_dtype in (torch.bfloat16, torch.float32) else torch.float32,
                                  dw_dtype=torch.float32, check_finite=nonfinite_flag(dy.device), token_offset=ctx.shard[0],
                                  total_tokens=ctx.shard[1])
        ctx.lctx = None
        return dx.reshape(ctx.x_shape), dw.to(ctx.w_dtype), None, None, None, None, None, None


class QuartetLinearGroupFn(torch.autograd.Function):
    """Several Quartet linears reading the same x (q/k/v, gate/up): X_q and M_x = QuEST(H32 x) are computed
    once (they depend on x alone; the first layer's fused quantizer pass also gives its own X_t), the other
    layers derive their X_t (their own xi) from X_q's codes, and the
    input gradients of the layers are summed in x's dtype (as autograd accumulates separate layers' dx).
    Outputs and weight gradients are bit-identical to separate QuartetLinearFn calls."""

    @staticmethod
    def forward(ctx, x, xis, rounding, hadamard, scheme, shard, xi_devs, *ws):
        lead = x.shape[:-1]
        x2 = x.reshape(-1, x.shape[-1])
        if x2.dtype not in (torch.bfloat16, torch.float32):
            x2 = x2.float()
        ctx.shard = shard
        out_dtype = x.dtype if x.dtype in (torch.bfloat16, torch.float32) else torch.float32
        ys, ctx.lctxs = [], []
        # the first layer quantizes x in one fused pass (X_q, M_x and its own X_t); the others reuse its X_q
        x_q = None
        for w, xi, xd in zip(ws, xis, xi_devs):
            y, lctx = qlinear.forward(x2, w.detach(), scheme=scheme, hadamard=hadamard, out_dtype=out_dtype,
                                      check_finite=nonfinite_flag(x.device), bwd_xi=int(xi), bwd_rounding=rounding,
                                      token_offset=shard[0], total_tokens=shard[1], x_q=x_q, bwd_xi_dev=xd)
            x_q = lctx.x_q
            ys.append(y.reshape(*lead, w.shape[0]))
            ctx.lctxs.append(lctx)
        ctx.xis, ctx.rounding, ctx.x_shape, ctx.x_dtype = [int(v) for v in xis], rounding, x.shape, x.dtype
        ctx.w_dtypes = [w.dtype for w in ws]
        return tuple(ys)

    @staticmethod
    def backward(ctx, *dys):
        dx_dtype = ctx.x_dtype if ctx.x_dtype in (torch.bfloat16, torch.float32) else torch.float32
        dx_sum, dws = None, []
        for dy, lctx, xi, wdt in zip(dys, ctx.lctxs, ctx.xis, ctx.w_dtypes):
            dy2 = dy.reshape(-1, dy.shape[-1])
            if dy2.dtype not in (torch.bfloat16, torch.float32):
                dy2 = dy2.float()
            # the layers' dx are summed in x's dtype (as autograd would accumulate them) by the dx GEMM's
            # epilogue adding into the first layer's dx (QT_EPI_ACCUMULATE): no separate add pass
            dx_sum, dw = qlinear.backward(dy2.contiguous(), lctx, xi, ctx.rounding, dx_dtype=dx_dtype,
                                          dw_dtype=torch.float32, check_finite=nonfinite_flag(dy2.device),
                                          token_offset=ctx.shard[0], total_tokens=ctx.shard[1],
                                          dx_accumulate=dx_sum)
            dws.append(dw.to(wdt))
        ctx.lctxs = None
        return (dx_sum.reshape(ctx.x_shape), None, None, None, None, None, None, *dws)


def quartet_linear_group(x, mods):
    """Apply QuartetLinear modules that share the input x with one forward quantization of x."""
    m0 = mods[0]
    if (m0.scheme.kind == "sr_absmax" or any(m.rounding != m0.rounding or m.hadamard != m0.hadamard
                                             or m.scheme is not m0.scheme or m.token_shard != m0.token_shard
                                             for m in mods)):
        return tuple(m(x) for m in mods)
    xis = []
    for m in mods:
        xis.append(m.xi())
        if m.training:
            m.step += 1
    return QuartetLinearGroupFn.apply(x, xis, m0.rounding, m0.hadamard, m0.scheme, m0.token_shard,
                                      [m.xi_slot for m in mods], *[m.weight for m in mods])


def quartet_linear(x, w, xi: int, rounding: str = "rtn", hadamard: bool = True,
                   scheme: qlinear.QuantScheme = qlinear.QUEST, token_offset: int = 0,
                   total_tokens: int | None = None):
    return QuartetLinearFn.apply(x, w, xi, rounding, hadamard, scheme, (int(token_offset), total_tokens))


def set_token_shard(model: torch.nn.Module, token_offset: int, total_tokens: int | None) -> None:
    """Place every QuartetLinear of `model` on a data-parallel token shard: this rank's rows are tokens
    [token_offset, token_offset + local) of a global batch of `total_tokens` (row = sequence * seq_len +
    position).  Their token-axis randomized-Hadamard signs and stochastic-rounding stream positions are then
    the single-GPU ones, so the ranks together compute the single-GPU step."""
    for m in model.modules():
        if isinstance(m, QuartetLinear):
            m.token_shard = (int(token_offset), None if total_tokens is None else int(total_tokens))


class QuartetLinear(torch.nn.Module):
    """Bias-free MXFP4 linear layer (Quartet Alg. 1) with an fp32 master weight."""

    def __init__(self, in_features: int, out_features: int, *, seed: int = 0, layer_id: int = 0,
                 rounding: str = "rtn", hadamard: bool = True, scheme: qlinear.QuantScheme = qlinear.QUEST,
                 device=None, dtype=torch.float32):
        super().__init__()
        if in_features % 32 or out_features % 32:
            raise ValueError("Quartet linear dimensions must be multiples of 32")
        self.in_features, self.out_features = in_features, out_features
        self.weight = torch.nn.Parameter(torch.empty(out_features, in_features, device=device, dtype=dtype))
        self.seed, self.layer_id = int(seed), int(layer_id)
        self.rounding, self.hadamard, self.scheme = rounding, hadamard, scheme
        self.step = 0
        self.token_shard: tuple = (0, None)   # (token offset, global tokens) of this rank: set_token_shard
        # (uint64 device tensor, index): the backward seed of the current step lives on the device (a training step
        # captured as one CUDA graph, llama.LlamaQuartet.use_device_seeds); xi() is then a placeholder
        self.xi_slot = None
        torch.nn.init.normal_(self.weight, std=1.0 / math.sqrt(in_features))

    def xi(self) -> int:
        if self.xi_slot is not None:
            return DEVICE_XI
        return derive_seed(derive_seed(self.seed, 4, self.step), self.layer_id)

    def forward(self, x):
        xi = self.xi()
        if self.training:
            self.step += 1
        return QuartetLinearFn.apply(x, self.weight, xi, self.rounding, self.hadamard, self.scheme, self.token_shard,
                                     self.xi_slot)

    def extra_repr(self) -> str:
        return (f"in_features={self.in_features}, out_features={self.out_features}, "
                f"scheme={self.scheme.kind}, rounding={self.rounding}, hadamard={self.hadamard}")
