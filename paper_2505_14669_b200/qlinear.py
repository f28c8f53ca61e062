"""Quartet linear layer (Alg. 1) on B200: the functional forward / backward pair.

Mirrors the reference's layer seam one-to-one (mx4train/qlinear.py):

    forward(x, w, scheme=QUEST, policy=DEFAULT_POLICY, hadamard=True, seed=None) -> (y, LayerContext)
        qlinear.py:114-165
    backward(dy, ctx, xi, rounding="rtn") -> (dx, dw)
        qlinear.py:178-252

same argument meaning, same ValueError cases, same seeds / stream tags, bit-identical quantizer
outputs.  Tensors are CUDA torch tensors; every step runs in libquartet_b200.so:

    forward : X_q, M_x = QuEST(H32(x));  W_q, M_w = QuEST(H32(w));  y = tcgen05(X_q, W_q)
    dy      : G_q  = Q(H32(dy . s) * 3/4),  Gt_q = Q(H32(dy^T . s) * 3/4)   (qt_quant_dual, one read)
    dX      : Wt_q = Q(H32(deq(W_q)^T . s) * 3/4)  (qt_requant_t)
              dx   = H32(tcgen05(G_q, Wt_q) . M_x) * 16/9   (fused epilogue)
    dW      : Xt_q = Q(H32(deq(X_q)^T . s) * 3/4)  (qt_requant_t)
              dw   = H32(tcgen05(Gt_q, Xt_q) . M_w) * 16/9

Only the reference's default GemmPolicy (single accumulation, quantized operands) runs on the GPU;
its double / exact policies are CPU test modes and are served by the oracle, not here.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .mxfp4 import (GROUP, MXOperand, derive_seed, gemm, quant_cols, quant_dual, quant_fused, quant_rows, sign_bits,
                    sign_bits_pair, sign_bits_pair_dev)

PRE_SCALE = 0.75                     # qlinear.py:36
POST_SCALE = 16.0 / 9.0              # qlinear.py:37
_POST_F32 = float(torch.tensor(16.0 / 9.0, dtype=torch.float32))  # dt(POST_SCALE), qlinear.py:210
_TAG_FWD_X, _TAG_FWD_W = 11, 12      # qlinear.py:40
_TAG_BWD_G1, _TAG_BWD_W, _TAG_BWD_G2, _TAG_BWD_X = 21, 22, 23, 24   # qlinear.py:41

KINDS = ("rtn_absmax", "sr_absmax", "quest")


@dataclass(frozen=True)
class QuantScheme:
    """quantizers.QuantScheme (quantizers.py:29-53)."""

    kind: str
    group_size: int = GROUP
    clip_candidates: int = 64
    clip_range: tuple = (1.0 / 16.0, 1.0)

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown scheme kind {self.kind!r}")
        lo, hi = self.clip_range
        if not (0.0 < lo <= hi <= 1.0):
            raise ValueError(f"invalid clip_range {self.clip_range}")
        if self.clip_candidates < 2:
            raise ValueError("clip_candidates must be >= 2")


RTN_ABSMAX = QuantScheme("rtn_absmax")
SR_ABSMAX = QuantScheme("sr_absmax")
QUEST = QuantScheme("quest")


@dataclass(frozen=True)
class GemmPolicy:
    """qlinear.GemmPolicy (qlinear.py:44-71)."""

    accumulation: str = "single"
    operand_path: str = "quantized"

    def __post_init__(self):
        if self.accumulation not in ("single", "double"):
            raise ValueError(f"unknown accumulation {self.accumulation!r}")
        if self.operand_path not in ("quantized", "exact"):
            raise ValueError(f"unknown operand path {self.operand_path!r}")

    @property
    def exact(self) -> bool:
        return self.operand_path == "exact"


DEFAULT_POLICY = GemmPolicy()
EXACT_POLICY = GemmPolicy(accumulation="double", operand_path="exact")


@dataclass
class LayerContext:
    """qlinear.LayerContext (qlinear.py:74-87); masks live in the operands as bitmaps."""

    x_q: MXOperand
    w_q: MXOperand
    scheme: QuantScheme
    policy: GemmPolicy
    hadamard: bool
    batch: int
    d_in: int
    d_out: int

    # transposed backward operands built at forward time (forward(..., bwd_xi=...)); see _Eager
    eager: "_Eager | None" = None

    @property
    def m_x(self) -> torch.Tensor:
        return self.x_q.mask_bool()

    @property
    def m_w(self) -> torch.Tensor:
        return self.w_q.mask_bool()


@dataclass
class _Eager:
    """X_t, W_t and the sign bitmaps of backward(xi) quantized during forward (qt_quant_fused).

    They are exactly what backward would compute from the saved X_q / W_q (qlinear.py:206-207, 215, 235),
    so backward uses them when called with the same xi, rounding and token shard, and recomputes
    them otherwise."""

    xi: int
    rounding: str
    token_offset: int
    total: int
    xt_q: MXOperand
    wt_q: MXOperand
    d_signs: torch.Tensor | None
    t_signs: torch.Tensor | None


def _check_policy(policy: GemmPolicy, scheme: QuantScheme) -> None:
    if policy.exact or policy.accumulation != "single":
        raise NotImplementedError(
            "the B200 path implements the default policy (fp32 accumulation of MXFP4 operands); "
            "double/exact policies are CPU test modes of the reference (see oracle/)")
    if scheme.group_size != GROUP:
        raise NotImplementedError("MXFP4 on tcgen05 uses 32-element scale groups")
    if scheme.kind == "quest" and scheme.clip_range[0] != 1.0 / 16.0:
        raise NotImplementedError("QuEST kernel is specialised for clip_range[0] = 1/16")


def _err_flag(device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


def _err_for(check_finite, device):
    """check_finite: True -> a fresh device flag, checked (one host sync) before returning; False -> no check;
    a device int32 tensor -> OR the quantizers' non-finite bit into it and return without syncing (the caller
    checks once later, e.g. nn.raise_if_nonfinite at the end of a training step)."""
    if isinstance(check_finite, torch.Tensor):
        return check_finite
    return _err_flag(device) if check_finite else None


def _raise_if_nonfinite(err: torch.Tensor | None, check_finite=True) -> None:
    if err is not None and not isinstance(check_finite, torch.Tensor) and int(err.item()) != 0:
        raise ValueError("non-finite input")


def quantize_operand(m: torch.Tensor, scheme: QuantScheme, hadamard: bool, seed: int | None = None,
                     err: torch.Tensor | None = None, row_offset: int = 0) -> MXOperand:
    """transform_last_axis + apply_scheme (qlinear.py:139-157) as one fused kernel.  row_offset: the first
    row's index in the full matrix (a data-parallel token shard), so that sr_absmax draws the single-GPU
    stream positions (row * cols + col, quantizers.py:79-84)."""
    transform = _lib.QT_TRANSFORM_HADAMARD if hadamard else _lib.QT_TRANSFORM_NONE
    if scheme.kind == "quest":
        return quant_rows(m, transform, _lib.QT_ROUND_QUEST, want_mask=True, err=err)
    if scheme.kind == "rtn_absmax":
        op = quant_rows(m, transform, _lib.QT_ROUND_RTN, want_mask=True, err=err)
    else:
        op = quant_rows(m, transform, _lib.QT_ROUND_SR, sr_seed=seed, counter_start=row_offset * m.shape[1],
                        want_mask=True, err=err)
    return op


def forward(x: torch.Tensor, w: torch.Tensor, scheme: QuantScheme = QUEST, policy: GemmPolicy = DEFAULT_POLICY,
            hadamard: bool = True, seed: int | None = None, out_dtype: torch.dtype = torch.float32,
            check_finite: bool = True, bwd_xi: int | None = None, bwd_rounding: str = "rtn", token_offset: int = 0,
            total_tokens: int | None = None, x_q: MXOperand | None = None, bwd_xi_dev: tuple | None = None):
    """y = x @ w.T through the quantized pipeline; returns (y, context)  (qlinear.py:114-165).

    ``x_q``: the forward operand of x (``quantize_operand(x, ...)``) when several layers read the same x
    (q/k/v, gate/up): X_q and its trust mask depend on x alone, so they are computed once; each layer then
    derives its own X_t from X_q's codes (its own signs), exactly as backward does without eager operands.

    B200 extension: when the backward seed is already known (the training loop derives it per step and
    layer, train.py:346-348), pass it as ``bwd_xi`` (with the backward ``bwd_rounding`` and, for a
    data-parallel token shard, ``token_offset`` / ``total_tokens``): the same single read of x (and of w)
    then also produces the transposed backward operands X_t and W_t (qt_quant_fused), which backward
    reuses instead of re-reading X_q / W_q.  Results are identical either way."""
    _check_policy(policy, scheme)
    _check_out_dtype("out_dtype", out_dtype)
    if x.dim() != 2 or w.dim() != 2:
        raise ValueError("x and w must be 2-D")
    batch, d_in = x.shape
    d_out, d_in_w = w.shape
    if d_in != d_in_w:
        raise ValueError(f"shape mismatch: x has {d_in} features, w has {d_in_w}")
    g = scheme.group_size
    if d_in % g != 0:
        raise ValueError(f"input dimension {d_in} not divisible by block size {g}")
    sx = sw = None
    if scheme.kind == "sr_absmax":
        if seed is None:
            raise ValueError("sr_absmax forward requires a seed")
        sx = derive_seed(seed, _TAG_FWD_X)
        sw = derive_seed(seed, _TAG_FWD_W)
    err = _err_for(check_finite, x.device)
    eager = None
    if x_q is not None and (x_q.rows != batch or x_q.cols != d_in):
        raise ValueError("shared x_q does not match x")
    if bwd_xi_dev is not None and (bwd_xi is None or batch % g or d_out % g or scheme.kind == "sr_absmax"):
        raise NotImplementedError("device-resident seeds need bwd_xi, 32-multiple batch / d_out and a QuEST or RTN "
                                  "forward scheme")
    if bwd_xi is not None and bwd_rounding in ("rtn", "sr", "sr_fast") and batch % g == 0 and d_out % g == 0:
        total = batch if total_tokens is None else int(total_tokens)
        if token_offset % g or token_offset < 0 or token_offset + batch > total:
            raise ValueError(f"token shard [{token_offset}, +{batch}) invalid for {total} tokens (block {g})")
        rc = _rounding_code(bwd_rounding)
        sr = bwd_rounding in ("sr", "sr_fast")
        row_rc = {"quest": _lib.QT_ROUND_QUEST, "rtn_absmax": _lib.QT_ROUND_RTN, "sr_absmax": _lib.QT_ROUND_SR}[scheme.kind]
        fwd_t = _lib.QT_TRANSFORM_HADAMARD if hadamard else _lib.QT_TRANSFORM_NONE
        bwd_t = _lib.QT_TRANSFORM_RANDOMIZED if hadamard else _lib.QT_TRANSFORM_NONE
        if bwd_xi_dev is not None and sr:
            raise NotImplementedError("device-resident seeds (captured training steps) support rounding='rtn'")
        if not hadamard:
            d_signs, t_signs = None, None
        elif bwd_xi_dev is not None:   # the step's seed lives on the device (a captured training step)
            d_signs, t_signs = sign_bits_pair_dev(bwd_xi_dev, d_out, batch, x.device, start_b=token_offset)
        else:
            d_signs, t_signs = sign_bits_pair(bwd_xi, d_out, batch, x.device, start_b=token_offset)
        x_seed = derive_seed(bwd_xi, _TAG_BWD_X) if sr else 0
        if x_q is None:
            x_q, xt_q = quant_fused(x, row_rc, rc, transform=fwd_t, col_transform=bwd_t, col_signs=t_signs,
                                    col_prescale=PRE_SCALE, sr_seed=sx or 0, counter_start=token_offset * d_in,
                                    col_seed=x_seed, col_counter_start=token_offset, col_counter_ld=total, err=err)
        else:  # shared X_q: this layer's X_t from its codes, as backward does without eager operands
            xt_q = quant_cols(x_q, rc, transform=bwd_t, signs=t_signs, prescale=PRE_SCALE, sr_seed=x_seed,
                              counter_start=token_offset, counter_ld=total, err=err)
        w_q, wt_q = quant_fused(w, row_rc, rc, transform=fwd_t, col_transform=bwd_t, col_signs=d_signs,
                                col_prescale=PRE_SCALE, sr_seed=sw or 0,
                                col_seed=derive_seed(bwd_xi, _TAG_BWD_W) if sr else 0, err=err)
        eager = _Eager(int(bwd_xi), bwd_rounding, int(token_offset), total, xt_q, wt_q, d_signs, t_signs)
    else:
        if token_offset % g or token_offset < 0:
            raise ValueError(f"token offset {token_offset} must be a non-negative multiple of {g}")
        if x_q is None:
            x_q = quantize_operand(x, scheme, hadamard, sx, err, row_offset=token_offset)
        w_q = quantize_operand(w, scheme, hadamard, sw, err)
    if d_out % g:   # ragged d_out (the GEMM's N axis is whole blocks): zero rows of W_q, sliced off y
        y = gemm(x_q, w_q.pad_rows(-(-d_out // g) * g), out_dtype=out_dtype)[:, :d_out].contiguous()
    else:
        y = gemm(x_q, w_q, out_dtype=out_dtype)
    _raise_if_nonfinite(err, check_finite)
    ctx = LayerContext(x_q=x_q, w_q=w_q, scheme=scheme, policy=policy, hadamard=hadamard,
                       batch=batch, d_in=d_in, d_out=d_out, eager=eager)
    return y, ctx


def _backward_ragged(dy, ctx, xi, rounding, rc, dx_dtype, dw_dtype, check_finite, return_operands, token_offset,
                     total, dx_accumulate):
    """backward with hadamard=False and d_out or batch not a multiple of 32: the reference quantizes a
    ragged trailing group of G (along d_out), W_t (along d_out), G_t and X_t (along tokens) (qlinear.py:
    212-250, codec ragged groups).  Every operand is built from the zero-padded matrix: a zero pads a group
    without changing its absmax scale, encodes as code 0 under RTN and SR alike (p = 0), and adds nothing
    to the dx / dw contractions; the SR stream positions are those of the unpadded matrices (counter
    leading dimensions d_out and the token count).  Operands are returned padded (return_operands)."""
    g = ctx.scheme.group_size
    B, D = ctx.batch, ctx.d_out
    Bp, Dp = -(-B // g) * g, -(-D // g) * g
    sr = rounding in ("sr", "sr_fast")
    none = _lib.QT_TRANSFORM_NONE
    err = _err_for(check_finite, dy.device)
    dy_p = torch.zeros((Bp, Dp), dtype=dy.dtype if dy.dtype in (torch.bfloat16, torch.float32) else torch.float32,
                       device=dy.device)
    dy_p[:B, :D] = dy
    x_q, w_q = ctx.x_q.pad_rows(Bp), ctx.w_q.pad_rows(Dp)
    g_q = quant_rows(dy_p, none, rc, prescale=PRE_SCALE, sr_seed=derive_seed(xi, _TAG_BWD_G1) if sr else 0,
                     counter_start=token_offset * D, counter_ld=D, err=err)
    wt_q = quant_cols(w_q, rc, transform=none, prescale=PRE_SCALE, sr_seed=derive_seed(xi, _TAG_BWD_W) if sr else 0,
                      counter_ld=D, err=err)
    dx_dt = dx_accumulate.dtype if dx_accumulate is not None else dx_dtype
    dx = gemm(g_q, wt_q, out_dtype=dx_dt, mask=x_q.mask, hadamard=False, scale=_POST_F32)[:B]
    if dx_accumulate is not None:
        dx = dx_accumulate.add_(dx)
    gt_q = quant_cols(dy_p, rc, transform=none, prescale=PRE_SCALE,
                      sr_seed=derive_seed(xi, _TAG_BWD_G2) if sr else 0, counter_start=token_offset,
                      counter_ld=total, err=err)
    xt_q = quant_cols(x_q, rc, transform=none, prescale=PRE_SCALE, sr_seed=derive_seed(xi, _TAG_BWD_X) if sr else 0,
                      counter_start=token_offset, counter_ld=total, err=err)
    dw = gemm(gt_q, xt_q, out_dtype=dw_dtype, mask=w_q.mask, hadamard=False, scale=_POST_F32)[:D]
    _raise_if_nonfinite(err, check_finite)
    if return_operands:
        return dx, dw, {"g_q": g_q, "wt_q": wt_q, "gt_q": gt_q, "xt_q": xt_q}
    return dx, dw


def _check_out_dtype(name: str, dt: torch.dtype) -> None:
    """The GEMM epilogues store bf16 or fp32 only; reject anything else before any device work."""
    if dt not in (torch.float32, torch.bfloat16):
        raise ValueError(f"{name} must be torch.float32 or torch.bfloat16, got {dt}")


def _rounding_code(rounding: str) -> int:
    if rounding == "rtn":
        return _lib.QT_ROUND_RTN
    if rounding == "sr":
        return _lib.QT_ROUND_SR
    if rounding == "sr_fast":   # B200 extension: hardware SR (cvt.rs), unbiased to 2^-16 of a step (not the reference's draws)
        return _lib.QT_ROUND_SR_FAST
    if rounding == "exact":
        raise NotImplementedError("rounding='exact' skips quantization: a CPU test mode (oracle), not a GPU path")
    raise ValueError(f"unknown backward rounding {rounding!r}")


def backward(dy: torch.Tensor, ctx: LayerContext, xi: int, rounding: str = "rtn",
             dx_dtype: torch.dtype = torch.float32, dw_dtype: torch.dtype = torch.float32,
             check_finite: bool = True, return_operands: bool = False, token_offset: int = 0,
             total_tokens: int | None = None, dx_accumulate: torch.Tensor | None = None):
    """Input and weight gradients from the saved context and upstream dy (qlinear.py:178-252).

    dx_accumulate: an existing [batch, d_in] gradient buffer that this layer's dx is added into by the
    GEMM epilogue (several layers reading the same x, nn.QuartetLinearGroupFn); the returned dx is that
    buffer, bit-identical to dx_accumulate.add_(dx).

    Data-parallel shards: a rank holding tokens [token_offset, token_offset + batch) of a global batch of
    `total_tokens` passes both; its randomized-Hadamard signs and stochastic-rounding stream positions
    along the token axis are then the global ones, so its G / G_t / X_t operands are exactly the
    corresponding slices of the single-GPU operands, its dx rows are exactly the single-GPU dx rows,
    and the sum of the ranks' dw equals the single-GPU dw up to fp32 summation order (the masked
    Hadamard epilogue is linear).  token_offset must be a multiple of 32.

    d_out and batch must be multiples of the block size with hadamard=True (ValueError, as the reference);
    with hadamard=False the reference quantizes a ragged trailing group, and so does this path
    (_backward_ragged)."""
    if rounding not in ("exact", "rtn", "sr", "sr_fast"):
        raise ValueError(f"unknown backward rounding {rounding!r}")
    rc = _rounding_code(rounding)
    _check_out_dtype("dw_dtype", dw_dtype)
    if dx_accumulate is None:
        _check_out_dtype("dx_dtype", dx_dtype)
    if tuple(dy.shape) != (ctx.batch, ctx.d_out):
        raise ValueError(f"dy shape {tuple(dy.shape)}, expected {(ctx.batch, ctx.d_out)}")
    g = ctx.scheme.group_size
    if ctx.hadamard and ctx.d_out % g != 0:
        raise ValueError(f"output dimension {ctx.d_out} not divisible by block size {g}")
    if ctx.hadamard and ctx.batch % g != 0:
        raise ValueError(f"batch size {ctx.batch} not divisible by block size {g}")
    total = ctx.batch if total_tokens is None else int(total_tokens)
    if token_offset % g or token_offset < 0 or token_offset + ctx.batch > total:
        raise ValueError(f"token shard [{token_offset}, +{ctx.batch}) invalid for {total} tokens (block {g})")
    if ctx.d_out % g or ctx.batch % g:
        return _backward_ragged(dy, ctx, xi, rounding, rc, dx_dtype, dw_dtype, check_finite, return_operands,
                                token_offset, total, dx_accumulate)
    dev = dy.device
    transform = _lib.QT_TRANSFORM_RANDOMIZED if ctx.hadamard else _lib.QT_TRANSFORM_NONE
    ea = ctx.eager
    if ea is not None and (ea.xi, ea.rounding, ea.token_offset, ea.total) != (int(xi), rounding, token_offset, total):
        ea = None
    if ea is not None:
        d_signs, t_signs = ea.d_signs, ea.t_signs
    else:
        # along d_out and along tokens, one launch
        d_signs, t_signs = (sign_bits_pair(xi, ctx.d_out, ctx.batch, dev, start_b=token_offset) if ctx.hadamard
                            else (None, None))
    sr = rounding in ("sr", "sr_fast")
    err = _err_for(check_finite, dev)

    # both dy operands from one read of dy: G (rows, qlinear.py:214) and G_t (cols, qlinear.py:234)
    g_q, gt_q = quant_dual(dy, rc, transform=transform, signs=d_signs, col_signs=t_signs, prescale=PRE_SCALE,
                           seed_rows=derive_seed(xi, _TAG_BWD_G1) if sr else 0,
                           row_counter_start=token_offset * ctx.d_out,
                           seed_cols=derive_seed(xi, _TAG_BWD_G2) if sr else 0,
                           col_counter_start=token_offset, col_counter_ld=total, err=err)

    # input gradient: contract over d_out (qlinear.py:212-230)
    wt_q = ea.wt_q if ea is not None else quant_cols(ctx.w_q, rc, transform=transform, signs=d_signs,
                                                     prescale=PRE_SCALE,
                                                     sr_seed=derive_seed(xi, _TAG_BWD_W) if sr else 0, err=err)
    dx = gemm(g_q, wt_q, out_dtype=dx_dtype, mask=ctx.x_q.mask, hadamard=ctx.hadamard, scale=_POST_F32,
              out=dx_accumulate, accumulate=dx_accumulate is not None)

    # weight gradient: contract over batch (qlinear.py:232-250)
    xt_q = ea.xt_q if ea is not None else quant_cols(ctx.x_q, rc, transform=transform, signs=t_signs,
                                                     prescale=PRE_SCALE,
                                                     sr_seed=derive_seed(xi, _TAG_BWD_X) if sr else 0,
                                                     counter_start=token_offset, counter_ld=total, err=err)
    dw = gemm(gt_q, xt_q, out_dtype=dw_dtype, mask=ctx.w_q.mask, hadamard=ctx.hadamard, scale=_POST_F32)
    _raise_if_nonfinite(err, check_finite)
    if return_operands:
        return dx, dw, {"g_q": g_q, "wt_q": wt_q, "gt_q": gt_q, "xt_q": xt_q}
    return dx, dw
