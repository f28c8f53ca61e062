"""Llama-style causal LM whose every linear layer is a Quartet MXFP4 layer (BASELINE configs 2, 4, 5).

The caller of the hot path: token embedding -> N x [RMSNorm -> attention (q, k, v,
o: QuartetLinear, RoPE, causal SDPA in bf16) -> RMSNorm -> SwiGLU MLP (gate, up, down: QuartetLinear)]
-> RMSNorm -> LM head (QuartetLinear).  Attention and norms stay in bf16/fp32 torch; every matmul with a
weight runs through libquartet_b200 (forward QuEST + H32, backward RHT + RTN/SR, tcgen05 MXFP4 GEMMs).

Training follows the reference's loop semantics (mx4train/train.py:58-85, 325-382) at Llama scale:
AdamW (beta 0.9 / 0.95, eps 1e-8, decoupled weight decay 0.1) on fp32 master weights, global-norm
clipping at 1.0, linear warm-up over 10 % of the steps then cosine decay (lr_at, train.py:76-85), and a
fresh backward seed per step and layer (derive_seed(derive_seed(seed, 4, step), layer), train.py:346-348).
Model shapes follow PAPER.md Appendix (hyper-parameter table): 30M = 6 x 640 (5 heads), 200M = 10 x 1280
(10 heads), sequence 512; the 7B block uses the Llama-2-7B dims 4096 / 11008 / 32 heads.

Data parallelism: one process per GPU; each rank holds whole sequences, so the only exchange is the
gradient all-reduce (bf16 on the wire, NCCL over NVLink), done once per step over one flat bucket.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import _lib
from .mxfp4 import _stream
from .nn import QuartetLinear, nonfinite_flag, quartet_linear_group, set_token_shard

GROUP = 32


@dataclass(frozen=True)
class LlamaConfig:
    n_layer: int
    d_model: int
    n_head: int
    vocab: int = 32000
    seq_len: int = 512
    d_ff: int | None = None          # SwiGLU hidden size; default 8/3 d rounded up to 256
    rounding: str = "rtn"
    rope_base: float = 10000.0
    linear: str = "quartet"          # "quartet" (MXFP4, the product) or "bf16" (the comparator arm)

    @property
    def hidden(self) -> int:
        if self.d_ff is not None:
            return self.d_ff
        h = int(8 * self.d_model / 3)
        return (h + 255) // 256 * 256

    def n_params(self, embeddings: bool = False) -> int:
        d, h = self.d_model, self.hidden
        n = self.n_layer * (4 * d * d + 3 * d * h + 2 * d) + d
        return n + (2 * self.vocab * d if embeddings else 0)


PRESETS = {
    "30m": LlamaConfig(n_layer=6, d_model=640, n_head=5),
    "50m": LlamaConfig(n_layer=7, d_model=768, n_head=6),
    "100m": LlamaConfig(n_layer=8, d_model=1024, n_head=8),
    "200m": LlamaConfig(n_layer=10, d_model=1280, n_head=10),
    "7b": LlamaConfig(n_layer=32, d_model=4096, n_head=32, d_ff=11008, seq_len=8192),
}
PAPER_LR = {"30m": 1.2e-3, "50m": 1.2e-3, "100m": 6e-4, "200m": 3e-4, "7b": 9.375e-6}


class RMSNorm(torch.nn.Module):
    def __init__(self, d: int, eps: float = 1e-6, device=None):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.ones(d, device=device))
        self.eps = eps

    def forward(self, x):  # bf16 in / out, fp32 statistics and weight
        d = x.shape[-1]
        if _fused_norm_ok(d):  # csrc/glue.cu, one pass each way
            return _RMSNormFn.apply(x.to(torch.bfloat16), self.weight, self.eps)
        return F.rms_norm(x.to(torch.bfloat16), (d,), self.weight.to(torch.bfloat16), self.eps)


def _fused_norm_ok(d: int) -> bool:
    return d % 8 == 0 and (d <= 2048 or (d % 2048 == 0 and d <= 8192))


class _AddRMSNormFn(torch.autograd.Function):
    """(h, n) = (x + y, rmsnorm(x + y)) in one pass (y None: h = x passed through).  Backward gets the gradients of
    both outputs and returns dx = dh + rmsnorm'(dn) from one kernel (qt_rmsnorm_res), so the residual stream's two
    consumers need no separate gradient accumulation.  Bit-identical to `h = x + y; n = norm(h)` with autograd's
    bf16 accumulation (each sum is rounded once to bf16, as torch's add)."""

    @staticmethod
    def forward(ctx, x, y, w, eps):
        x2 = x.contiguous().view(-1, x.shape[-1])
        n = torch.empty_like(x2)
        rstd = torch.empty(x2.shape[0], dtype=torch.float32, device=x.device)
        if y is None:
            h = x2
            rc = _lib.load().qt_rmsnorm(x2.data_ptr(), w.data_ptr(), None, n.data_ptr(), rstd.data_ptr(), None,
                                        x2.shape[0], x2.shape[1], float(eps), 0, _stream(x.device))
        else:
            y2 = y.contiguous().view(x2.shape)
            h = torch.empty_like(x2)
            rc = _lib.load().qt_rmsnorm_res(x2.data_ptr(), y2.data_ptr(), w.data_ptr(), None, n.data_ptr(),
                                            h.data_ptr(), rstd.data_ptr(), None, x2.shape[0], x2.shape[1], float(eps),
                                            0, _stream(x.device))
        _lib.check(rc, "qt_rmsnorm_res")
        ctx.save_for_backward(h, w, rstd)
        ctx.eps = eps
        ctx.has_y = y is not None
        h_out = h.view(x.shape) if y is not None else x.view_as(x)
        return h_out, n.view(x.shape)

    @staticmethod
    def backward(ctx, dh, dn):
        h2, w, rstd = ctx.saved_tensors
        dw = torch.zeros(h2.shape[1], dtype=torch.float32, device=h2.device)
        if dn is None:
            dx = dh.contiguous().view(h2.shape)
        else:
            dn2 = dn.contiguous().view(h2.shape)
            dx = torch.empty_like(h2)
            res = None if dh is None else dh.contiguous().view(h2.shape)
            _lib.check(_lib.load().qt_rmsnorm_res(h2.data_ptr(), None if res is None else res.data_ptr(), w.data_ptr(),
                                                  dn2.data_ptr(), dx.data_ptr(), None, rstd.data_ptr(), dw.data_ptr(),
                                                  h2.shape[0], h2.shape[1], float(ctx.eps), 1, _stream(h2.device)),
                       "qt_rmsnorm_res")
        shape = dn.shape if dn is not None else dh.shape
        return dx.view(shape), (dx.view(shape) if ctx.has_y else None), dw.to(w.dtype), None


def add_rmsnorm(x, y, norm: "RMSNorm"):
    """(x + y, norm(x + y)) with the residual add fused into the norm's kernels (y None: (x, norm(x)) with the
    residual gradient fused into the norm's backward)."""
    d = x.shape[-1]
    if _fused_norm_ok(d):
        return _AddRMSNormFn.apply(x.to(torch.bfloat16), None if y is None else y.to(torch.bfloat16), norm.weight,
                                   norm.eps)
    h = x if y is None else x + y
    return h, norm(h)


class _RMSNormFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, w, eps):
        x2 = x.contiguous().view(-1, x.shape[-1])
        out = torch.empty_like(x2)
        rstd = torch.empty(x2.shape[0], dtype=torch.float32, device=x.device)
        _lib.check(_lib.load().qt_rmsnorm(x2.data_ptr(), w.data_ptr(), None, out.data_ptr(), rstd.data_ptr(), None,
                                          x2.shape[0], x2.shape[1], float(eps), 0, _stream(x.device)), "qt_rmsnorm")
        ctx.save_for_backward(x2, w, rstd)
        ctx.eps = eps
        return out.view(x.shape)

    @staticmethod
    def backward(ctx, dy):
        x2, w, rstd = ctx.saved_tensors
        dy2 = dy.contiguous().view(x2.shape)
        dx = torch.empty_like(x2)
        dw = torch.zeros(x2.shape[1], dtype=torch.float32, device=x2.device)
        _lib.check(_lib.load().qt_rmsnorm(x2.data_ptr(), w.data_ptr(), dy2.data_ptr(), dx.data_ptr(), rstd.data_ptr(),
                                          dw.data_ptr(), x2.shape[0], x2.shape[1], float(ctx.eps), 1,
                                          _stream(x2.device)), "qt_rmsnorm")
        return dx.view(dy.shape), dw.to(w.dtype), None


def _rope(seq: int, dh: int, base: float, device):
    """Rotary tables in the half-split (GPT-NeoX) layout, bf16 [seq, dh]."""
    inv = 1.0 / (base ** (torch.arange(0, dh, 2, device=device, dtype=torch.float32) / dh))
    t = torch.arange(seq, device=device, dtype=torch.float32)
    f = torch.outer(t, inv)
    f = torch.cat((f, f), dim=-1)
    return torch.cos(f).to(torch.bfloat16), torch.sin(f).to(torch.bfloat16)


def _apply_rope_torch(x, cos, sin):  # x [B, H, S, dh] bf16 (reference formulation, tests)
    h = x.shape[-1] // 2
    rot = torch.cat((-x[..., h:], x[..., :h]), dim=-1)
    S = x.shape[2]
    return x * cos[:S] + rot * sin[:S]


def _rope_call(x, cos, sin, backward: bool):
    """x [B, S, H, dh] bf16 (any strides with dh contiguous, e.g. the transposed gradient of attention) ->
    rotated contiguous copy (csrc/glue.cu, one pass)."""
    B, S, H, dh = x.shape
    if x.stride(3) != 1 or any(st % 8 for st in x.stride()[:3]) or x.data_ptr() % 16:
        x = x.contiguous()
    out = torch.empty((B, S, H, dh), dtype=x.dtype, device=x.device)
    _lib.check(_lib.load().qt_rope(x.data_ptr(), out.data_ptr(), B * S, H, dh, S, cos.data_ptr(), sin.data_ptr(),
                                   int(backward), x.stride(0), x.stride(1), x.stride(2), _stream(x.device)),
               "qt_rope")
    return out


class _Rope(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, cos, sin):
        ctx.save_for_backward(cos, sin)
        return _rope_call(x, cos, sin, False)

    @staticmethod
    def backward(ctx, dy):
        cos, sin = ctx.saved_tensors
        return _rope_call(dy, cos, sin, True), None, None


class _SwiGLU(torch.autograd.Function):
    @staticmethod
    def forward(ctx, g, u):
        g, u = g.contiguous(), u.contiguous()
        ctx.save_for_backward(g, u)
        out = torch.empty_like(g)
        _lib.check(_lib.load().qt_swiglu(g.data_ptr(), u.data_ptr(), None, out.data_ptr(), None, g.numel(), 0,
                                         _stream(g.device)), "qt_swiglu")
        return out

    @staticmethod
    def backward(ctx, dy):
        g, u = ctx.saved_tensors
        dy = dy.contiguous()
        dg, du = torch.empty_like(g), torch.empty_like(u)
        _lib.check(_lib.load().qt_swiglu(g.data_ptr(), u.data_ptr(), dy.data_ptr(), dg.data_ptr(), du.data_ptr(),
                                         g.numel(), 1, _stream(g.device)), "qt_swiglu")
        return dg, du


class _CrossEntropy(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, targets):
        logits, targets = logits.contiguous(), targets.contiguous().to(torch.int64)
        rows, vocab = logits.shape
        lse = torch.empty(rows, dtype=torch.float32, device=logits.device)
        loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
        _lib.check(_lib.load().qt_cross_entropy(logits.data_ptr(), targets.data_ptr(), rows, vocab, lse.data_ptr(),
                                                loss.data_ptr(), None, None, 1.0, 0, _stream(logits.device)),
                   "qt_cross_entropy")
        # targets outside [0, vocab) (e.g. ignore_index = -100) contribute nothing and are not counted, as in
        # F.cross_entropy's mean reduction; the count stays on the device (no sync)
        n_valid = ((targets >= 0) & (targets < vocab)).sum().to(torch.float32)
        ctx.save_for_backward(logits, targets, lse, n_valid)
        return loss.sum() / n_valid

    @staticmethod
    def backward(ctx, g):
        logits, targets, lse, n_valid = ctx.saved_tensors
        rows, vocab = logits.shape
        g = (g.detach().to(torch.float32) / n_valid).reshape(1).contiguous()
        d = torch.empty_like(logits)
        _lib.check(_lib.load().qt_cross_entropy(logits.data_ptr(), targets.data_ptr(), rows, vocab, lse.data_ptr(),
                                                None, d.data_ptr(), g.data_ptr(), 1.0, 1,
                                                _stream(logits.device)), "qt_cross_entropy")
        return d, None


def cross_entropy(logits, targets):
    """Mean cross-entropy of bf16 logits [rows, vocab] (vocab % 8 == 0): one pass forward (online
    log-sum-exp), one pass backward (softmax - onehot); torch's F.cross_entropy otherwise."""
    if logits.dtype == torch.bfloat16 and logits.shape[-1] % 8 == 0:
        return _CrossEntropy.apply(logits, targets)
    return F.cross_entropy(logits.float(), targets)


def swiglu(g, u):
    """silu(g) * u, fused forward and backward (bf16)."""
    return _SwiGLU.apply(g, u)


def rope(x, cos, sin):
    """Rotary embedding of x [B, S, H, dh] bf16 (half-split layout), fused forward and backward."""
    return _Rope.apply(x, cos[: x.shape[1]], sin[: x.shape[1]])


class Bf16Linear(torch.nn.Module):
    """The comparator arm of the training benchmarks: a bias-free linear with the same fp32 master weight
    and initialisation as QuartetLinear, computed as a bf16 cuBLAS matmul (standard bf16 mixed precision,
    the paper's BF16 baseline).  Everything else in the model is shared with the Quartet arm."""

    def __init__(self, in_features: int, out_features: int, device=None):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.empty(out_features, in_features, device=device))
        torch.nn.init.normal_(self.weight, std=1.0 / math.sqrt(in_features))

    def forward(self, x):
        return F.linear(x, self.weight.to(x.dtype))


def make_linear(cfg: LlamaConfig, i: int, o: int, seed: int, layer_id: int, device=None):
    if cfg.linear == "bf16":
        return Bf16Linear(i, o, device=device)
    if cfg.linear != "quartet":
        raise ValueError(f"unknown linear kind {cfg.linear!r}")
    return QuartetLinear(i, o, seed=seed, layer_id=layer_id, rounding=cfg.rounding, device=device)


def linear_group(x, mods):
    if isinstance(mods[0], QuartetLinear):
        return quartet_linear_group(x, mods)
    return tuple(m(x) for m in mods)


class Block(torch.nn.Module):
    def __init__(self, cfg: LlamaConfig, index: int, seed: int, device=None):
        super().__init__()
        d, h = cfg.d_model, cfg.hidden
        lid = 16 * index

        def ql(i, o, k):
            return make_linear(cfg, i, o, seed, lid + k, device)

        self.n_head = cfg.n_head
        self.attn_norm, self.mlp_norm = RMSNorm(d, device=device), RMSNorm(d, device=device)
        self.q, self.k, self.v, self.o = ql(d, d, 0), ql(d, d, 1), ql(d, d, 2), ql(d, d, 3)
        self.gate, self.up, self.down = ql(d, h, 4), ql(d, h, 5), ql(h, d, 6)

    def forward(self, x, cos, sin, y=None):
        """x [B, S, d] bf16 residual stream; y: the previous block's pending branch output (added to x inside this
        block's first norm).  Returns (h, y_out) with the block's output h + y_out; the add is left pending for
        the next norm (LlamaQuartet.forward), so every residual add runs fused into an RMSNorm pass."""
        B, S, d = x.shape
        H, dh = self.n_head, d // self.n_head
        x, a = add_rmsnorm(x, y, self.attn_norm)
        q, k, v = linear_group(a, (self.q, self.k, self.v))  # one QuEST read of a for q/k/v
        q = rope(q.view(B, S, H, dh), cos, sin).transpose(1, 2)
        k = rope(k.view(B, S, H, dh), cos, sin).transpose(1, 2)
        v = v.view(B, S, H, dh).transpose(1, 2)
        att = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x, m = add_rmsnorm(x, self.o(att.transpose(1, 2).reshape(B, S, d)), self.mlp_norm)
        g, u = linear_group(m, (self.gate, self.up))
        return x, self.down(swiglu(g, u))


class LlamaQuartet(torch.nn.Module):
    """Decoder-only Llama with all linear layers (attention, MLP, LM head) in Quartet MXFP4."""

    def __init__(self, cfg: LlamaConfig, seed: int = 0, device=None, blocks_only: bool = False):
        super().__init__()
        self.cfg = cfg
        self._seeds = None
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.embed = None if blocks_only else torch.nn.Parameter(
            (torch.randn(cfg.vocab, cfg.d_model, generator=g) * 0.02).to(device))
        self.blocks = torch.nn.ModuleList(Block(cfg, i, seed, device) for i in range(cfg.n_layer))
        self.norm = RMSNorm(cfg.d_model, device=device)
        self.head = None if blocks_only else make_linear(cfg, cfg.d_model, cfg.vocab, seed, 16 * 4096, device)
        # every linear weight from the model's own generator (N(0, 1/d_in), in registration order): the same
        # seed gives the same model in every process, which data-parallel ranks rely on
        with torch.no_grad():
            for m in self.modules():
                if isinstance(m, (QuartetLinear, Bf16Linear)):
                    w = m.weight
                    w.copy_(torch.randn(w.shape, generator=g).div_(math.sqrt(w.shape[1])).to(w.device, w.dtype))
        cos, sin = _rope(cfg.seq_len, cfg.d_model // cfg.n_head, cfg.rope_base, device)
        self.register_buffer("cos", cos, persistent=False)
        self.register_buffer("sin", sin, persistent=False)

    def use_device_seeds(self) -> None:
        """Keep the per-step, per-layer backward seeds on the device (for a training step captured as one CUDA
        graph): every forward in training mode first runs qt_layer_seeds -- xi_l = derive_seed(derive_seed(seed,
        4, step), layer_l) for all Quartet layers, step++ (train.py:346-348, the same values QuartetLinear.xi()
        computes on the host) -- and the layers' sign kernels read xi_l from there.  RTN backward only."""
        mods = [m for m in self.modules() if isinstance(m, QuartetLinear)]
        if not mods or self._seeds is not None:
            return
        steps = {m.step for m in mods}
        seeds = {m.seed for m in mods}
        if len(steps) != 1 or len(seeds) != 1 or any(m.rounding != "rtn" for m in mods):
            raise ValueError("device seeds need Quartet layers at the same step with one seed and rtn rounding")
        dev = mods[0].weight.device
        ids = torch.tensor([m.layer_id for m in mods], dtype=torch.int64, device=dev)
        xi = torch.zeros(len(mods), dtype=torch.int64, device=dev)
        step = torch.tensor([steps.pop()], dtype=torch.int64, device=dev)
        for i, m in enumerate(mods):
            m.xi_slot = (xi, i)
        self._seeds = (xi, ids, step, seeds.pop(), len(mods))

    def _launch_seeds(self) -> None:
        xi, ids, step, seed, n = self._seeds
        rc = _lib.load().qt_layer_seeds(xi.data_ptr(), ids.data_ptr(), n, seed & 0xFFFFFFFFFFFFFFFF, step.data_ptr(),
                                        1, _stream(xi.device))
        if rc:
            raise RuntimeError(f"qt_layer_seeds failed: {rc}")

    def forward(self, tokens=None, x=None):
        if self._seeds is not None and self.training:
            self._launch_seeds()
        if x is None:
            x = F.embedding(tokens, self.embed).to(torch.bfloat16)
        y = None
        for blk in self.blocks:
            x, y = blk(x, self.cos, self.sin, y)
        if self.head is None:
            return x + y
        return self.head(add_rmsnorm(x, y, self.norm)[1])


def lr_at(step: int, steps: int, lr: float, warmup_frac: float = 0.1, lr_floor: float = 0.0) -> float:
    """train.py:76-85: linear warm-up to the peak at warmup_frac * steps, then cosine decay."""
    warmup = max(1, int(round(warmup_frac * steps)))
    if step < warmup:
        return lr * (step + 1) / warmup
    span = max(1, steps - 1 - warmup)
    t = min(step - warmup, span)
    return lr_floor + 0.5 * (lr - lr_floor) * (1.0 + math.cos(math.pi * t / span))


class GradBucket:
    """One flat gradient bucket, all-reduced in bf16 (SUM, then / world) -- the data-parallel exchange."""

    def __init__(self, params, comm_dtype=torch.bfloat16):
        self.params = [p for p in params if p.requires_grad]
        n = sum(p.numel() for p in self.params)
        dev = self.params[0].device
        self.buf = torch.empty(n, dtype=comm_dtype, device=dev)

    def allreduce(self, group=None) -> None:
        import torch.distributed as dist

        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
            return
        world = dist.get_world_size(group)
        off = 0
        for p in self.params:
            n = p.numel()
            self.buf[off:off + n].copy_(p.grad.reshape(-1))
            off += n
        dist.all_reduce(self.buf, group=group)
        self.buf.div_(world)
        off = 0
        for p in self.params:
            n = p.numel()
            p.grad.copy_(self.buf[off:off + n].view_as(p.grad))
            off += n


class OverlappedGradBuckets:
    """Bucketed data-parallel gradient exchange overlapped with backward: parameters are grouped,
    in reverse registration order (roughly the order backward produces their gradients), into buckets of
    about `bucket_mb`; a post-accumulate-grad hook launches a bucket's bf16 all-reduce (async) as soon as its
    last gradient is ready, while backward keeps running on the remaining layers.  finish() waits, divides by
    the world size and copies the means back into .grad.  Same values as GradBucket (bf16 on the wire, one
    SUM per element)."""

    def __init__(self, params, bucket_mb: float = 25.0, comm_dtype=torch.bfloat16, group=None):
        self.params = [p for p in params if p.requires_grad]
        self.group, self.comm_dtype = group, comm_dtype
        self.buckets, cur, size = [], [], 0
        limit = int(bucket_mb * 2**20)
        for p in reversed(self.params):
            cur.append(p)
            size += p.numel() * torch.finfo(comm_dtype).bits // 8
            if size >= limit:
                self.buckets.append(cur)
                cur, size = [], 0
        if cur:
            self.buckets.append(cur)
        self.bucket_of = {}
        for i, b in enumerate(self.buckets):
            for p in b:
                self.bucket_of[p] = i
        self.bufs = [torch.empty(sum(p.numel() for p in b), dtype=comm_dtype, device=b[0].device)
                     for b in self.buckets]
        self._pending = [len(b) for b in self.buckets]
        self._work = [None] * len(self.buckets)
        self._hooks = [p.register_post_accumulate_grad_hook(self._ready) for p in self.params]

    def _active(self) -> bool:
        import torch.distributed as dist

        return dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1

    def _ready(self, p) -> None:
        if not self._active():
            return
        i = self.bucket_of[p]
        self._pending[i] -= 1
        if self._pending[i] == 0:
            import torch.distributed as dist

            off = 0
            for q in self.buckets[i]:
                n = q.numel()
                self.bufs[i][off:off + n].copy_(q.grad.reshape(-1))
                off += n
            self._work[i] = dist.all_reduce(self.bufs[i], group=self.group, async_op=True)

    def finish(self) -> None:
        if not self._active():
            return
        import torch.distributed as dist

        world = dist.get_world_size(self.group)
        for i, b in enumerate(self.buckets):
            if self._work[i] is None:  # a bucket whose grads were not all produced this step
                raise RuntimeError(f"gradient bucket {i} was not reduced (unused parameters?)")
            self._work[i].wait()
            self.bufs[i].div_(world)
            off = 0
            for q in b:
                n = q.numel()
                q.grad.copy_(self.bufs[i][off:off + n].view_as(q.grad))
                off += n
            self._work[i] = None
            self._pending[i] = len(b)


class Trainer:
    """AdamW / clip / schedule of the reference loop (train.py:325-382) around LlamaQuartet, data parallel."""

    def __init__(self, model: torch.nn.Module, steps: int, lr: float, weight_decay: float = 0.1,
                 grad_clip: float = 1.0, betas=(0.9, 0.95), eps: float = 1e-8, graph: bool = False):
        """graph=True (one GPU): after two eager warm-up steps the whole training step -- forward, loss,
        backward, clipping, AdamW -- is captured once as a CUDA graph and replayed, with the per-step layer
        seeds (LlamaQuartet.use_device_seeds) and the learning rate (a device scalar) updated on the device, so
        the host launches one graph per step instead of ~1000 kernels."""
        self.model, self.steps, self.lr, self.grad_clip = model, steps, lr, grad_clip
        params = [p for p in model.parameters() if p.requires_grad]
        self.graph = bool(graph)
        if self.graph:
            self.lr_t = torch.tensor(float(lr_at(0, steps, lr)), dtype=torch.float32, device=params[0].device)
            self.opt = torch.optim.AdamW(params, lr=self.lr_t, betas=betas, eps=eps, weight_decay=weight_decay,
                                         fused=True, capturable=True)
            if hasattr(model, "use_device_seeds"):
                model.use_device_seeds()
        else:
            self.opt = torch.optim.AdamW(params, lr=lr, betas=betas, eps=eps, weight_decay=weight_decay,
                                         fused=params[0].is_cuda)
        self._cuda_graph = None
        self.bucket = OverlappedGradBuckets(params)
        self.step_i = 0
        # non-finite quantizer inputs (the reference raises / stops on them, codec.py:164-170,
        # train.py:341-343): the Quartet layers OR them into a device flag; each step copies it to pinned host
        # memory without a sync and the NEXT step checks the copy, so the check never stalls the launch queue
        dev = params[0].device
        self._flag = nonfinite_flag(dev) if dev.type == "cuda" else None
        self._pending: list = []   # (step, pinned host copy of the flag, event) not yet known to be complete
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            with torch.no_grad():   # data parallel: every rank starts from rank 0's weights
                for p in model.parameters():
                    dist.broadcast(p.data, src=0)
        self._shard_tokens = None

    def _place_shard(self, n_tokens: int) -> None:
        """Data parallel: rank r holds sequences [r B, (r+1) B) of the global batch, i.e. tokens
        [r n, (r+1) n) -- its Quartet layers use the global token offset, so the
        ranks together reproduce the single-GPU step on the concatenated batch."""
        import torch.distributed as dist

        if self._shard_tokens == n_tokens:
            return
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            set_token_shard(self.model, dist.get_rank() * n_tokens, dist.get_world_size() * n_tokens)
        else:
            set_token_shard(self.model, 0, None)
        self._shard_tokens = n_tokens

    def check_finite(self, wait: bool = False) -> None:
        """Raise ValueError if a finished step quantized a non-finite value.  Without `wait` only the copies
        whose events have completed are read (event.query(), never a stall of the launch queue), so a
        divergence is reported a step or two after it happened; wait=True checks every step so far."""
        while self._pending:
            step, host, ev = self._pending[0]
            if not wait and not ev.query():
                break
            ev.synchronize()
            self._pending.pop(0)
            if int(host.item()) != 0:
                self._flag.zero_()
                self._pending.clear()
                raise ValueError(f"non-finite input to a Quartet layer at or before step {step} (training diverged)")

    def _body(self, tokens, targets):
        logits = self.model(tokens)
        loss = cross_entropy(logits.view(-1, logits.shape[-1]), targets.reshape(-1))
        loss.backward()
        self.bucket.finish()
        torch.nn.utils.clip_grad_norm_(self.bucket.params, self.grad_clip, foreach=True)
        self.opt.step()
        return loss.detach()

    def _graph_step(self, tokens, targets) -> torch.Tensor:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            raise NotImplementedError("graph=True captures a one-GPU step (the bucket all-reduces run eagerly)")
        self.lr_t.fill_(lr_at(self.step_i, self.steps, self.lr))
        if self._cuda_graph is None and self.step_i >= 2:
            self._tok, self._tgt = tokens.clone(), targets.clone()
            self.opt.zero_grad(set_to_none=True)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._loss = self._body(self._tok, self._tgt)
            self._cuda_graph = g
            # the capture only recorded the step: run it (the capture advanced no state on the device)
        if self._cuda_graph is None:   # warm-up steps (optimizer state, kernels' one-time setup) on a side stream
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                self.opt.zero_grad(set_to_none=True)
                loss = self._body(tokens, targets)
            torch.cuda.current_stream().wait_stream(st)
            return loss
        if tokens.data_ptr() != self._tok.data_ptr():
            self._tok.copy_(tokens, non_blocking=True)
            self._tgt.copy_(targets, non_blocking=True)
        self._cuda_graph.replay()
        return self._loss

    def step(self, tokens: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        self.check_finite()
        if self.graph:
            self._place_shard(tokens.numel())
            loss = self._graph_step(tokens, targets)
            self._after_step()
            return loss
        self._place_shard(tokens.numel())
        lr = lr_at(self.step_i, self.steps, self.lr)
        for gr in self.opt.param_groups:
            gr["lr"] = lr
        logits = self.model(tokens)
        loss = cross_entropy(logits.view(-1, logits.shape[-1]), targets.reshape(-1))
        self.opt.zero_grad(set_to_none=True)   # backward assigns each gradient (no fill, no accumulate pass)
        loss.backward()                # bucket all-reduces start inside backward (hooks)
        self.bucket.finish()
        torch.nn.utils.clip_grad_norm_(self.bucket.params, self.grad_clip)
        self.opt.step()
        self._after_step()
        return loss.detach()

    def _after_step(self) -> None:
        if self._flag is not None:
            host = torch.empty(1, dtype=torch.int32, pin_memory=True)
            host.copy_(self._flag, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self._pending.append((self.step_i, host, ev))
        self.step_i += 1


def synthetic_batch(cfg: LlamaConfig, batch: int, seed: int, device) -> tuple[torch.Tensor, torch.Tensor]:
    """Synthetic token stream of the configured shape (no datasets offline): a noisy periodic sequence
    so that the loss has structure to learn."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    base = torch.randint(0, cfg.vocab, (batch, 1), generator=g)
    step = torch.randint(1, 97, (batch, 1), generator=g)
    pos = torch.arange(cfg.seq_len + 1).view(1, -1)
    seq = (base + step * pos) % cfg.vocab
    noise = torch.rand(seq.shape, generator=g) < 0.1
    seq = torch.where(noise, torch.randint(0, cfg.vocab, seq.shape, generator=g), seq)
    seq = seq.to(device)
    return seq[:, :-1].contiguous(), seq[:, 1:].contiguous()
