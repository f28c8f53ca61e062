"""GPU quantizer diagnostics: the reference's Table-2 quality metrics
(mx4train/diagnostics.py:65-186, Table 2) estimated at scale with the B200 quantizers.

* gaussian_mse(kind)   mean per-element squared reconstruction error of N(0, I) vectors
                       (diagnostics.py:65-89); QuEST in the Hadamard domain like the reference
* misalignment(kind)   1 - E[1/S], S = <x, x> / <H(x . s), q(H(x . s))> (diagnostics.py:92-186)

Differences from the CPU reference, by design: samples are fp32 (the B200 quantizers are bit-exact on
fp32 inputs; the reference draws f64 Gaussians), drawn with torch's device generator, and one
randomized-Hadamard sign vector serves a batch of samples instead of one per sample -- each sample's
(x, s) pair is still independent of its quantization noise, so the expectations are unchanged.  Values
agree with the reference's own reproduction within Monte-Carlo error (tests/test_gpu_diagnostics.py).
The quantize / dequantize round trip uses the production kernels; only the reduction is torch.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from .mxfp4 import derive_seed, quant_rows, sign_bits

KINDS = {"rtn": _lib.QT_ROUND_RTN, "sr": _lib.QT_ROUND_SR, "quest": _lib.QT_ROUND_QUEST}


@dataclass
class Estimate:
    value: float
    stderr: float
    samples: int


def _roundtrip(x: torch.Tensor, kind: str, transform: int, signs, seed: int) -> torch.Tensor:
    op = quant_rows(x, transform, KINDS[kind], signs=signs, sr_seed=seed)
    return op.dequantize(torch.float64)


def _estimate(per_sample: torch.Tensor) -> Estimate:
    n = per_sample.numel()
    return Estimate(float(per_sample.mean()), float(per_sample.std() / n ** 0.5) if n > 1 else 0.0, n)


def gaussian_mse(kind: str, dim: int = 4096, samples: int = 16384, seed: int = 0, batch: int = 4096,
                 device="cuda") -> Estimate:
    """diagnostics.gaussian_mse on the GPU (QuEST measured in the Hadamard domain, diagnostics.py:65-89)."""
    g = torch.Generator(device=device).manual_seed(seed)
    out = []
    for start in range(0, samples, batch):
        b = min(batch, samples - start)
        x = torch.randn(b, dim, device=device, generator=g)
        if kind == "quest":
            from .mxfp4 import fwht32

            x = fwht32(x, _lib.QT_TRANSFORM_HADAMARD)
        d = _roundtrip(x, kind, _lib.QT_TRANSFORM_NONE, None, derive_seed(seed, 0x51, start))
        out.append(((x.double() - d) ** 2).mean(dim=1))
    return _estimate(torch.cat(out))


def misalignment(kind: str, dim: int = 2048, samples: int = 65536, seed: int = 0, batch: int = 4096,
                 device="cuda") -> Estimate:
    """1 - E[1/S] (diagnostics.py:92-186): y = H32(x . s), S^-1 = <y, q(y)> / <x, x>."""
    from .mxfp4 import fwht32

    g = torch.Generator(device=device).manual_seed(seed)
    inv = []
    for start in range(0, samples, batch):
        b = min(batch, samples - start)
        x = torch.randn(b, dim, device=device, generator=g)
        s = sign_bits(derive_seed(seed, 0x5849, start), dim, device)
        y = fwht32(x, _lib.QT_TRANSFORM_RANDOMIZED, s)
        qy = _roundtrip(y, kind, _lib.QT_TRANSFORM_NONE, None, derive_seed(seed, 0x51, start))
        inv.append((y.double() * qy).sum(dim=1) / (x.double() ** 2).sum(dim=1))
    est = _estimate(torch.cat(inv))
    return Estimate(1.0 - est.value, est.stderr, est.samples)
