"""Quantizer diagnostics on the B200: the reference's Table-2 quality metrics,
bit-identical to mx4train.diagnostics (diagnostics.py:65-186).

* gaussian_mse(kind)          mean per-element squared reconstruction error of N(0, I) vectors
                              (diagnostics.py:65-89); QuEST measured in the Hadamard domain
* misalignment_suite(kinds)   1 - E[1/S], S = <x, x> / <H(x . s), q(H(x . s))>, over one shared sample
                              stream (diagnostics.py:121-170); misalignment(kind) for one scheme
* rescale_factor_S(x, xi)     S of one vector (diagnostics.py:92-113)

Same sample streams as the reference: the N(0, I) vectors are rng.gaussians (splitmix64 positions through
the inverse normal CDF, rng.py:65-69) and the misalignment pairs are one Philox stream per sample keyed
by (derive_seed(seed, 0x5849), i) (diagnostics.py:116-134) -- generated on the host with numpy / scipy
exactly as the reference does, since they ARE the definition of the estimate.  Everything after that runs
on the GPU through the exact seam kernels (csrc/seam.cu): the f64 FWHT-32, the f64 quantize-dequantize of
each scheme (rtn_values / sr_values / quest_values, _native.pyx:248-350) and the per-sample reductions in
numpy's pairwise order, so every per-sample value -- and therefore every estimate and its standard error --
equals the reference's bit for bit (tests/test_gpu_diagnostics.py checks against estimates produced by
the reference itself).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .mxfp4 import derive_seed, seam_fwht, seam_quantize, seam_row_sums

SCHEME_IDS = ("exact", "rtn_absmax", "sr_absmax", "quest")   # diagnostics.py:22
GROUP_SIZE = 32
QUEST_RATIO_LO = 1.0 / 16.0                                   # quantizers.py QUEST.clip_range[0]
_DOMAIN_XI = 0x5849                                           # diagnostics.py:24
_DOMAIN_SRQ = 0x5153                                          # diagnostics.py:25
_DOMAIN_GAUSS = 0x4755                                        # rng.py:23
_DOMAIN_SIGNS = 0x5347                                        # rng.py:22
_U64 = np.uint64
_GOLDEN = _U64(0x9E3779B97F4A7C15)


@dataclass(frozen=True)
class MonteCarloEstimate:
    """diagnostics.py:28-34"""
    value: float
    stderr: float
    samples: int
    seed: int
    excluded: int = 0


# ------------------------------------------------------------------ sample streams (host, rng.py)
def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
    return z ^ (z >> _U64(31))


def _raw_at(seed: int, domain: int, start: int, count: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        s = np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=_U64)
        d = np.array([domain & 0xFFFFFFFFFFFFFFFF], dtype=_U64)
        base = _mix64(s ^ _mix64(d))[0]
        idx = np.arange(start, start + count, dtype=_U64)
        return _mix64(base + (idx + _U64(1)) * _GOLDEN)


def gaussians(seed: int, domain: int, start: int, count: int) -> np.ndarray:
    """rng.gaussians (rng.py:65-69): ndtri of open-interval uniforms at stream positions."""
    from scipy.special import ndtri

    h = _raw_at(seed, domain, start, count)
    u = ((h >> _U64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    return ndtri(u)


def _flipped_gaussian_batch(seed: int, start: int, count: int, dim: int) -> np.ndarray:
    """diagnostics.py:116-134: one Philox stream per sample, dim normals then dim flip bits."""
    out = np.empty((count, dim))
    key_hi = derive_seed(seed, _DOMAIN_XI)
    for i in range(count):
        gen = np.random.Generator(np.random.Philox(key=np.array([key_hi, start + i], dtype=np.uint64)))
        x = gen.standard_normal(dim)
        flips = gen.integers(0, 2, size=dim)
        np.multiply(x, 1.0 - 2.0 * flips, out=out[i])
    return out


# ---------------------------------------------------------------------------- GPU pieces
def _quantize_values(y: torch.Tensor, kind: str, seed: int) -> torch.Tensor:
    """diagnostics.py:49-62 on the device (f64 in, f64 values out)."""
    if kind == "exact":
        return y
    if kind == "rtn_absmax":
        return seam_quantize(y, GROUP_SIZE, _lib.QT_ROUND_RTN, values=True)
    if kind == "sr_absmax":
        return seam_quantize(y, GROUP_SIZE, _lib.QT_ROUND_SR, seed=seed & 0xFFFFFFFFFFFFFFFF, counter_start=0,
                             values=True)
    if kind == "quest":
        return seam_quantize(y, GROUP_SIZE, _lib.QT_ROUND_QUEST, ratio_lo=QUEST_RATIO_LO, values=True)[0]
    raise ValueError(f"unknown scheme {kind!r}")


def _check_kind(kind: str) -> None:
    if kind not in SCHEME_IDS:
        raise ValueError(f"unknown scheme {kind!r}")


def gaussian_mse(kind: str, dim: int = 4096, samples: int = 256, seed: int = 0, batch: int = 512,
                 device="cuda") -> MonteCarloEstimate:
    """diagnostics.gaussian_mse (diagnostics.py:65-89), per-vector errors on the GPU."""
    _check_kind(kind)
    if dim % GROUP_SIZE:
        raise ValueError(f"dim must be a multiple of {GROUP_SIZE}")
    per_vector = np.empty(samples)
    done = 0
    while done < samples:
        b = min(batch, samples - done)
        x = torch.from_numpy(gaussians(seed, _DOMAIN_GAUSS, done * dim, b * dim).reshape(b, dim)).to(device)
        if kind == "quest":
            x = seam_fwht(x, GROUP_SIZE)
        d = _quantize_values(x, kind, derive_seed(seed, _DOMAIN_SRQ, done))
        per_vector[done:done + b] = seam_row_sums(x, d, 0).cpu().numpy() / dim
        done += b
    value = float(per_vector.mean())
    stderr = float(per_vector.std(ddof=1) / np.sqrt(samples)) if samples > 1 else 0.0
    return MonteCarloEstimate(value=value, stderr=stderr, samples=samples, seed=seed)


def misalignment_suite(kinds: tuple[str, ...], dim: int = 2048, samples: int = 100_000, seed: int = 0,
                       batch: int = 2048, device="cuda") -> dict[str, MonteCarloEstimate]:
    """diagnostics.misalignment_suite (diagnostics.py:137-178): 1 - E[1/S] for several schemes over one
    shared sample stream; degenerate samples (zero denominator) are excluded and counted."""
    if dim % GROUP_SIZE:
        raise ValueError(f"dim must be a multiple of {GROUP_SIZE}")
    for kind in kinds:
        _check_kind(kind)
    inv_s = {kind: np.empty(samples) for kind in kinds}
    done = 0
    while done < samples:
        b = min(batch, samples - done)
        flipped = torch.from_numpy(_flipped_gaussian_batch(seed, done, b, dim)).to(device)
        y = seam_fwht(flipped, GROUP_SIZE)
        den = seam_row_sums(flipped, None, 1).cpu().numpy()
        bad = den == 0.0
        for kind in kinds:
            qy = _quantize_values(y, kind, derive_seed(seed, _DOMAIN_SRQ, done))
            num = seam_row_sums(y, qy, 1).cpu().numpy()
            inv_s[kind][done:done + b] = np.divide(num, den, out=np.full(b, np.nan), where=~bad)
        done += b
    out = {}
    for kind in kinds:
        good = inv_s[kind][np.isfinite(inv_s[kind])]
        excluded = samples - good.size
        value = float(1.0 - good.mean())
        stderr = float(good.std(ddof=1) / np.sqrt(good.size)) if good.size > 1 else 0.0
        out[kind] = MonteCarloEstimate(value=value, stderr=stderr, samples=samples, seed=seed, excluded=excluded)
    return out


def misalignment(kind: str, dim: int = 2048, samples: int = 100_000, seed: int = 0, batch: int = 2048,
                 device="cuda") -> MonteCarloEstimate:
    """diagnostics.misalignment (diagnostics.py:181-192)."""
    return misalignment_suite((kind,), dim=dim, samples=samples, seed=seed, batch=batch, device=device)[kind]


def rescale_factor_S(x: np.ndarray, xi: int, kind: str = "rtn_absmax", seed: int = 0, device="cuda") -> float:
    """diagnostics.rescale_factor_S (diagnostics.py:92-113) for one vector."""
    v = np.asarray(x, dtype=np.float64).reshape(1, -1)
    n = v.shape[1]
    if n % GROUP_SIZE:
        raise ValueError(f"length must be a multiple of {GROUP_SIZE}")
    if not np.any(v):
        raise ValueError("zero input vector")
    d = np.where((_raw_at(xi, _DOMAIN_SIGNS, 0, n) >> _U64(63)) == _U64(1), -1.0, 1.0)   # rng.signs
    vt = torch.from_numpy(np.ascontiguousarray(v * d)).to(device)
    y = seam_fwht(vt, GROUP_SIZE)
    qy = _quantize_values(y, kind, seed)
    den = float(seam_row_sums(y, qy, 1).cpu().numpy()[0])
    if den == 0.0:
        raise ZeroDivisionError("degenerate quantization: zero denominator")
    vv = torch.from_numpy(np.ascontiguousarray(v)).to(device)
    return float(seam_row_sums(vv, None, 1).cpu().numpy()[0]) / den
