"""Shared helpers for the GPU parity tests (tests only)."""

import numpy as np
import torch


def bf16_values(a: np.ndarray) -> np.ndarray:
    """f32 -> bf16 (RNE) -> f32, as numpy (the values the B200 path consumes)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32)


def to_dev(a: np.ndarray, dtype=torch.float32) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda").to(dtype)


def op_codes(op) -> np.ndarray:
    return op.unpacked_codes().cpu().numpy()


def op_scales(op) -> np.ndarray:
    return op.scales_rowmajor().cpu().numpy()


def assert_operand_equal(op, codes: np.ndarray, scales: np.ndarray, what: str = ""):
    got_c, got_s = op_codes(op), op_scales(op)
    if got_c.shape != codes.shape:   # operand of the zero-padded matrix (the reference's ragged trailing groups)
        R, C = codes.shape
        assert got_c.shape[0] >= R and got_c.shape[1] >= C, f"{what}: shape {got_c.shape} vs {codes.shape}"
        assert not got_c[R:].any() and not got_c[:, C:].any(), f"{what}: padding encodes nonzero codes"
        got_c, got_s = got_c[:R, :C], got_s[:R, :scales.shape[1]]
    bad = np.argwhere(got_s != scales)
    assert bad.size == 0, f"{what}: {len(bad)} scale mismatches, first at {bad[0]}: {got_s[tuple(bad[0])]} vs {scales[tuple(bad[0])]}"
    bad = np.argwhere(got_c != codes)
    assert bad.size == 0, f"{what}: {len(bad)} code mismatches, first at {bad[0]}: {got_c[tuple(bad[0])]} vs {codes[tuple(bad[0])]}"


def rel_err(got: np.ndarray, ref: np.ndarray) -> float:
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(got - ref) / (den if den > 0 else 1.0))
