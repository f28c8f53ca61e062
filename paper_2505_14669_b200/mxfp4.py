"""Device-resident MXFP4 operands and the thin torch wrappers around the C ABI.

An ``MXOperand`` is the B200 form of the reference's ``QuantizedTensor`` (codec.py:39-72): the
same packed code bytes (element 2k in the low nibble), the same E8M0 exponent values, but the
scales live in tcgen05 scale-factor atoms (see include/quartet_b200.h) so the GEMM can stage them
straight into tensor memory.  ``scales_rowmajor()`` recovers the reference's [rows, cols/32]
``scales`` matrix for parity checks.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check

GROUP = 32


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the Quartet B200 path has no CPU fallback)")


@dataclass
class MXOperand:
    codes: torch.Tensor          # uint8 [rows, cols/2]
    sf: torch.Tensor             # uint8 scale atoms, qt_sf_bytes(rows, cols)
    rows: int
    cols: int
    mask: torch.Tensor | None = None   # int32 [rows, cols/32] bitmap (QuEST trust mask)

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def katoms(self) -> int:
        return 2 * ((self.cols + 255) // 256)

    @staticmethod
    def empty(rows: int, cols: int, device, with_mask: bool = False) -> "MXOperand":
        L = _lib.load()
        if cols % GROUP:
            raise ValueError(f"axis length {cols} not divisible by block size {GROUP}")
        codes = torch.empty((rows, cols // 2), dtype=torch.uint8, device=device)
        # scale atoms: padding (rows to 256, groups to 8) must hold a finite exponent; without padding the
        # quantizer writes every byte, so no fill kernel is needed
        alloc = torch.empty if rows % 256 == 0 and cols % 256 == 0 else torch.zeros
        sf = alloc(int(L.qt_sf_bytes(rows, cols)), dtype=torch.uint8, device=device)
        mask = torch.empty((rows, cols // GROUP), dtype=torch.int32, device=device) if with_mask else None
        return MXOperand(codes, sf, rows, cols, mask)

    def pad_rows(self, rows: int) -> "MXOperand":
        """This operand with zero rows appended up to `rows` (codes 0, E8M0 byte 0, mask 0): the operand of
        the zero-padded matrix.  Used where the reference quantizes a ragged trailing group along this
        operand's rows (qlinear.backward with hadamard=False)."""
        if rows < self.rows:
            raise ValueError(f"pad_rows: {rows} < {self.rows}")
        if rows == self.rows:
            return self
        dev = self.codes.device
        codes = torch.zeros((rows, self.cols // 2), dtype=torch.uint8, device=dev)
        codes[:self.rows] = self.codes
        sf = torch.zeros(int(_lib.load().qt_sf_bytes(rows, self.cols)), dtype=torch.uint8, device=dev)
        off = self._sf_offsets()
        sf[off] = self.sf[off]
        mask = None
        if self.mask is not None:
            mask = torch.zeros((rows, self.cols // GROUP), dtype=torch.int32, device=dev)
            mask[:self.rows] = self.mask
        return MXOperand(codes, sf, rows, self.cols, mask)

    # ---------------------------------------------------------------- parity helpers
    def _sf_offsets(self) -> torch.Tensor:
        """[rows, cols/32] byte offsets of the E8M0 scales in the scale-atom buffer."""
        r = torch.arange(self.rows, device=self.sf.device).view(-1, 1)
        g = torch.arange(self.cols // GROUP, device=self.sf.device).view(1, -1)
        return ((r >> 7) * self.katoms + (g >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (g & 3)

    def scales_rowmajor(self) -> torch.Tensor:
        """uint8 [rows, cols/32] in the reference layout (QuantizedTensor.scales)."""
        return self.sf[self._sf_offsets()]

    def mask_bool(self) -> torch.Tensor:
        """bool [rows, cols]: the reference's m_x / m_w."""
        bits = torch.arange(32, device=self.codes.device, dtype=torch.int64)
        m = (self.mask.to(torch.int64).unsqueeze(-1) >> bits) & 1
        return m.reshape(self.rows, self.cols).bool()

    def unpacked_codes(self) -> torch.Tensor:
        c = self.codes
        return torch.stack([c & 0x0F, c >> 4], dim=-1).reshape(self.rows, self.cols)

    def dequantize(self, dtype=torch.float32) -> torch.Tensor:
        """Exact code * 2^(e-127) (codec.py:204-211); parity/debug helper, not on the hot path."""
        grid = torch.tensor([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0], dtype=torch.float64, device=self.codes.device)
        dec = torch.cat([grid, -grid])
        vals = dec[self.unpacked_codes().long()]
        s = torch.exp2(self.scales_rowmajor().to(torch.float64) - 127.0)
        return (vals * s.repeat_interleave(GROUP, dim=1)).to(dtype)


# ------------------------------------------------------------------------ C-ABI calls

def _in_dtype(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.QT_IN_BF16
    if t.dtype == torch.float32:
        return _lib.QT_IN_F32
    raise ValueError(f"unsupported input dtype {t.dtype} (bf16 or fp32)")


def derive_seed(*parts: int) -> int:
    """rng.derive_seed (rng.py:72-78), computed by the library."""
    import ctypes

    arr = (ctypes.c_uint64 * len(parts))(*[int(p) & 0xFFFFFFFFFFFFFFFF for p in parts])
    return int(_lib.load().qt_derive_seed(ctypes.cast(arr, ctypes.c_void_p), len(parts)))


def sign_bits(xi: int, n: int, device, start: int = 0) -> torch.Tensor:
    """Device bitmap of rng.signs(xi, start, n) (rng.py:57-62): int32 [ceil(n/32)]."""
    out = torch.empty(((n + 31) // 32,), dtype=torch.int32, device=device)
    check(_lib.load().qt_sign_bits_at(out.data_ptr(), int(start), n, int(xi) & 0xFFFFFFFFFFFFFFFF,
                                      _stream(out.device)), "qt_sign_bits_at")
    return out


def sign_bits_pair(xi: int, n_a: int, n_b: int, device, start_a: int = 0, start_b: int = 0):
    """sign_bits(xi, n_a, start=start_a), sign_bits(xi, n_b, start=start_b) in one launch."""
    a = torch.empty(((n_a + 31) // 32,), dtype=torch.int32, device=device)
    b = torch.empty(((n_b + 31) // 32,), dtype=torch.int32, device=device)
    check(_lib.load().qt_sign_bits_pair(a.data_ptr(), int(start_a), n_a, b.data_ptr(), int(start_b), n_b,
                                        int(xi) & 0xFFFFFFFFFFFFFFFF, _stream(a.device)), "qt_sign_bits_pair")
    return a, b


def sign_bits_pair_dev(xi_slot, n_a: int, n_b: int, device, start_a: int = 0, start_b: int = 0):
    """sign_bits_pair with xi read on the device: xi_slot = (uint64 tensor, index) -- the seed of the current
    training step inside a captured CUDA graph (qt_sign_bits_pair_dev)."""
    buf, idx = xi_slot
    a = torch.empty(((n_a + 31) // 32,), dtype=torch.int32, device=device)
    b = torch.empty(((n_b + 31) // 32,), dtype=torch.int32, device=device)
    check(_lib.load().qt_sign_bits_pair_dev(a.data_ptr(), int(start_a), n_a, b.data_ptr(), int(start_b), n_b,
                                            buf.data_ptr() + 8 * int(idx), _stream(a.device)), "qt_sign_bits_pair_dev")
    return a, b


def fwht32(x: torch.Tensor, transform: int = 1, signs: torch.Tensor | None = None,
           prescale: float = 1.0) -> torch.Tensor:
    """prescale * FWHT32(x (.) s) along the last axis, fp32 (kernels.fwht, _native.pyx:353-379)."""
    _require_cuda(x, "x")
    x = x.contiguous().float()
    out = torch.empty_like(x)
    check(_lib.load().qt_fwht32(x.data_ptr(), out.data_ptr(), x.shape[0], x.shape[1], transform,
                                signs.data_ptr() if signs is not None else None, float(prescale),
                                _stream(x.device)), "qt_fwht32")
    return out


def quant_rows(x: torch.Tensor, transform: int, rounding: int, *, signs: torch.Tensor | None = None,
               prescale: float = 1.0, sr_seed: int = 0, counter_start: int = 0, counter_ld: int = 0,
               want_mask: bool = False,
               err: torch.Tensor | None = None, fallbacks: torch.Tensor | None = None,
               out: MXOperand | None = None) -> MXOperand:
    _require_cuda(x, "x")
    if x.dim() != 2:
        raise ValueError("expected a 2-D matrix")
    if x.stride(1) != 1:
        x = x.contiguous()
    rows, cols = x.shape
    if cols % GROUP:
        raise ValueError(f"axis length {cols} not divisible by block size {GROUP}")
    op = out if out is not None else MXOperand.empty(rows, cols, x.device, with_mask=want_mask)
    L = _lib.load()
    rc = L.qt_quant_rows(x.data_ptr(), _in_dtype(x), x.stride(0), rows, cols, transform,
                         signs.data_ptr() if signs is not None else None, float(prescale), rounding,
                         int(sr_seed) & 0xFFFFFFFFFFFFFFFF, int(counter_start), int(counter_ld),
                         op.codes.data_ptr(), op.codes.stride(0), op.sf.data_ptr(), op.katoms,
                         op.mask.data_ptr() if op.mask is not None else None,
                         err.data_ptr() if err is not None else None,
                         fallbacks.data_ptr() if fallbacks is not None else None, _stream(x.device))
    check(rc, "qt_quant_rows")
    return op


def quant_cols(x, rounding: int, *, transform: int, signs: torch.Tensor | None = None, prescale: float = 1.0,
               sr_seed: int = 0, counter_start: int = 0, counter_ld: int = 0, err: torch.Tensor | None = None,
               out: MXOperand | None = None) -> MXOperand:
    """Quantize the transpose of x ([rows, cols] dense tensor or MXOperand) along `rows`."""
    L = _lib.load()
    if isinstance(x, MXOperand):
        rows, cols, dev = x.rows, x.cols, x.codes.device
        args = (None, _lib.QT_IN_MXFP4, 0, x.codes.data_ptr(), x.codes.stride(0), x.sf.data_ptr(), x.katoms)
    else:
        _require_cuda(x, "x")
        if x.stride(1) != 1:
            x = x.contiguous()
        rows, cols = x.shape
        dev = x.device
        args = (x.data_ptr(), _in_dtype(x), x.stride(0), None, 0, None, 0)
    if rows % GROUP or cols % GROUP:
        raise ValueError(f"transposed quantization needs both axes divisible by {GROUP}: {rows}x{cols}")
    op = out if out is not None else MXOperand.empty(cols, rows, dev)
    rc = L.qt_quant_cols(*args, rows, cols, transform, signs.data_ptr() if signs is not None else None,
                         float(prescale), rounding, int(sr_seed) & 0xFFFFFFFFFFFFFFFF, int(counter_start),
                         int(counter_ld), op.codes.data_ptr(), op.codes.stride(0), op.sf.data_ptr(), op.katoms,
                         err.data_ptr() if err is not None else None, _stream(dev))
    check(rc, "qt_quant_cols")
    return op


def quant_fused(x: torch.Tensor, rounding: int, col_rounding: int, *, transform: int, col_transform: int,
                col_signs: torch.Tensor | None = None, prescale: float = 1.0, col_prescale: float = 0.75,
                sr_seed: int = 0, counter_start: int = 0, col_seed: int = 0, col_counter_start: int = 0,
                col_counter_ld: int = 0, want_mask: bool = True, err: torch.Tensor | None = None, fallbacks: torch.Tensor | None = None):
    """A forward operand and its transposed backward requantization from ONE read of x[rows, cols]
    (qt_quant_fused): returns (row operand [rows, cols] = Q(T(x)), col operand [cols, rows] =
    Q_col(T_col(deq(row operand)^T) * col_prescale)), i.e. (X_q, X_t) or (W_q, W_t) of qlinear.py:139-157
    and 206-207 / 215 / 235.  `col_signs` flips the row axis (the backward contraction axis).  counter_start:
    SR stream position of the row operand's element (0, 0) (row shard r0 of a [R, cols] matrix: r0 * cols)."""
    _require_cuda(x, "x")
    if x.stride(1) != 1:
        x = x.contiguous()
    rows, cols = x.shape
    if rows % GROUP or cols % GROUP:
        raise ValueError(f"fused quantization needs both axes divisible by {GROUP}: {rows}x{cols}")
    r_op = MXOperand.empty(rows, cols, x.device, with_mask=want_mask)
    c_op = MXOperand.empty(cols, rows, x.device)
    rc = _lib.load().qt_quant_fused(x.data_ptr(), _in_dtype(x), x.stride(0), rows, cols, transform, None,
                                    float(prescale), rounding, int(sr_seed) & 0xFFFFFFFFFFFFFFFF, int(counter_start), 0,
                                    r_op.codes.data_ptr(), r_op.codes.stride(0), r_op.sf.data_ptr(), r_op.katoms,
                                    r_op.mask.data_ptr() if r_op.mask is not None else None, col_transform,
                                    col_signs.data_ptr() if col_signs is not None else None, float(col_prescale),
                                    col_rounding, int(col_seed) & 0xFFFFFFFFFFFFFFFF, int(col_counter_start),
                                    int(col_counter_ld), c_op.codes.data_ptr(), c_op.codes.stride(0), c_op.sf.data_ptr(),
                                    c_op.katoms, err.data_ptr() if err is not None else None,
                                    fallbacks.data_ptr() if fallbacks is not None else None, _stream(x.device))
    check(rc, "qt_quant_fused")
    return r_op, c_op


def quant_dual(x: torch.Tensor, rounding: int, *, transform: int, signs: torch.Tensor | None = None,
               col_signs: torch.Tensor | None = None, prescale: float = 1.0, seed_rows: int = 0, seed_cols: int = 0,
               row_counter_start: int = 0, col_counter_start: int = 0, col_counter_ld: int = 0,
               err: torch.Tensor | None = None):
    """Both backward dy operands from ONE read of x[rows, cols]: (rows-operand [rows, cols] grouped along
    cols, cols-operand [cols, rows] grouped along rows) -- qlinear.py:214-245.  `signs` flips the column
    axis of the rows-operand, `col_signs` (default: `signs`) the row axis of the cols-operand."""
    col_signs = signs if col_signs is None else col_signs
    _require_cuda(x, "x")
    if x.stride(1) != 1:
        x = x.contiguous()
    rows, cols = x.shape
    if rows % GROUP or cols % GROUP:
        raise ValueError(f"dual quantization needs both axes divisible by {GROUP}: {rows}x{cols}")
    r_op = MXOperand.empty(rows, cols, x.device)
    c_op = MXOperand.empty(cols, rows, x.device)
    rc = _lib.load().qt_quant_dual(x.data_ptr(), _in_dtype(x), x.stride(0), rows, cols, transform,
                                   signs.data_ptr() if signs is not None else None,
                                   col_signs.data_ptr() if col_signs is not None else None, float(prescale), rounding,
                                   int(seed_rows) & 0xFFFFFFFFFFFFFFFF, int(row_counter_start),
                                   int(seed_cols) & 0xFFFFFFFFFFFFFFFF, int(col_counter_start), int(col_counter_ld),
                                   r_op.codes.data_ptr(), r_op.codes.stride(0), r_op.sf.data_ptr(), r_op.katoms, None,
                                   c_op.codes.data_ptr(), c_op.codes.stride(0), c_op.sf.data_ptr(), c_op.katoms,
                                   err.data_ptr() if err is not None else None, _stream(x.device))
    check(rc, "qt_quant_dual")
    return r_op, c_op


def gemm(a: MXOperand, b: MXOperand, *, out_dtype=torch.float32, mask: torch.Tensor | None = None,
         hadamard: bool = True, scale: float = 1.0, out: torch.Tensor | None = None,
         accumulate: bool = False) -> torch.Tensor:
    """deq(a) @ deq(b).T on tcgen05 (gemm_lp, qlinear.py:96-111); with `mask`, the fused
    H32(D * mask) * scale epilogue (qlinear.py:229-230).  accumulate=True adds the result (rounded to
    out's dtype) into `out` instead of overwriting it, bit-identical to out.add_(gemm(...))."""
    if a.cols != b.cols:
        raise ValueError(f"contraction mismatch: {a.cols} vs {b.cols}")
    M, N, K = a.rows, b.rows, a.cols
    if accumulate and (out is None or tuple(out.shape) != (M, N)):
        raise ValueError("accumulate=True needs an [M, N] out tensor")
    if out is None:
        if out_dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"gemm output dtype must be bfloat16 or float32, got {out_dtype}")
        out = torch.empty((M, N), dtype=out_dtype, device=a.codes.device)
    else:
        if out.dtype not in (torch.bfloat16, torch.float32):
            raise ValueError(f"gemm output dtype must be bfloat16 or float32, got {out.dtype}")
        if out.dim() != 2 or tuple(out.shape) != (M, N) or out.stride(1) != 1 or out.stride(0) < N:
            raise ValueError(f"gemm out must be a row-major [{M}, {N}] view with unit column stride, got "
                             f"shape {tuple(out.shape)} strides {tuple(out.stride())}")
        if out.device != a.codes.device:
            raise ValueError(f"gemm out is on {out.device}, operands on {a.codes.device}")
    odt = _lib.QT_OUT_BF16 if out.dtype == torch.bfloat16 else _lib.QT_OUT_F32
    epi = _lib.QT_EPI_STORE if mask is None else (_lib.QT_EPI_MASK_H if hadamard else _lib.QT_EPI_MASK)
    if accumulate:
        epi |= _lib.QT_EPI_ACCUMULATE
    rc = _lib.load().qt_gemm_mxf4(a.codes.data_ptr(), a.sf.data_ptr(), b.codes.data_ptr(), b.sf.data_ptr(),
                                  M, N, K, out.data_ptr(), odt, out.stride(0), epi,
                                  mask.data_ptr() if mask is not None else None, float(scale),
                                  _stream(out.device))
    check(rc, "qt_gemm_mxf4")
    return out


# ---- exact plugin seam (qt_seam_*, seam.cu): f64 / any-group replays of _native.pyx:104-396 -------------
def seam_quantize(x: torch.Tensor, group: int, rounding: int, *, seed: int = 0, counter_start: int = 0,
                  ratio_lo: float = 1.0 / 16.0, values: bool = False):
    """quantize_{rtn,sr,quest} (values=False: unpacked codes u8 [R, C], scales u8 [R, ceil(C/g)], QuEST mask)
    or *_values (values=True: f64 values [R, C], QuEST mask) of a f64 device matrix, bit-identical to the
    reference's kernels for every input (_native.pyx:104-350)."""
    _require_cuda(x, "x")
    if x.dtype != torch.float64 or x.dim() != 2:
        raise ValueError("seam quantizers take a 2-D float64 matrix")
    x = x.contiguous()
    rows, cols = x.shape
    ng = -(-cols // group) if group > 0 else 0
    dev = x.device
    quest = rounding == _lib.QT_ROUND_QUEST
    mask = torch.empty((rows, cols), dtype=torch.uint8, device=dev) if quest else None
    if values:
        out = torch.empty((rows, cols), dtype=torch.float64, device=dev)
        codes = scales = None
    else:
        out = None
        codes = torch.empty((rows, cols), dtype=torch.uint8, device=dev)
        scales = torch.empty((rows, ng), dtype=torch.uint8, device=dev)
    ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
    rc = _lib.load().qt_seam_quantize(x.data_ptr(), rows, cols, int(group), int(rounding), int(values),
                                      int(seed) & 0xFFFFFFFFFFFFFFFF, int(counter_start) & 0xFFFFFFFFFFFFFFFF,
                                      float(ratio_lo), ptr(codes), ptr(scales), ptr(mask), ptr(out), _stream(dev))
    check(rc, "qt_seam_quantize")
    if values:
        return (out, mask) if quest else out
    return (codes, scales, mask) if quest else (codes, scales)


def seam_fwht(x: torch.Tensor, g: int) -> torch.Tensor:
    """Blockwise FWHT of a f32 / f64 device matrix along its rows, any power-of-two block g
    (_native.pyx:353-379), on a copy."""
    _require_cuda(x, "x")
    if x.dtype not in (torch.float32, torch.float64) or x.dim() != 2:
        raise ValueError("seam fwht takes a 2-D float32 / float64 matrix")
    out = x.contiguous().clone()
    rc = _lib.load().qt_seam_fwht(out.data_ptr(), int(out.dtype == torch.float64), out.shape[0], out.shape[1],
                                  int(g), _stream(out.device))
    check(rc, "qt_seam_fwht")
    return out


def seam_gemm_nt(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """a @ b.T with the reference's fixed ascending-k order per output (_native.pyx:382-396), f32 or f64."""
    _require_cuda(a, "a")
    if a.dtype != b.dtype or a.dtype not in (torch.float32, torch.float64):
        raise ValueError("seam gemm_nt takes two float32 or two float64 matrices")
    a, b = a.contiguous(), b.contiguous()
    m, k = a.shape
    n = b.shape[0]
    c = torch.empty((m, n), dtype=a.dtype, device=a.device)
    rc = _lib.load().qt_seam_gemm_nt(a.data_ptr(), b.data_ptr(), c.data_ptr(), int(a.dtype == torch.float64), m, n,
                                     k, _stream(a.device))
    check(rc, "qt_seam_gemm_nt")
    return c


def seam_row_sums(a: torch.Tensor, b: torch.Tensor | None, op: int) -> torch.Tensor:
    """numpy's add.reduce along rows of (a - b)^2 (op 0) or a * b (op 1; b None = a), pairwise order."""
    _require_cuda(a, "a")
    a = a.contiguous()
    if b is not None:
        b = b.contiguous()
    rows, n = a.shape
    out = torch.empty(rows, dtype=torch.float64, device=a.device)
    rc = _lib.load().qt_seam_row_sums(a.data_ptr(), b.data_ptr() if b is not None else None, int(op), rows, n,
                                      out.data_ptr(), _stream(a.device))
    check(rc, "qt_seam_row_sums")
    return out
