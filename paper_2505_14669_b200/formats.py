"""Wire formats for exporting / checkpointing quantized operands.

* ``MXF4`` container -- the reference's QuantizedTensor serialization (codec.py:214-244): little-endian
  header ``<4sHIIHH`` = (b"MXF4", version 1, rows, cols, group_size, 0), then the packed code bytes
  (rows x ceil(cols/2), element 2k in the low nibble) and the E8M0 scale bytes (rows x ceil(cols/32)).
  An ``MXOperand``'s code bytes ARE those bytes; only the scales move between the reference's row-major
  matrix and the tcgen05 scale-factor atoms.
* ``MSK1`` mask -- the reference's packed-bit trust-mask file (matio.py:93-115): header ``<4sII`` =
  (b"MSK1", rows, cols), then per row ceil(cols/8) bytes, bit order little.  The operand's uint32 mask
  words (bit j of word g = element 32 g + j) laid out little-endian are exactly that payload.

Parsing errors raise ``FormatError`` (a ValueError), like the reference.
"""

from __future__ import annotations

import struct

import torch

from .mxfp4 import GROUP, MXOperand

MXF4_HEADER = struct.Struct("<4sHIIHH")
MXF4_MAGIC, MXF4_VERSION = b"MXF4", 1
MSK1_HEADER = struct.Struct("<4sII")
MSK1_MAGIC = b"MSK1"


class FormatError(ValueError):
    pass


def _sf_index(rows: int, cols: int, katoms: int, device) -> torch.Tensor:
    r = torch.arange(rows, device=device).view(-1, 1)
    g = torch.arange(cols // GROUP, device=device).view(1, -1)
    return ((r >> 7) * katoms + (g >> 2)) * 512 + (r & 31) * 16 + ((r >> 5) & 3) * 4 + (g & 3)


def to_mxf4(op: MXOperand) -> bytes:
    """codec.serialize (codec.py:214-216) of an operand."""
    header = MXF4_HEADER.pack(MXF4_MAGIC, MXF4_VERSION, op.rows, op.cols, GROUP, 0)
    codes = op.codes.contiguous().cpu().numpy().tobytes()
    scales = op.scales_rowmajor().contiguous().cpu().numpy().tobytes()
    return header + codes + scales


def from_mxf4(data: bytes, device="cuda") -> MXOperand:
    """codec.deserialize (codec.py:219-244) into a device operand (scales scattered into the atoms)."""
    if len(data) < MXF4_HEADER.size:
        raise FormatError("truncated header")
    magic, version, rows, cols, group, _ = MXF4_HEADER.unpack_from(data)
    if magic != MXF4_MAGIC:
        raise FormatError(f"bad magic {magic!r}")
    if version != MXF4_VERSION:
        raise FormatError(f"unsupported version {version}")
    if group == 0:
        raise FormatError("zero group size")
    if group != GROUP or cols % GROUP:
        raise FormatError(f"the tcgen05 operand layout needs group 32 and cols % 32 == 0 (got {group}, {cols})")
    ncode, nscale = rows * ((cols + 1) // 2), rows * (-(-cols // group))
    if len(data) != MXF4_HEADER.size + ncode + nscale:
        raise FormatError(f"payload length {len(data)}, expected {MXF4_HEADER.size + ncode + nscale}")
    raw = torch.frombuffer(bytearray(data), dtype=torch.uint8)
    codes = raw[MXF4_HEADER.size:MXF4_HEADER.size + ncode].view(rows, (cols + 1) // 2)
    scales = raw[MXF4_HEADER.size + ncode:].view(rows, cols // group)
    if bool((scales == 255).any()):
        raise FormatError("invalid scale byte 255")
    op = MXOperand.empty(rows, cols, device)
    op.codes.copy_(codes)
    op.sf.zero_()
    op.sf[_sf_index(rows, cols, op.katoms, op.sf.device)] = scales.to(op.sf.device)
    return op


def to_msk1(op: MXOperand) -> bytes:
    """matio.write_mask (matio.py:93-98) of the operand's trust mask."""
    if op.mask is None:
        raise FormatError("operand has no trust mask")
    body = op.mask.contiguous().cpu().numpy().astype("<u4").tobytes()
    return MSK1_HEADER.pack(MSK1_MAGIC, op.rows, op.cols) + body


def from_msk1(data: bytes, device="cuda") -> torch.Tensor:
    """matio.read_mask (matio.py:101-115) -> int32 [rows, cols/32] mask words on `device`."""
    if len(data) < MSK1_HEADER.size:
        raise FormatError("truncated mask header")
    magic, rows, cols = MSK1_HEADER.unpack_from(data)
    if magic != MSK1_MAGIC:
        raise FormatError(f"bad mask magic {magic!r}")
    per_row = (cols + 7) // 8
    if len(data) != MSK1_HEADER.size + rows * per_row:
        raise FormatError(f"mask payload length {len(data)}, expected {MSK1_HEADER.size + rows * per_row}")
    if cols % GROUP:
        raise FormatError("mask width must be a multiple of 32 for the operand layout")
    body = torch.frombuffer(bytearray(data[MSK1_HEADER.size:]), dtype=torch.uint8)
    return body.view(torch.int32).view(rows, cols // GROUP).to(device)
