"""MXF4 / MSK1 wire formats (paper_2505_14669_b200.formats) against the reference's byte layouts
(codec.py:214-244, matio.py:93-115) -- CPU only: operands built from oracle-quantized matrices."""

import struct

import numpy as np
import pytest
import torch


def _operand(oracle, rows=160, cols=96, seed=3):
    from paper_2505_14669_b200.mxfp4 import MXOperand

    x = np.random.default_rng(seed).standard_t(3, size=(rows, cols))
    codes, scales, mask = oracle.quantize_quest(x, 32, 1 / 16)
    op = MXOperand.empty(rows, cols, "cpu", with_mask=True)
    packed = (codes[:, 0::2] | (codes[:, 1::2] << 4)).astype(np.uint8)
    op.codes.copy_(torch.from_numpy(packed))
    op.sf.zero_()
    from paper_2505_14669_b200.formats import _sf_index

    op.sf[_sf_index(rows, cols, op.katoms, "cpu")] = torch.from_numpy(scales)
    bits = np.packbits(mask.astype(bool), axis=1, bitorder="little")
    op.mask.copy_(torch.from_numpy(bits.view("<u4").astype(np.int64).astype(np.uint32).view(np.int32)))
    return op, packed, scales, mask


def test_mxf4_bytes_match_reference_layout(oracle):
    from paper_2505_14669_b200.formats import from_mxf4, to_mxf4

    op, packed, scales, _ = _operand(oracle)
    data = to_mxf4(op)
    ref = struct.pack("<4sHIIHH", b"MXF4", 1, op.rows, op.cols, 32, 0) + packed.tobytes() + scales.tobytes()
    assert data == ref
    back = from_mxf4(data, device="cpu")
    assert torch.equal(back.codes, op.codes) and torch.equal(back.sf, op.sf)
    assert to_mxf4(back) == data


def test_msk1_bytes_match_reference_layout(oracle):
    from paper_2505_14669_b200.formats import from_msk1, to_msk1

    op, _, _, mask = _operand(oracle)
    data = to_msk1(op)
    ref = struct.pack("<4sII", b"MSK1", op.rows, op.cols) + np.packbits(mask.astype(bool), axis=1,
                                                                         bitorder="little").tobytes()
    assert data == ref
    assert torch.equal(from_msk1(data, device="cpu"), op.mask)
    assert np.array_equal(op.mask_bool().numpy(), mask.astype(bool))


@pytest.mark.parametrize("mutate, msg", [
    (lambda d: d[:10], "truncated"),
    (lambda d: b"MXF5" + d[4:], "magic"),
    (lambda d: d[:4] + struct.pack("<H", 2) + d[6:], "version"),
    (lambda d: d + b"\x00", "payload"),
    (lambda d: d[:-1] + b"\xff", "255"),
])
def test_mxf4_rejects_malformed(oracle, mutate, msg):
    from paper_2505_14669_b200.formats import FormatError, from_mxf4, to_mxf4

    op, *_ = _operand(oracle, rows=32, cols=64)
    with pytest.raises(FormatError, match=msg):
        from_mxf4(mutate(to_mxf4(op)), device="cpu")
