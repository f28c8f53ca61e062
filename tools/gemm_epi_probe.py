"""Epilogue staging variants of the 2-CTA GEMM on the bench's nine GEMMs (16384 tokens, Llama-7B shapes):
time per variant (variants interleaved, 3 rounds, best) and bit-equality with the production path.

    python tools/gemm_epi_probe.py [dbg ...]      (timing knobs: 0x100 no epilogue, 0x200 no TMA stores, 0x400 no mask/FWHT/scale)
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200 import _lib  # noqa: E402

L = qt.load()
L.qt_debug_set_gemm.argtypes = [ctypes.c_int]
T = 16384
VARIANTS = [0] + [int(a, 0) for a in sys.argv[1:]] if len(sys.argv) > 1 else [0, 0x100, 0x200, 0x400]


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


def operand(r, c):
    return qt.quant_rows(torch.randn(r, c, device="cuda").to(torch.bfloat16), 0, _lib.QT_ROUND_RTN)


totals = {v: 0.0 for v in VARIANTS}
for d_in, d_out in [(4096, 4096), (4096, 11008), (11008, 4096)]:
    cases = [("fwd", operand(T, d_in), operand(d_out, d_in), torch.bfloat16, None),
             ("dx", operand(T, d_out), operand(d_in, d_out), torch.bfloat16,
              torch.randint(-2**31, 2**31 - 1, (T, d_in // 32), device="cuda", dtype=torch.int32)),
             ("dw", operand(d_out, T), operand(d_in, T), torch.float32,
              torch.randint(-2**31, 2**31 - 1, (d_out, d_in // 32), device="cuda", dtype=torch.int32))]
    for name, A, B, odt, mask in cases:
        kw = {} if mask is None else {"mask": mask, "hadamard": True, "scale": 16 / 9}
        out = torch.empty(A.rows, B.rows, device="cuda", dtype=odt)
        L.qt_debug_set_gemm(0)
        ref = qt.gemm(A, B, out_dtype=odt, **kw)
        best = {v: 1e30 for v in VARIANTS}
        same = {v: True for v in VARIANTS}
        for _ in range(3):
            for v in VARIANTS:
                L.qt_debug_set_gemm(v)
                best[v] = min(best[v], timed(lambda: qt.gemm(A, B, out=out, **kw)))
                same[v] &= torch.equal(out, ref)
        L.qt_debug_set_gemm(0)
        for v in VARIANTS:
            totals[v] += best[v]
        print(f"{d_in}->{d_out} {name:3s} M{A.rows} N{B.rows} K{A.cols}: " +
              " | ".join(f"{v:#x} {best[v]:7.1f}{'' if same[v] else ' MISMATCH'}" for v in VARIANTS), flush=True)
        del out, ref
print("sum over the 9 GEMMs (us): " + " | ".join(f"{v:#x} {t:.1f}" for v, t in totals.items()))
