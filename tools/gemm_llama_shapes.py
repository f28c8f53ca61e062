"""GEMM throughput at the Llama-200M training shapes (64 x 512 tokens, d = 1280, ffn 3584, vocab 32000):
2-CTA pair kernel (default) vs the 1-CTA kernel (0x40000).  Timing only."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200 import _lib  # noqa: E402

L = qt.load()
L.qt_debug_set_gemm.argtypes = [ctypes.c_int]


def operand(r, c):
    return qt.quant_rows(torch.randn(r, c, device="cuda").to(torch.bfloat16), 0, _lib.QT_ROUND_RTN)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


T = 32768
for (M, N, K) in [(T, 1280, 1280), (T, 3584, 1280), (T, 1280, 3584), (1280, 1280, T), (3584, 1280, T),
                  (T, 32000, 1280), (T, 4096, 4096)]:
    A, B = operand(M, K), operand(N, K)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    line = []
    for dbg, name in [(0, "2-CTA"), (0x40000, "1-CTA"), (0x100, "2-CTA no epi")]:
        L.qt_debug_set_gemm(dbg)
        us = timed(lambda: qt.gemm(A, B, out=out))
        line.append(f"{name} {us:7.1f} us {2 * M * N * K / us / 1e6:6.0f} TF")
    L.qt_debug_set_gemm(0)
    print(f"M{M} N{N} K{K}: " + " | ".join(line), flush=True)
