"""Short-K, wide-output GEMMs of the Llama loops (LM head forward, K = d_model): where the time goes (timing
only).  dbg 0x200: no TMA stores; 0x100: no epilogue; 0x4: one of the four MMAs per K tile."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200 import _lib  # noqa: E402

L = qt.load()
L.qt_debug_set_gemm.argtypes = [ctypes.c_int]


def t(f):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 100


for (M, N, K) in [(32768, 32000, 640), (32768, 32000, 1280), (32768, 1280, 1280), (32768, 3584, 1280),
                  (16384, 4096, 4096)]:
    A = qt.quant_rows(torch.randn(M, K, device="cuda").to(torch.bfloat16), 0, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(torch.randn(N, K, device="cuda").to(torch.bfloat16), 0, _lib.QT_ROUND_RTN)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    row = []
    for dbg, name in [(0, "full"), (0x200, "no stores"), (0x100, "no epi"), (0x4, "1/4 MMA"), (0x104, "1/4MMA no epi")]:
        L.qt_debug_set_gemm(dbg)
        row.append(f"{name} {t(lambda: qt.gemm(A, B, out=out)):7.1f}")
    L.qt_debug_set_gemm(0)
    print(f"M{M} N{N} K{K} bf16 out {M * N * 2 / 1e6:.0f} MB: " + " | ".join(row), flush=True)
