"""GEMM mainloop experiments (timing only; results are wrong for dbg != 0)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200 import _lib  # noqa: E402

L = qt.load()
L.qt_debug_set_gemm.argtypes = [ctypes.c_int]
dev = "cuda"
for (M, N, K) in [(16384, 4096, 4096), (16384, 4096, 16384)]:
    x = torch.randn(M, K, device=dev).to(torch.bfloat16)
    w = torch.randn(N, K, device=dev).to(torch.bfloat16)
    A = qt.quant_rows(x, 0, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(w, 0, _lib.QT_ROUND_RTN)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    # knobs 1/2/4/8 (scale copies, B loads, MMA count) exist in the 1-CTA kernel only: run them with 0x40000
    C1 = 0x40000
    for dbg, name in [(0, "baseline (2-CTA pairs)"), (0x80000, "pairs in clusters of 8, multicast"),
                      (0x100, "no epilogue math/stores"), (0x4000, "grouped-2 walk"), (0x1000, "grouped-4 walk"),
                      (0x2000, "grouped-16 walk"), (C1, "1-CTA 128x256 tiles"),
                      (C1 | 1, "1-CTA, no SF tcgen05.cp after k0"), (C1 | 3, "1-CTA, no SF loads+cp after k0"),
                      (C1 | 4, "1-CTA, 1 MMA per k-tile (1/4 math)"), (C1 | 8, "1-CTA, no B TMA after k0"),
                      (C1 | 12, "1-CTA, no B + 1 MMA"), (C1 | 11, "1-CTA, no B, no SF")]:
        L.qt_debug_set_gemm(dbg)
        for _ in range(3):
            qt.gemm(A, B, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            qt.gemm(A, B, out=out)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 100
        print(f"M{M} N{N} K{K} {name:32s} {us:8.1f} us  {2 * M * N * K / us / 1e6:7.1f} TF")
    L.qt_debug_set_gemm(0)
    out32 = torch.empty(M, N, device=dev, dtype=torch.float32)
    for _ in range(3):
        qt.gemm(A, B, out=out32)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        qt.gemm(A, B, out=out32)
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 100
    print(f"M{M} N{N} K{K} {'fp32 output':32s} {us:8.1f} us  {2 * M * N * K / us / 1e6:7.1f} TF")
    del out32
    # dx-like epilogue (trust mask, FWHT-32, 16/9) at the same shape
    mask = torch.randint(0, 2**31 - 1, (M, N // 32), device=dev, dtype=torch.int32)
    for dbg, name in [(0, "dx epilogue (mask, FWHT, 16/9)"), (0x100, "dx, no epilogue math/stores")]:
        L.qt_debug_set_gemm(dbg)
        for _ in range(3):
            qt.gemm(A, B, mask=mask, hadamard=True, scale=16 / 9, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            qt.gemm(A, B, mask=mask, hadamard=True, scale=16 / 9, out=out)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) * 100
        print(f"M{M} N{N} K{K} {name:32s} {us:8.1f} us  {2 * M * N * K / us / 1e6:7.1f} TF")
    L.qt_debug_set_gemm(0)
