"""2-CTA vs 1-CTA GEMM timing with mainloop knobs (results wrong for dbg != 0)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
L = qt.load()
for (M, N, K) in [(16384, 4096, 4096), (16384, 4096, 16384)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    A = qt.quant_rows(x, 0, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(w, 0, _lib.QT_ROUND_RTN)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for dbg, name in [(0, "1cta"), (0x20, "1cta SF pre-issue"), (0x1, "1cta no SF cp"), (0x20000, "2sm"),
                      (0x20001, "2sm no SF cp"), (0x20004, "2sm 1 MMA"), (0x20005, "2sm 1 MMA no SF cp")]:
        L.qt_debug_set_gemm(dbg)
        for _ in range(3): qt.gemm(A, B, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10): qt.gemm(A, B, out=out)
        e.record(); torch.cuda.synchronize()
        us = s.elapsed_time(e) * 100
        print(f"M{M} N{N} K{K} {name:22s} {us:8.1f} us  {2 * M * N * K / us / 1e6:7.1f} TF")
    L.qt_debug_set_gemm(0)
