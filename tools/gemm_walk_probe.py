import sys, os
sys.path.insert(0, "/root/repo")
import ctypes, torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
L = qt.load(); L.qt_debug_set_gemm.argtypes = [ctypes.c_int]
for (M, N, K) in [(16384, 4096, 4096), (16384, 11008, 4096), (16384, 4096, 11008)]:
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16); w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    A = qt.quant_rows(x, 0, _lib.QT_ROUND_RTN); B = qt.quant_rows(w, 0, _lib.QT_ROUND_RTN)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    res = {}
    for rep in range(3):
        for dbg, name in [(0, "row-major/g8"), (0x4000, "g2"), (0x1000, "g4"), (0x2000, "g16")]:
            L.qt_debug_set_gemm(dbg)
            for _ in range(3): qt.gemm(A, B, out=out)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20): qt.gemm(A, B, out=out)
            e.record(); torch.cuda.synchronize()
            res.setdefault(name, []).append(s.elapsed_time(e) * 50)
    L.qt_debug_set_gemm(0)
    print(M, N, K, {k: [round(v, 1) for v in vs] for k, vs in res.items()})
