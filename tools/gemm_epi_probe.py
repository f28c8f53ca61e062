"""2-CTA GEMM epilogue experiments (timing only): cost of the output stores and of the epilogue math.

profiles/r02_gemm_epilogue_probe.txt also holds a "direct st.global" arm (a dbg knob, since removed, that
stored the accumulator rows from registers with epi_store instead of the staged TMA stores): 4-35 % slower
than the staged stores at every shape, so the staged path stays."""
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


def t(f):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    best = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            f()
        e.record()
        torch.cuda.synchronize()
        best.append(s.elapsed_time(e) * 100)
    return sorted(best)[1]


for (M, N, K) in [(16384, 4096, 4096), (16384, 11008, 4096), (16384, 4096, 11008), (4096, 4096, 16384)]:
    x = torch.randn(M, K, device=dev).to(torch.bfloat16)
    w = torch.randn(N, K, device=dev).to(torch.bfloat16)
    A = qt.quant_rows(x, 0, _lib.QT_ROUND_RTN)
    B = qt.quant_rows(w, 0, _lib.QT_ROUND_RTN)
    mask = torch.randint(0, 2**31 - 1, (M, N // 32), device=dev, dtype=torch.int32)
    for odt in (torch.bfloat16, torch.float32):
        out = torch.empty(M, N, device=dev, dtype=odt)
        for epi in ("store", "maskH"):
            kw = dict(mask=mask, hadamard=True, scale=16 / 9) if epi == "maskH" else {}
            ref = None
            for dbg, name in [(0, "staged TMA"), (0x200, "no TMA stores"),
                              (0x400, "no math"), (0x100, "no epilogue")]:
                L.qt_debug_set_gemm(dbg)
                us = t(lambda: qt.gemm(A, B, out=out, **kw))
                if dbg == 0:
                    o = out.clone()
                    if ref is None:
                        ref = o
                    same = bool(torch.equal(ref, o))
                else:
                    same = ""
                print(f"M{M} N{N} K{K} {str(odt)[6:]:8s} {epi:5s} {name:18s} {us:8.1f} us "
                      f"{2 * M * N * K / us / 1e6:7.1f} TF {same}", flush=True)
            L.qt_debug_set_gemm(0)
        del out
