"""Fused forward quantizer (X -> X_q + M_x + X_t) at the Llama widths, 32768 rows: tensor-core kernel (production)
vs the CUDA-core kernel (qt_debug_set_quant mode 1), alternating order, best of 3.  Timing only."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import quant_fused, sign_bits
L = qt.load()
H, RT, Q, RTN = _lib.QT_TRANSFORM_HADAMARD, _lib.QT_TRANSFORM_RANDOMIZED, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN
def t(f, n=20):
    for _ in range(5): f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000 / n
for C in (640, 1280, 1792, 3584):
    x = torch.randn(32768, C, device="cuda").to(torch.bfloat16)
    s = sign_bits(3, 32768, "cuda")
    f = lambda: quant_fused(x, Q, RTN, transform=H, col_transform=RT, col_signs=s)
    res = {0: [], 1: []}
    for rep in range(3):
        for mode in ((0, 1) if rep % 2 == 0 else (1, 0)):
            L.qt_debug_set_quant(mode, None); res[mode].append(t(f))
    L.qt_debug_set_quant(0, None)
    print(f"C={C} rows=32768: tensor-core {min(res[0]):7.1f} us | cuda-core {min(res[1]):7.1f} us", flush=True)
