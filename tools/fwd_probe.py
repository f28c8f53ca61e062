"""Fused forward quantizer variants (development aid; timings only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import quant_fused, quant_rows, sign_bits
L = qt.load()
C = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
x = torch.randn(16384, C, device="cuda").to(torch.bfloat16)
s = sign_bits(3, 16384, "cuda")
H, RT, Q, RTN = _lib.QT_TRANSFORM_HADAMARD, _lib.QT_TRANSFORM_RANDOMIZED, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN
def t(f, n=10):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000 / n
fb = torch.zeros(3, dtype=torch.int32, device="cuda")
f = lambda: quant_fused(x, Q, RTN, transform=H, col_transform=RT, col_signs=s)  # noqa: E731
for mode, name in ((3, "tc full (QuEST+RTN)"), (3 | 4 << 4, "hybrid: exact rows"), (3 | 1 << 4, "tc full, no QuEST"),
                   (3 | 2 << 4, "tc full, no col RTN"), (3 | 3 << 4, "tc full, skeleton"), (0, "production (= tc full)"),
                   (1, "cuda-core fused")):
    L.qt_debug_set_quant(mode, None)
    us = t(f)
    fb.zero_()
    L.qt_debug_set_quant(mode, fb.data_ptr())
    f()
    torch.cuda.synchronize()
    print(f"{name:22s} {us:8.1f} us  fallbacks {fb.tolist()}", flush=True)
L.qt_debug_set_quant(0, None)
print(f"{'rows only (k_quant)':22s} {t(lambda: quant_rows(x, H, Q, want_mask=True)):8.1f} us")
