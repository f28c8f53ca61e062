"""Bottleneck probe of the tensor-core dual quantizer (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import quant_dual, sign_bits
L = qt.load()
x = torch.randn(16384, 4096, device="cuda").to(torch.bfloat16)
rs, cs = sign_bits(5, x.shape[1], "cuda"), sign_bits(9, x.shape[0], "cuda")
f = lambda: quant_dual(x, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs, col_signs=cs, prescale=0.75)
for dbg, name in ((0, "full"), (1, "skip quantize"), (2, "skip B build"), (3, "skip both"), (4, "skip TMEM ld"), (5, "skip ld+quant"), (7, "skip all"), (8, "skip stores")):
    L.qt_debug_set_quant(dbg << 4, None)
    f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): f()
    e.record(); torch.cuda.synchronize()
    print(f"{name:16s} {s.elapsed_time(e) * 100:8.1f} us")
L.qt_debug_set_quant(1, None)
f(); torch.cuda.synchronize()
s.record()
for _ in range(10): f()
e.record(); torch.cuda.synchronize()
print(f"{'cuda-core path':16s} {s.elapsed_time(e) * 100:8.1f} us")
