"""One dual quantizer call at 16384 x 4096 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import quant_dual, sign_bits
qt.load()
x = torch.randn(16384, int(sys.argv[1]) if len(sys.argv) > 1 else 4096, device="cuda").to(torch.bfloat16)
rs, cs = sign_bits(5, x.shape[1], "cuda"), sign_bits(9, x.shape[0], "cuda")
for _ in range(3):
    quant_dual(x, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs, col_signs=cs, prescale=0.75)
torch.cuda.synchronize()
