"""One tensor-core forward quantizer launch (qt_debug_set_quant mode 3) for ncu (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import quant_fused, sign_bits
L = qt.load()
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 3
x = torch.randn(16384, 4096, device="cuda").to(torch.bfloat16)
s = sign_bits(3, 16384, "cuda")
L.qt_debug_set_quant(mode, None)
for _ in range(3):
    quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_HADAMARD,
                col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=s)
torch.cuda.synchronize()
