"""One fused forward quantizer call (X -> X_q + M_x + X_t) at 16384 x d (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import quant_fused, sign_bits
L = qt.load()
if os.environ.get("QT_PROF_QMODE"):  # e.g. 51 = tensor-core path, skeleton only (tools/fwd_probe.py)
    L.qt_debug_set_quant(int(os.environ["QT_PROF_QMODE"]), None)
d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
dt = torch.float32 if len(sys.argv) > 2 and sys.argv[2] == "f32" else torch.bfloat16
x = torch.randn(16384 if dt == torch.bfloat16 else 4096, d, device="cuda").to(dt)
cs = sign_bits(9, x.shape[0], "cuda")
for _ in range(3):
    quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_HADAMARD,
                col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=cs, col_prescale=0.75)
torch.cuda.synchronize()
