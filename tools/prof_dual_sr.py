"""One exact-SR dual quantizer call (CUDA-core k_quant, the reference's splitmix64 stream) at 16384 x 4096 (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200 import _lib  # noqa: E402
from paper_2505_14669_b200.mxfp4 import quant_dual, sign_bits  # noqa: E402

qt.load()
x = torch.randn(16384, 4096, device="cuda").to(torch.bfloat16)
rs, cs = sign_bits(5, 4096, "cuda"), sign_bits(9, 16384, "cuda")
for _ in range(3):
    quant_dual(x, _lib.QT_ROUND_SR, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs, col_signs=cs, prescale=0.75,
               seed_rows=1, seed_cols=2)
torch.cuda.synchronize()
