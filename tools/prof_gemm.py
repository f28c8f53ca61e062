"""One fwd GEMM at T x d_in -> d_out (for ncu; not a bench number)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import gemm, quant_rows
qt.load()
T, di, do = 16384, int(sys.argv[1]) if len(sys.argv) > 1 else 4096, int(sys.argv[2]) if len(sys.argv) > 2 else 4096
x = torch.randn(T, di, device="cuda").to(torch.bfloat16)
w = torch.randn(do, di, device="cuda")
xq = quant_rows(x, 1, _lib.QT_ROUND_QUEST)
wq = quant_rows(w, 1, _lib.QT_ROUND_QUEST)
for _ in range(3):
    gemm(xq, wq, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
