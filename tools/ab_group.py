"""A/B of the shared-input group quantization: rows-only X_q + one requantization per layer vs the fused
X_q + X_t of the first layer + requantizations of the others (nn.QuartetLinearGroupFn)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib, qlinear
from paper_2505_14669_b200.mxfp4 import quant_fused, quant_cols, sign_bits
qt.load()
def timeit(f, reps=10, rounds=5):
    f(); torch.cuda.synchronize(); ts = []
    for _ in range(rounds):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps): f()
        e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e) * 1000 / reps)
    return sorted(ts)[len(ts) // 2]
for R, C in ((32768, 4096), (32768, 1280), (16384, 4096)):
    x = torch.randn(R, C, device="cuda").to(torch.bfloat16)
    cs = [sign_bits(9 + i, R, "cuda") for i in range(3)]
    H, RT = _lib.QT_TRANSFORM_HADAMARD, _lib.QT_TRANSFORM_RANDOMIZED
    def a():
        xq = qlinear.quantize_operand(x, qlinear.QUEST, True)
        for s in cs: quant_cols(xq, _lib.QT_ROUND_RTN, transform=RT, signs=s, prescale=0.75)
    def b():
        xq, _ = quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN, transform=H, col_transform=RT, col_signs=cs[0], col_prescale=0.75)
        for s in cs[1:]: quant_cols(xq, _lib.QT_ROUND_RTN, transform=RT, signs=s, prescale=0.75)
    def rows(): qlinear.quantize_operand(x, qlinear.QUEST, True)
    xq = qlinear.quantize_operand(x, qlinear.QUEST, True)
    def cols(): quant_cols(xq, _lib.QT_ROUND_RTN, transform=RT, signs=cs[0], prescale=0.75)
    def fused(): quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN, transform=H, col_transform=RT, col_signs=cs[0], col_prescale=0.75)
    print(R, C, {k: round(timeit(f), 1) for k, f in (("rows+3cols", a), ("fused+2cols", b), ("rows", rows), ("cols", cols), ("fused", fused))}, flush=True)
