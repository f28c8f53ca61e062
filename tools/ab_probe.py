"""A/B timing of the hot kernels for one library build (QT_LIB_PATH selects an experiment build).

    QT_LIB_PATH=exp/v1/libquartet_b200.so python tools/ab_probe.py [tag]

Prints one line per kernel: median of 5 rounds of 10 back-to-back launches (CUDA events), at the bench's
16384-token shapes, plus the dual quantizer's exact-path fallback count.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200 import _lib  # noqa: E402
from paper_2505_14669_b200.mxfp4 import gemm, quant_dual, quant_fused, sign_bits  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("QT_LIB_PATH", "prod")
L = qt.load()
torch.manual_seed(0)


def timeit(f, reps=10, rounds=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(rounds):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            f()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1000 / reps)
    return sorted(ts)[len(ts) // 2]


out = {}
for d in (4096, 11008):
    dy = torch.randn(16384, d, device="cuda").to(torch.bfloat16)
    rs, cs = sign_bits(5, d, "cuda"), sign_bits(9, 16384, "cuda")
    out[f"dual_{d}"] = timeit(lambda: quant_dual(dy, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_RANDOMIZED,
                                                 signs=rs, col_signs=cs, prescale=0.75))
    x = torch.randn(16384, d, device="cuda").to(torch.bfloat16)
    out[f"fusedX_{d}"] = timeit(lambda: quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN,
                                                    transform=_lib.QT_TRANSFORM_HADAMARD,
                                                    col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=cs,
                                                    col_prescale=0.75))
dy = torch.randn(16384, 4096, device="cuda").to(torch.bfloat16)
rs, cs = sign_bits(5, 4096, "cuda"), sign_bits(9, 16384, "cuda")
for name, rc in (("sr", _lib.QT_ROUND_SR), ("srfast", _lib.QT_ROUND_SR_FAST)):
    out[f"dual_{name}_4096"] = timeit(lambda: quant_dual(dy, rc, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs,
                                                         col_signs=cs, prescale=0.75, seed_rows=1, seed_cols=2))
    out[f"fusedX_{name}_4096"] = timeit(lambda: quant_fused(dy, _lib.QT_ROUND_QUEST, rc,
                                                            transform=_lib.QT_TRANSFORM_HADAMARD,
                                                            col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=cs,
                                                            col_prescale=0.75, col_seed=3))
w = torch.randn(4096, 4096, device="cuda") / 64
ws = sign_bits(3, 4096, "cuda")
out["fusedW_4096"] = timeit(lambda: quant_fused(w, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN,
                                                transform=_lib.QT_TRANSFORM_HADAMARD,
                                                col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=ws,
                                                col_prescale=0.75))
fb = torch.zeros(1, dtype=torch.int32, device="cuda")
L.qt_debug_set_quant(0, fb.data_ptr())
dy = torch.randn(16384, 4096, device="cuda").to(torch.bfloat16)
rs, cs = sign_bits(5, 4096, "cuda"), sign_bits(9, 16384, "cuda")
quant_dual(dy, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_RANDOMIZED, signs=rs, col_signs=cs, prescale=0.75)
torch.cuda.synchronize()
L.qt_debug_set_quant(0, None)
out["dual_fallback_groups"] = int(fb.item())
xq, _ = quant_fused(torch.randn(16384, 4096, device="cuda").to(torch.bfloat16), _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN,
                    transform=_lib.QT_TRANSFORM_HADAMARD, col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=cs)
wq, _ = quant_fused(torch.randn(4096, 4096, device="cuda"), _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN,
                    transform=_lib.QT_TRANSFORM_HADAMARD, col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=ws)
yb = torch.empty(16384, 4096, device="cuda", dtype=torch.bfloat16)
out["gemm_fwd_4096"] = timeit(lambda: gemm(xq, wq, out=yb))
print(tag, " ".join(f"{k}={v:.1f}" if isinstance(v, float) else f"{k}={v}" for k, v in out.items()), flush=True)
