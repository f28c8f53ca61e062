"""GEMM launch times at the Llama-30M training shapes (64 x 512 tokens, d = 640, ffn 1792, vocab 32000), each
with its multiplicity per training step, next to torch bf16 matmul of the same shape.  Timing only."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200 import _lib  # noqa: E402

L = qt.load()
L.qt_debug_set_gemm.argtypes = [ctypes.c_int]
preset = sys.argv[1] if len(sys.argv) > 1 else "30m"
T = 32768
d, h, V, nl = {"30m": (640, 1792, 32000, 6), "200m": (1280, 3584, 32000, 10)}[preset]


def operand(r, c):
    return qt.quant_rows(torch.randn(r, c, device="cuda").to(torch.bfloat16), 0, _lib.QT_ROUND_RTN)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e3 / reps


# (name, M, N, K, out dtype, launches per step)
shapes = [("fwd qkvo", T, d, d, torch.bfloat16, 4 * nl), ("fwd gate/up", T, h, d, torch.bfloat16, 2 * nl),
          ("fwd down", T, d, h, torch.bfloat16, nl), ("fwd head", T, V, d, torch.bfloat16, 1),
          ("dx qkvo", T, d, d, torch.bfloat16, 4 * nl), ("dx gate/up", T, d, h, torch.bfloat16, 2 * nl),
          ("dx down", T, h, d, torch.bfloat16, nl), ("dx head", T, d, V, torch.bfloat16, 1),
          ("dw qkvo", d, d, T, torch.float32, 4 * nl), ("dw gate/up", h, d, T, torch.float32, 2 * nl),
          ("dw down", d, h, T, torch.float32, nl), ("dw head", V, d, T, torch.float32, 1)]
tot = tot_bf = 0.0
for name, M, N, K, dt, n in shapes:
    A, B = operand(M, K), operand(N, K)
    out = torch.empty(M, N, device="cuda", dtype=dt)
    us = timed(lambda: qt.gemm(A, B, out=out))
    a16 = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b16 = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    ub = timed(lambda: torch.matmul(a16, b16))
    tot += us * n
    tot_bf += ub * n
    print(f"{name:12s} M{M:6d} N{N:6d} K{K:6d} x{n:3d}: {us:7.1f} us {2 * M * N * K / us / 1e6:6.0f} TF | "
          f"bf16 {ub:7.1f} us", flush=True)
print(f"per step: mxfp4 {tot / 1e3:.2f} ms, bf16 {tot_bf / 1e3:.2f} ms")
