"""One Quartet fwd+bwd step for ncu / per-kernel timing (not a bench number).

    python tools/prof_step.py [--din 4096] [--dout 4096] [--tokens 16384] [--iters 2] [--rounding rtn]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--din", type=int, default=4096)
    ap.add_argument("--dout", type=int, default=4096)
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--rounding", default="rtn")
    ap.add_argument("--events", action="store_true", help="print per-call CUDA-event times")
    ap.add_argument("--all-shapes", action="store_true", help="the bench step: 4096->4096, 4096->11008, 11008->4096")
    a = ap.parse_args()
    qt.load()
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    if a.all_shapes:
        data = []
        for d_in, d_out in ((4096, 4096), (4096, 11008), (11008, 4096)):
            data.append((torch.randn(a.tokens, d_in, device=dev, generator=g).to(torch.bfloat16),
                         torch.randn(d_out, d_in, device=dev, generator=g) / d_in ** 0.5,
                         torch.randn(a.tokens, d_out, device=dev, generator=g).to(torch.bfloat16)))
        for it in range(a.iters):
            for i, (x, w, dy) in enumerate(data):
                y, ctx = qt.forward(x, w, out_dtype=torch.bfloat16, check_finite=False, bwd_xi=it * 3 + i,
                                    bwd_rounding=a.rounding)
                qt.backward(dy, ctx, xi=it * 3 + i, rounding=a.rounding, dx_dtype=torch.bfloat16, check_finite=False)
        torch.cuda.synchronize()
        return
    x = torch.randn(a.tokens, a.din, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(a.dout, a.din, device=dev, generator=g) / a.din ** 0.5
    dy = torch.randn(a.tokens, a.dout, device=dev, generator=g).to(torch.bfloat16)
    import paper_2505_14669_b200.qlinear as ql

    times = []
    if a.events:
        def wrap(fn, name):
            def f(*args, **kw):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                o = fn(*args, **kw)
                e.record()
                times.append((name, s, e))
                return o
            return f
        ql.gemm = wrap(ql.gemm, "gemm")
        ql.quant_rows = wrap(ql.quant_rows, "quant_rows")
        ql.quant_cols = wrap(ql.quant_cols, "quant_cols")
    import time
    for it in range(a.iters):
        times.clear()
        s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s0.record()
        y, ctx = qt.forward(x, w, out_dtype=torch.bfloat16, check_finite=False, bwd_xi=it, bwd_rounding=a.rounding)
        dx, dw = qt.backward(dy, ctx, xi=it, rounding=a.rounding, dx_dtype=torch.bfloat16, check_finite=False)
        t1 = time.perf_counter()
        e0.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"iter {it}: gpu {s0.elapsed_time(e0) * 1e3:.1f} us, cpu launch {1e6 * (t1 - t0):.1f} us, "
              f"wall {1e6 * (t2 - t0):.1f} us")
    torch.cuda.synchronize()
    for name, s, e in times:
        print(f"{name:12s} {s.elapsed_time(e) * 1e3:9.1f} us")


if __name__ == "__main__":
    main()
