"""RMSNorm glue kernels at the Llama shapes (32768 rows): forward / backward, with and without the fused
residual stream (qt_rmsnorm_res), next to torch's bf16 add of the same size.  Timing only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_14669_b200 import _lib  # noqa: E402

L = _lib.load()


def t(f, n=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000 / n


for d in (640, 1280, 4096):
    R = 32768
    x, y, dy = (torch.randn(R, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    w = torch.rand(d, device="cuda") + 0.5
    out, h = torch.empty_like(x), torch.empty_like(x)
    rstd = torch.empty(R, device="cuda")
    dw = torch.zeros(d, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    P = lambda a: a.data_ptr() if a is not None else None  # noqa: E731

    def run(res, bwd):
        return lambda: L.qt_rmsnorm_res(P(x), P(res), P(w), P(dy) if bwd else None, P(out), None if bwd else P(h),
                                        P(rstd), P(dw) if bwd else None, R, d, 1e-6, int(bwd), s)
    run(None, False)()
    mb = R * d * 2 / 1e6
    rows = [("fwd", run(None, False), 2), ("fwd+res", run(y, False), 4), ("bwd", run(None, True), 3),
            ("bwd+res", run(y, True), 4), ("torch add", lambda: torch.add(x, y, out=out), 3)]
    print(f"d={d}: " + " | ".join(f"{n} {t(f):6.1f} us ({k * mb / t(f):4.1f} TB/s)" for n, f, k in rows),
          flush=True)
