"""Cross-entropy kernel timing at the Llama vocab ([32768, 32000] bf16 logits): forward (log-sum-exp) and
backward (softmax - onehot) of paper_2505_14669_b200.llama.cross_entropy, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from paper_2505_14669_b200.llama import cross_entropy  # noqa: E402

qt.load()
x = (torch.randn(32768, 32000, device="cuda") * 2).to(torch.bfloat16).requires_grad_()
t = torch.randint(0, 32000, (32768,), device="cuda")


def timed(f, reps=10):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        f()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1000


fwd = timed(lambda: cross_entropy(x, t))
both = timed(lambda: cross_entropy(x, t).backward())
ref = torch.nn.functional.cross_entropy(x.float(), t)
got = cross_entropy(x, t)
print(f"xent fwd {fwd:.1f} us, fwd+bwd {both:.1f} us; loss {float(got.detach()):.6f} vs torch fp32 {float(ref.detach()):.6f}", flush=True)
