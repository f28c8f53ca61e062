"""torch.profiler breakdown of one Llama-Quartet training step (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import llama
qt.load()
preset = sys.argv[1] if len(sys.argv) > 1 else "200m"
cfg = llama.PRESETS[preset]
m = llama.LlamaQuartet(cfg, device="cuda")
tr = llama.Trainer(m, steps=100, lr=3e-4)
tok, tgt = llama.synthetic_batch(cfg, 64, seed=0, device="cuda")
for _ in range(2): tr.step(tok, tgt)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as p:
    tr.step(tok, tgt)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=160))
