import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import llama
qt.load()
cfg = llama.PRESETS["200m"]
m = llama.LlamaQuartet(cfg, device="cuda")
tr = llama.Trainer(m, steps=100, lr=3e-4)
tok, tgt = llama.synthetic_batch(cfg, 64, seed=0, device="cuda")
for _ in range(2): tr.step(tok, tgt)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], record_shapes=True) as p:
    tr.step(tok, tgt)
    torch.cuda.synchronize()
for e in sorted(p.key_averages(group_by_input_shape=True), key=lambda e: -e.self_device_time_total)[:25]:
    if e.self_device_time_total > 300:
        print(f"{e.self_device_time_total/1e3:7.2f} ms  x{e.count:3d}  {e.key[:60]:60s} {str(e.input_shapes)[:90]}")
