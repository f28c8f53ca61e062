"""Quantizer-only timing table (development aid; bench.py is the contract)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_14669_b200 as qt
from bench import kernel_table, SHAPES

qt.load()
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
T = 16384
data = [(torch.randn(T, di, device=dev, generator=g).to(torch.bfloat16),
         torch.randn(do, di, device=dev, generator=g) / di ** 0.5,
         torch.randn(T, do, device=dev, generator=g).to(torch.bfloat16)) for di, do in SHAPES]
tot = {}
for r in kernel_table(qt, data, dev, reps=10):
    tot[r["kind"]] = tot.get(r["kind"], 0) + r["us"]
    print(f"{r['kernel']:14s} {r['shape']:12s} {r['us']:8.1f} us  " + (f"{r['gbs']:7.1f} GB/s" if r['kind'] == 'quant' else f"{r['tflops']:7.1f} TF/s"))
print({k: round(v, 1) for k, v in tot.items()})
