"""Llama-Quartet training throughput (BASELINE configs 2 / 4 / 5).

    python tools/train_llama.py --preset 200m --batch 64 --steps 5          # 1 GPU
    torchrun --nproc-per-node 8 tools/train_llama.py --preset 200m          # data parallel
    python tools/train_llama.py --preset 7b --block --batch 4               # one 7B block, 8k seq
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200 import llama

    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="200m")
    ap.add_argument("--batch", type=int, default=64, help="sequences per GPU")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--block", action="store_true", help="one transformer block (fwd+bwd), no embedding/head")
    ap.add_argument("--linear", default="quartet", choices=["quartet", "bf16"])
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    qt.load()
    dev = torch.device("cuda", local)
    print(json.dumps(run(llama, a.preset, a.batch, a.steps, a.warmup, a.block, dev, world, rank, a.linear)) if rank == 0 else "",
          flush=True)
    if world > 1:
        dist.destroy_process_group()


def run(llama, preset, batch, steps, warmup, block, dev, world=1, rank=0, linear="quartet", graph=None):
    """linear: "quartet" (every linear MXFP4 through libquartet_b200) or "bf16" (the comparator arm: the
    same model, glue kernels, optimizer and data with bf16 cuBLAS linears).  graph (default: one GPU): the
    training step is captured once as a CUDA graph and replayed (Trainer(graph=True)); both arms alike."""
    if graph is None:
        graph = world == 1
    import torch
    import torch.distributed as dist

    cfg = llama.LlamaConfig(**{**llama.PRESETS[preset].__dict__, "linear": linear})
    if block:
        cfg = llama.LlamaConfig(**{**cfg.__dict__, "n_layer": 1})
    model = llama.LlamaQuartet(cfg, seed=0, device=dev, blocks_only=block)
    tokens = batch * cfg.seq_len
    if block:
        x = (torch.randn(batch, cfg.seq_len, cfg.d_model, device=dev) * 0.5).to(torch.bfloat16).requires_grad_()
        params = list(model.parameters())

        def body():
            y = model(x=x)
            y.float().square().mean().backward()

        def step(i):
            body()
            return None

        if graph:   # as Trainer(graph=True): device-resident layer seeds, two eager warm-ups, one captured fwd+bwd
            if hasattr(model, "use_device_seeds"):
                model.use_device_seeds()
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                for _ in range(2):
                    for p in params + [x]:
                        p.grad = None
                    body()
            torch.cuda.current_stream().wait_stream(st)
            for p in params + [x]:
                p.grad = None
            cg = torch.cuda.CUDAGraph()
            with torch.cuda.graph(cg):
                body()

            def step(i):
                cg.replay()
                return None
    else:
        tr = llama.Trainer(model, steps=1000, lr=llama.PAPER_LR[preset], graph=graph)
        tok, tgt = llama.synthetic_batch(cfg, batch, seed=rank, device=dev)

        def step(i):
            return tr.step(tok, tgt)
    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(steps):
        loss = step(warmup + i)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    lin = cfg.n_layer * (4 * cfg.d_model ** 2 + 3 * cfg.d_model * cfg.hidden) + (0 if block else cfg.d_model * cfg.vocab)
    out = {"preset": preset, "linear": linear, "block_only": block, "n_layer": cfg.n_layer, "d_model": cfg.d_model,
           "launch": ("CUDA graph of the whole training step" if not block else "CUDA graph of the block's fwd+bwd")
           if graph else "eager",
           "seq_len": cfg.seq_len, "seqs_per_gpu": batch, "n_gpus": world, "ms_per_step": round(ms, 3),
           "tokens_per_s": round(world * tokens / (ms * 1e-3), 1),
           "linear_tflops": round(world * 6 * tokens * lin / (ms * 1e-3) / 1e12, 1)}
    if not block:
        out["loss"] = float(loss)
    return out


if __name__ == "__main__":
    main()
