"""Data-parallel gradient bucket (paper_2505_14669_b200.llama.GradBucket) on CPU with gloo, world size 2:
after the all-reduce every rank holds the mean gradient (bf16 on the wire)."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_14669_b200.llama import GradBucket

        torch.manual_seed(0)
        lin = torch.nn.Linear(64, 32, bias=True)
        x = torch.randn(8, 64) * (rank + 1)
        lin(x).square().sum().backward()
        grads = [p.grad.clone() for p in lin.parameters()]
        GradBucket(lin.parameters()).allreduce()
        q.put((rank, [g.numpy() for g in grads], [p.grad.numpy().copy() for p in lin.parameters()]))
    finally:
        dist.destroy_process_group()


def test_bucket_allreduce_mean_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (g, a)) for r, g, a in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
    import numpy as np

    for i in range(2):
        mean = (out[0][0][i].astype(np.float64) + out[1][0][i]) / 2
        for r in range(2):
            got = out[r][1][i]
            assert np.allclose(got, mean, rtol=2e-2, atol=1e-2 * np.abs(mean).max())
        assert np.array_equal(out[0][1][i], out[1][1][i])
