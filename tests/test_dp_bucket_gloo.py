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


def _worker_overlap(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import copy

        from paper_2505_14669_b200.llama import GradBucket, OverlappedGradBuckets

        torch.manual_seed(0)
        net = torch.nn.Sequential(torch.nn.Linear(64, 96), torch.nn.GELU(), torch.nn.Linear(96, 80),
                                  torch.nn.GELU(), torch.nn.Linear(80, 32))
        ref = copy.deepcopy(net)
        x = torch.randn(8, 64) * (rank + 1)
        # tiny buckets: several all-reduces launched from inside backward
        ob = OverlappedGradBuckets(net.parameters(), bucket_mb=0.004)
        assert len(ob.buckets) > 2
        for _ in range(2):  # two steps: the hooks re-arm after finish()
            for p in net.parameters():
                p.grad = None
            net(x).square().sum().backward()
            ob.finish()
        ref(x).square().sum().backward()
        GradBucket(ref.parameters()).allreduce()
        q.put((rank, [p.grad.numpy().copy() for p in net.parameters()], [p.grad.numpy().copy() for p in ref.parameters()]))
    finally:
        dist.destroy_process_group()


def test_overlapped_buckets_equal_flat_bucket_world2():
    """Bucketed all-reduce launched from post-accumulate-grad hooks during backward gives the same mean
    gradients as the single flat bucket (same bf16 wire values, one SUM per element)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker_overlap, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (a, b)) for r, a, b in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
    import numpy as np

    for r in range(2):
        for got, ref in zip(*out[r]):
            assert np.array_equal(got, ref)
