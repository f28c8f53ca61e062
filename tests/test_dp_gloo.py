"""Data-parallel decomposition of the Quartet layer, world_size 2 over gloo on CPU.

Each rank runs the reference algorithm (the CPU oracle stands in for its GPU) on its token shard
with the global token offset that paper_2505_14669_b200.dp / qlinear.backward(token_offset=...) use,
then the dW partials are summed with torch.distributed (the NCCL all-reduce on B200 nodes).  Checked
against one single-process run over all tokens:
  * the shard's quantized operands G_t / X_t are bit-exact column slices of the full ones,
  * dx rows are bit-exact,
  * sum_r dw_r matches dw within 1e-6 relative Frobenius (fp32 summation order only).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(T, d_in, d_out):
    r = np.random.default_rng(123)
    x = r.normal(size=(T, d_in)).astype(np.float32)
    w = (r.normal(size=(d_out, d_in)) / np.sqrt(d_in)).astype(np.float32)
    dy = r.normal(size=(T, d_out)).astype(np.float32)
    return x, w, dy


def _worker(rank, world, port, rounding, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle
    from paper_2505_14669_b200.dp import allreduce_dw, token_shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T, d_in, d_out, xi = 128, 64, 96, 17
    x, w, dy = _inputs(T, d_in, d_out)
    off, n = token_shard(T, rank, world)
    _, ctx = oracle.forward(x[off:off + n], w)
    dx, dw = oracle.backward(dy[off:off + n], ctx, xi=xi, rounding=rounding, token_offset=off, total_tokens=T)
    dwt = torch.from_numpy(dw.astype(np.float64))
    allreduce_dw(dwt, comm_dtype=None)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), dx=dx, dw=dwt.numpy(), off=off,
             gt_c=ctx.inter["gtq"][0], gt_s=ctx.inter["gtq"][1], xt_c=ctx.inter["xtq"][0], xt_s=ctx.inter["xtq"][1])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("rounding", ["rtn", "sr"])
def test_dp_two_ranks_matches_single(tmp_path, rounding):
    from oracle import oracle

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), rounding, str(tmp_path)), nprocs=world, join=True)
    T, d_in, d_out, xi = 128, 64, 96, 17
    x, w, dy = _inputs(T, d_in, d_out)
    _, ctx = oracle.forward(x, w)
    dx_full, dw_full = oracle.backward(dy, ctx, xi=xi, rounding=rounding)
    gt_c, gt_s = ctx.inter["gtq"]
    xt_c, xt_s = ctx.inter["xtq"]
    for r in range(world):
        z = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        off, n = int(z["off"]), z["dx"].shape[0]
        assert np.array_equal(z["dx"], dx_full[off:off + n])
        assert np.array_equal(z["gt_c"], gt_c[:, off:off + n]) and np.array_equal(z["gt_s"], gt_s[:, off // 32:(off + n) // 32])
        assert np.array_equal(z["xt_c"], xt_c[:, off:off + n]) and np.array_equal(z["xt_s"], xt_s[:, off // 32:(off + n) // 32])
        dw = z["dw"]
        assert np.linalg.norm(dw - dw_full) <= 1e-6 * np.linalg.norm(dw_full)


def test_token_shard_rules():
    from paper_2505_14669_b200.dp import token_shard

    assert token_shard(256, 1, 2) == (128, 128)
    with pytest.raises(ValueError):
        token_shard(96, 0, 2)
