"""Data parallelism for the Quartet linear layer: token shards + one dW all-reduce.

The hot path shards along tokens: forward rows are independent, the dX GEMM
contracts over d_out, and the dW GEMM is a sum over tokens -- the only exchange step.  Each rank runs
its own token shard through the same kernels with the GLOBAL token offset (randomized-Hadamard signs
and stochastic-rounding stream positions along the token axis), so:

  * every quantized operand a rank builds is exactly the matching slice of the single-GPU operand,
  * its dx rows are exactly the single-GPU dx rows,
  * sum_r dw_r equals the single-GPU dw up to fp32 summation order (the masked FWHT-32 * 16/9
    epilogue is linear, so it commutes with the all-reduce).

The all-reduce runs on torch.distributed (NCCL over NVLink on B200 nodes, gloo in the CPU tests).
"""

from __future__ import annotations

import torch

GROUP = 32


def token_shard(total_tokens: int, rank: int, world: int) -> tuple[int, int]:
    """(offset, count) of rank's equal token shard; shards are whole 32-token Hadamard blocks."""
    if total_tokens % (GROUP * world):
        raise ValueError(f"{total_tokens} tokens do not split into {world} shards of whole {GROUP}-token blocks")
    count = total_tokens // world
    return rank * count, count


def allreduce_dw(dw: torch.Tensor, group=None, comm_dtype: torch.dtype | None = torch.bfloat16) -> torch.Tensor:
    """Sum dw over the data-parallel group in place (optionally communicating in bf16)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return dw
    if comm_dtype is None or comm_dtype == dw.dtype:
        dist.all_reduce(dw, group=group)
        return dw
    buf = dw.to(comm_dtype)
    dist.all_reduce(buf, group=group)
    dw.copy_(buf)
    return dw
