"""Data-parallel Llama step on one GPU: two ranks over gloo, each holding half of the
sequences, reproduce the one-rank step on the concatenated batch.

Each rank's Quartet layers use the global token offset (nn.set_token_shard via Trainer._place_shard), so their
G / G_t / X_t operands are exact slices of the single-rank operands and their dX rows are the single-rank
rows; the per-rank dW are partial token sums.  The remaining differences are the fp32 order of the dW sums and
the bf16 wire format of the gradient all-reduce (llama.OverlappedGradBuckets), i.e. ~2^-8 relative:
stated tolerance 2e-2 relative on every gradient, 1e-5 on the loss (mean of the ranks' losses)."""

import os

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(n_layer=2, d_model=128, n_head=4, vocab=512, seq_len=64, d_ff=256)
BATCH = 4   # global sequences; 2 per rank -> 128 tokens per rank (a multiple of 32)


def _step(model, tokens, targets):
    from paper_2505_14669_b200.llama import OverlappedGradBuckets, cross_entropy
    from paper_2505_14669_b200.nn import set_token_shard
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    set_token_shard(model, rank * tokens.numel(), world * tokens.numel() if world > 1 else None)
    params = [p for p in model.parameters() if p.requires_grad]
    bucket = OverlappedGradBuckets(params, bucket_mb=0.25)
    logits = model(tokens)
    loss = cross_entropy(logits.view(-1, logits.shape[-1]), targets.reshape(-1))
    loss.backward()
    bucket.finish()
    return float(loss.detach()), [p.grad.float().cpu() for p in params]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2505_14669_b200.llama import LlamaConfig, LlamaQuartet, synthetic_batch

        cfg = LlamaConfig(**CFG)
        model = LlamaQuartet(cfg, seed=3, device="cuda")
        tok, tgt = synthetic_batch(cfg, BATCH, seed=9, device="cuda")
        per = BATCH // world
        loss, grads = _step(model, tok[rank * per:(rank + 1) * per], tgt[rank * per:(rank + 1) * per])
        q.put((rank, loss, grads))
    finally:
        dist.destroy_process_group()


def test_two_rank_step_equals_one_rank_step():
    from paper_2505_14669_b200.llama import LlamaConfig, LlamaQuartet, synthetic_batch

    cfg = LlamaConfig(**CFG)
    model = LlamaQuartet(cfg, seed=3, device="cuda")
    tok, tgt = synthetic_batch(cfg, BATCH, seed=9, device="cuda")
    ref_loss, ref_grads = _step(model, tok, tgt)

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29400 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {r: (loss, grads) for r, loss, grads in (q.get(timeout=300) for _ in range(2))}
    for p in procs:
        p.join(timeout=60)
    assert abs((out[0][0] + out[1][0]) / 2 - ref_loss) <= 1e-5 * abs(ref_loss)
    for i, ref in enumerate(ref_grads):
        for r in range(2):
            got = out[r][1][i]
            err = float((got - ref).norm() / ref.norm().clamp_min(1e-30))
            assert err <= 2e-2, (i, r, err)
        assert torch.equal(out[0][1][i], out[1][1][i])   # every rank holds the same averaged gradient
