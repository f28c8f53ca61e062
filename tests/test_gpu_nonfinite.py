"""Non-finite inputs on the autograd / training path (the reference raises ValueError("non-finite input"),
codec.py:164-170, and its training loop stops on divergence, train.py:341-343).  The Quartet layers OR the
quantizers' non-finite bit into a per-device flag without a host sync; nn.raise_if_nonfinite checks it once,
and the Trainer checks the previous step's flag (copied asynchronously) at the start of the next step."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_layer_flag_and_raise():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200 import nn

    qt.load()
    nn.raise_if_nonfinite()                       # clean state
    layer = qt.QuartetLinear(64, 32, seed=1).cuda()
    x = torch.randn(64, 64, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    layer(x).float().sum().backward()
    nn.raise_if_nonfinite()                       # finite: no error
    x2 = x.detach().clone()
    x2[3, 5] = float("nan")
    layer(x2.requires_grad_()).float().sum().backward()
    with pytest.raises(ValueError, match="non-finite"):
        nn.raise_if_nonfinite()
    nn.raise_if_nonfinite()                       # the flag was cleared


def test_trainer_stops_on_divergence():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200 import nn
    from paper_2505_14669_b200.llama import LlamaConfig, LlamaQuartet, Trainer, synthetic_batch

    qt.load()
    nn.raise_if_nonfinite()
    cfg = LlamaConfig(n_layer=1, d_model=128, n_head=4, vocab=256, seq_len=64, d_ff=256)
    model = LlamaQuartet(cfg, seed=2, device="cuda")
    tr = Trainer(model, steps=4, lr=1e-3)
    tok, tgt = synthetic_batch(cfg, 2, seed=1, device="cuda")
    tr.step(tok, tgt)
    tr.step(tok, tgt)                             # finite steps pass the lagged check
    with torch.no_grad():
        model.blocks[0].q.weight[0, 0] = float("inf")
    tr.step(tok, tgt)                             # the non-finite weight is quantized here ...
    torch.cuda.synchronize()
    with pytest.raises(ValueError, match="non-finite"):
        tr.step(tok, tgt)                         # ... and reported once that step has finished
    tr.check_finite(wait=True)                    # the flag was cleared
