"""Llama-style model with every linear in Quartet MXFP4 (BASELINE configs 2/4/5 building blocks)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def llama():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200 import llama

    qt.load()
    return llama


def test_all_linears_are_quartet(llama):
    from paper_2505_14669_b200.nn import QuartetLinear

    cfg = llama.LlamaConfig(n_layer=2, d_model=256, n_head=2, vocab=1024, seq_len=64)
    m = llama.LlamaQuartet(cfg, device="cuda")
    assert not any(isinstance(mod, torch.nn.Linear) for mod in m.modules())
    assert sum(isinstance(mod, QuartetLinear) for mod in m.modules()) == 2 * 7 + 1


def test_training_reduces_loss(llama):
    torch.manual_seed(0)
    cfg = llama.LlamaConfig(n_layer=2, d_model=256, n_head=2, vocab=1024, seq_len=128)
    m = llama.LlamaQuartet(cfg, seed=1, device="cuda")
    tr = llama.Trainer(m, steps=40, lr=3e-3)
    tok, tgt = llama.synthetic_batch(cfg, 16, seed=3, device="cuda")
    losses = [float(tr.step(tok, tgt)) for _ in range(40)]
    assert all(l == l and l < 1e4 for l in losses)  # finite
    assert losses[-1] < losses[0] - 1.0, losses


def test_30m_forward_backward_shapes(llama):
    """BASELINE config 2 architecture (Llama-30M: 6 x 640, 5 heads), one step on a short batch."""
    cfg = llama.PRESETS["30m"]
    m = llama.LlamaQuartet(cfg, device="cuda")
    assert 25e6 < cfg.n_params() < 40e6
    tr = llama.Trainer(m, steps=10, lr=llama.PAPER_LR["30m"])
    tok, tgt = llama.synthetic_batch(cfg, 2, seed=0, device="cuda")
    loss = tr.step(tok, tgt)
    assert torch.isfinite(loss)
    assert all(p.grad is not None and torch.isfinite(p.grad).all() for p in m.parameters())


def test_lr_schedule_matches_reference(llama):
    """train.py:76-85 (warm-up 10 %, cosine to lr_floor)."""
    steps, lr = 100, 1.0
    assert llama.lr_at(0, steps, lr) == pytest.approx(0.1)
    assert llama.lr_at(9, steps, lr) == pytest.approx(1.0)
    assert llama.lr_at(99, steps, lr) == pytest.approx(0.0, abs=1e-12)
