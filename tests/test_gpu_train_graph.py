"""Graph-captured Llama training step (llama.Trainer(graph=True)): the device-resident layer seeds equal the
host seeds of the reference's loop (train.py:346-348), and the captured step trains like the eager step."""

import pytest
import torch

pytestmark = pytest.mark.gpu

CFG = dict(n_layer=2, d_model=128, n_head=4, vocab=512, seq_len=64, d_ff=256)


def test_device_seeds_equal_host_seeds():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200.llama import LlamaConfig, LlamaQuartet
    from paper_2505_14669_b200.nn import QuartetLinear

    qt.load()
    model = LlamaQuartet(LlamaConfig(**CFG), seed=11, device="cuda")
    mods = [m for m in model.modules() if isinstance(m, QuartetLinear)]
    for m in mods:
        m.step = 5
    host = [[(m.seed, m.layer_id)] for m in mods]
    model.use_device_seeds()
    xi_dev, _, step_dev, _, _ = model._seeds
    from paper_2505_14669_b200.mxfp4 import derive_seed

    for step in (5, 6, 7):
        model._launch_seeds()
        got = [int(v) & 0xFFFFFFFFFFFFFFFF for v in xi_dev.cpu().tolist()]
        want = [derive_seed(derive_seed(m.seed, 4, step), m.layer_id) for m in mods]
        assert got == want, step
    assert int(step_dev.item()) == 8


def test_graph_step_trains_like_eager_step():
    import paper_2505_14669_b200 as qt
    from paper_2505_14669_b200.llama import LlamaConfig, LlamaQuartet, Trainer, synthetic_batch

    qt.load()
    cfg = LlamaConfig(**CFG)
    tok, tgt = synthetic_batch(cfg, 4, seed=3, device="cuda")
    losses = {}
    for graph in (False, True):
        model = LlamaQuartet(cfg, seed=7, device="cuda")
        tr = Trainer(model, steps=20, lr=1e-3, graph=graph)
        losses[graph] = [float(tr.step(tok, tgt)) for _ in range(6)]
    # same kernels in the same order; the capturable AdamW takes lr as a device scalar
    for a, b in zip(losses[False], losses[True]):
        assert abs(a - b) <= 1e-3 * abs(a), (losses[False], losses[True])
    assert losses[True][-1] < losses[True][0]
