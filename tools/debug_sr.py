"""Debug helper: locate and explain SR code mismatches of the dual/col quantizer vs the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_14669_b200 as qt  # noqa: E402
from gpu_util import bf16_values, to_dev  # noqa: E402
from oracle import oracle  # noqa: E402

T, d_out, xi = 2048, 1024, 7
dy = bf16_values(oracle.gaussians(3, oracle.DOMAIN_GAUSS, 0, T * d_out).reshape(T, d_out).astype(np.float32))
signs = qt.sign_bits(xi, max(T, d_out), "cuda")
s_r, s_c = oracle.derive_seed(xi, 21), oracle.derive_seed(xi, 23)
L = qt._lib
for name, fn in (("dual", lambda: qt.quant_dual(to_dev(dy, torch.bfloat16), L.QT_ROUND_SR,
                                                 transform=L.QT_TRANSFORM_RANDOMIZED, signs=signs, prescale=0.75,
                                                 seed_rows=s_r, seed_cols=s_c)[1]),
                 ("cols", lambda: qt.quant_cols(to_dev(dy, torch.bfloat16), L.QT_ROUND_SR,
                                                transform=L.QT_TRANSFORM_RANDOMIZED, signs=signs, prescale=0.75,
                                                sr_seed=s_c))):
    op = fn()
    gt = oracle.fwht(np.ascontiguousarray(dy.T) * oracle.signs(xi, 0, T), 32) * np.float32(0.75)
    c, s = oracle.quantize_sr(gt.astype(np.float64), 32, s_c, 0)
    got = op.unpacked_codes().cpu().numpy()
    gs = op.scales_rowmajor().cpu().numpy()
    print(name, "scale mismatches", int((gs != s).sum()), "code mismatches", int((got != c).sum()))
    for (i, j) in np.argwhere(got != c)[:5]:
        x = np.float64(gt[i, j])
        e = int(s[i, j // 32])
        v = x / np.ldexp(1.0, e - 127)
        u = oracle.uniform(s_c, oracle.DOMAIN_SR, i * T + j, 1)[0]
        print(f"  [{i},{j}] gpu {got[i, j]} ref {c[i, j]} x={x!r} e={e} v={v!r} u={u!r}")
        grp = gt[i, (j // 32) * 32:(j // 32) * 32 + 32]
        print("   group absmax", np.abs(grp).max())
