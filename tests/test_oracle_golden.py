"""Pin the CPU oracle (oracle/quartet_oracle.c + oracle/oracle.py) to the reference's own outputs.

The fixtures were produced by running the reference (mx4train) itself -- see
tests/golden/make_golden.py.  Everything here is bit-exact except where the reference itself
is floating-point end to end (qlinear y/dx/dw are also bit-exact: same op order).
"""

import os

import numpy as np
import pytest


def _load(golden_dir, name):
    return np.load(os.path.join(golden_dir, name), allow_pickle=False)


def test_rng_derive_seed(oracle, golden_dir):
    z = _load(golden_dir, "rng.npz")
    for s, tag, want in z["derive"]:
        assert oracle.derive_seed(int(s), int(tag)) == int(want)
    assert oracle.derive_seed(3, 4, 5) == int(z["derive3"][0])


def test_rng_signs_uniform(oracle, golden_dir):
    z = _load(golden_dir, "rng.npz")
    assert np.array_equal(oracle.signs(7, 0, 4096, np.float64), z["signs_7"])
    assert np.array_equal(oracle.signs(2**64 - 1, 100, 333, np.float64), z["signs_big"])
    assert np.array_equal(oracle.uniform(1234, oracle.DOMAIN_SR, 17, 1000), z["uniform_sr"])
    assert np.array_equal(oracle.gaussians(1, oracle.DOMAIN_GAUSS, 0, 1000), z["gauss"])


def test_kernels_quantizers(oracle, golden_dir):
    z = _load(golden_dir, "kernels.npz")
    for i in range(int(z["n"])):
        x = z[f"x{i}"]
        c, s = oracle.quantize_rtn(x, 32)
        assert np.array_equal(c, z[f"rtn_codes{i}"]) and np.array_equal(s, z[f"rtn_scales{i}"]), i
        c, s = oracle.quantize_sr(x, 32, 1234 + i, 17)
        assert np.array_equal(c, z[f"sr_codes{i}"]) and np.array_equal(s, z[f"sr_scales{i}"]), i
        c, s, m = oracle.quantize_quest(x, 32, 1.0 / 16.0)
        assert np.array_equal(c, z[f"quest_codes{i}"]), i
        assert np.array_equal(s, z[f"quest_scales{i}"]), i
        assert np.array_equal(m, z[f"quest_mask{i}"]), i


@pytest.mark.parametrize("g", [2, 16, 32, 256])
@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_kernels_fwht(oracle, golden_dir, g, dt):
    z = _load(golden_dir, "fwht.npz")
    key = f"g{g}_{dt}"
    assert np.array_equal(oracle.fwht(z["x_" + key], g), z["y_" + key])


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_kernels_gemm(oracle, golden_dir, dt):
    z = _load(golden_dir, "gemm.npz")
    assert np.array_equal(oracle.gemm_nt(z["a_" + dt], z["b_" + dt]), z["c_" + dt])


def test_threads_do_not_change_results(oracle, golden_dir):
    z = _load(golden_dir, "kernels.npz")
    x = z["x6"]
    base = oracle.quantize_quest(x, 32, 1.0 / 16.0)
    oracle.set_threads(4)
    try:
        par = oracle.quantize_quest(x, 32, 1.0 / 16.0)
        g = _load(golden_dir, "gemm.npz")
        assert np.array_equal(oracle.gemm_nt(g["a_float32"], g["b_float32"]), g["c_float32"])
    finally:
        oracle.set_threads(1)
    for a, b in zip(base, par):
        assert np.array_equal(a, b)


CASES = ["quest_rtn", "quest_sr", "quest_rtn_t256", "rtnfwd_rtn", "quest_rtn_noh", "srfwd_sr", "srfwd_rtn_t256",
         "quest_rtn_noh_ragged", "quest_sr_noh_ragged", "rtnfwd_sr_noh_ragged"]


@pytest.mark.parametrize("case", CASES)
def test_qlinear_end_to_end(oracle, golden_dir, case):
    z = _load(golden_dir, f"qlinear_{case}.npz")
    seed = int(z["seed"]) if "seed" in z.files else None   # sr_absmax forward (qlinear.py:148-154)
    y, ctx = oracle.forward(z["x"], z["w"], scheme=str(z["scheme"]), hadamard=bool(z["hadamard"]), seed=seed)
    assert np.array_equal(oracle.pack_nibbles(ctx.x_codes), z["x_codes"])
    assert np.array_equal(ctx.x_scales, z["x_scales"])
    assert np.array_equal(oracle.pack_nibbles(ctx.w_codes), z["w_codes"])
    assert np.array_equal(ctx.w_scales, z["w_scales"])
    assert np.array_equal(ctx.m_x, z["m_x"]) and np.array_equal(ctx.m_w, z["m_w"])
    assert np.array_equal(y, z["y"])
    dx, dw = oracle.backward(z["dy"], ctx, xi=int(z["xi"]), rounding=str(z["rounding"]))
    assert np.array_equal(dx, z["dx"])
    assert np.array_equal(dw, z["dw"])


def test_golden_mxf4_container(oracle, golden_dir):
    # selftest.py:63-83 golden tensor: 5x67 gaussians*3, RTN, serialized (codec.py:214-216)
    x = oracle.gaussians(20240501, oracle.DOMAIN_GAUSS, 0, 5 * 67).reshape(5, 67) * 3.0
    c, s = oracle.quantize_rtn(x, 32)
    blob = oracle.serialize(c, s)
    with open(os.path.join(golden_dir, "golden.mxf4"), "rb") as f:
        assert blob == f.read()


def test_diagnostics_gaussian_stream_matches_reference(golden_dir):
    """The host sample stream of the GPU diagnostics is rng.gaussians itself (rng.py:65-69)."""
    from paper_2505_14669_b200 import diagnostics

    g = _load(golden_dir, "rng.npz")["gauss"]
    assert np.array_equal(diagnostics.gaussians(1, 0x4755, 0, 1000), g)
