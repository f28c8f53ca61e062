"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch dir under /tmp, builds the reference's Cython
backend there (python setup.py build_ext --inplace; numpy backend if that fails -- the
reference asserts both are bit-identical, tests/test_backends.py), imports ``mx4train`` from
that scratch copy and records inputs and outputs of the hot-path functions:

* rng.npz           derive_seed / signs / uniform_at        (rng.py:27-78)
* kernels.npz       quantize_rtn / quantize_sr / quantize_quest on the reference's own
                    adversarial inputs (test_backends.py:18-30) plus bf16-valued and
                    heavy-tailed matrices                    (_native.pyx:104-245)
* fwht.npz          fwht f32/f64 for g in {2,16,32,256}      (_native.pyx:353-379)
* gemm.npz          gemm_nt f32/f64                          (_native.pyx:382-396)
* qlinear_*.npz     qlinear.forward / backward end to end    (qlinear.py:114-252)
* golden.mxf4       serialize(_golden_tensor())              (selftest.py:63-83, codec.py:214-216)

Nothing under tests/ reads /root/reference at test time; only these committed files.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
SCRATCH = "/tmp/quartet_golden_ref"


def _import_reference():
    if not os.path.isdir(SCRATCH):
        shutil.copytree(REF, SCRATCH)
        r = subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                           capture_output=True, text=True)
        if r.returncode != 0:
            print("native build failed; using the numpy backend", file=sys.stderr)
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    import mx4train  # noqa: F401
    from mx4train._backend import BACKEND

    print("reference backend:", BACKEND)
    return mx4train


def bf16_values(a: np.ndarray) -> np.ndarray:
    """Round f32 to bf16 (RNE) and return as f32 -- the values the B200 path consumes."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32)


def kernel_inputs():
    r = np.random.default_rng(0)
    # test_backends.py:18-30 verbatim inputs
    out = [
        np.ascontiguousarray(r.normal(size=(7, 97))),
        np.ascontiguousarray(r.normal(size=(3, 32)) * 1e-6),
        np.ascontiguousarray(r.normal(size=(2, 64)) * 1e6),
        np.ascontiguousarray(r.standard_t(df=2, size=(5, 160))),
    ]
    x = np.zeros((2, 40))
    x[0, 0] = 6.0
    out.append(x)
    out.append(np.ascontiguousarray(
        np.array([[0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0, -0.75, -2.5, -0.0] + [6.0] * 22])))
    # B200-path shapes: f32 values (bf16-representable and not), multiples of 32
    r2 = np.random.default_rng(1)
    out.append(bf16_values(r2.normal(size=(64, 256)).astype(np.float32)).astype(np.float64))
    out.append(r2.standard_t(df=3, size=(32, 128)).astype(np.float32).astype(np.float64))
    out.append(bf16_values(r2.standard_t(df=1.5, size=(32, 128)).astype(np.float32)).astype(np.float64))
    g = r2.normal(size=(16, 256)).astype(np.float32)
    g[:, 5] *= 100.0  # outlier channel
    out.append(g.astype(np.float64))
    # huge / tiny dynamic range inside one group, exact grid points at several scales
    h = np.zeros((4, 64))
    h[0, :32] = np.ldexp(1.0, np.arange(-40, 24, 2))[:32]
    h[1, :] = np.tile([6.0, 3.0, -1.5, 0.5], 16) * 2.0 ** 10
    h[2, :] = np.tile([1.0, -1.0], 32)
    h[3, 0] = 1.5 * 2.0 ** -3
    out.append(h)
    return out


def main():
    ref = _import_reference()
    from mx4train import codec, qlinear, rng, selftest
    from mx4train._backend import kernels
    from mx4train.quantizers import QUEST, RTN_ABSMAX, SR_ABSMAX

    # ------------------------------------------------------------------ rng
    seeds = [0, 1, 7, 123456789, 2**63 + 5, 2**64 - 1]
    derive = {}
    rows = []
    for s in seeds:
        for tag in (21, 22, 23, 24):
            rows.append((s, tag, rng.derive_seed(s, tag)))
    np.savez_compressed(
        os.path.join(HERE, "rng.npz"),
        derive=np.array(rows, dtype=np.uint64),
        derive3=np.array([rng.derive_seed(3, 4, 5)], dtype=np.uint64),
        signs_7=rng.signs(7, 0, 4096),
        signs_big=rng.signs(2**64 - 1, 100, 333),
        uniform_sr=rng.uniform(1234, rng.DOMAIN_SR, 17, 1000),
        gauss=rng.gaussians(1, rng.DOMAIN_GAUSS, 0, 1000),
    )
    del derive

    # -------------------------------------------------------------- kernels
    store = {}
    for i, x in enumerate(kernel_inputs()):
        store[f"x{i}"] = x
        c, s = kernels.quantize_rtn(x, 32)
        store[f"rtn_codes{i}"], store[f"rtn_scales{i}"] = c, s
        c, s = kernels.quantize_sr(x, 32, 1234 + i, 17)
        store[f"sr_codes{i}"], store[f"sr_scales{i}"] = c, s
        c, s, m = kernels.quantize_quest(x, 32, 1.0 / 16.0)
        store[f"quest_codes{i}"], store[f"quest_scales{i}"], store[f"quest_mask{i}"] = c, s, m
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), n=len(kernel_inputs()), **store)

    # ----------------------------------------------------------------- fwht
    store = {}
    for g in (2, 16, 32, 256):
        for dt in (np.float32, np.float64):
            r = np.random.default_rng(g)
            x = np.ascontiguousarray(r.normal(size=(5, 2 * g)).astype(dt))
            key = f"g{g}_{np.dtype(dt).name}"
            store["x_" + key] = x
            store["y_" + key] = kernels.fwht(x, g)
    np.savez_compressed(os.path.join(HERE, "fwht.npz"), **store)

    # ----------------------------------------------------------------- gemm
    store = {}
    for dt in (np.float32, np.float64):
        r = np.random.default_rng(1)
        a = np.ascontiguousarray(r.normal(size=(13, 96)).astype(dt))
        b = np.ascontiguousarray(r.normal(size=(9, 96)).astype(dt))
        name = np.dtype(dt).name
        store["a_" + name], store["b_" + name], store["c_" + name] = a, b, kernels.gemm_nt(a, b)
    np.savez_compressed(os.path.join(HERE, "gemm.npz"), **store)

    # -------------------------------------------------------------- qlinear
    cases = [
        # name, T, d_in, d_out, scheme, hadamard, rounding, xi[, forward seed (sr_absmax, qlinear.py:148-154)]
        ("quest_rtn", 64, 128, 96, QUEST, True, "rtn", 7),
        ("quest_sr", 64, 128, 96, QUEST, True, "sr", 7),
        ("quest_rtn_t256", 256, 128, 96, QUEST, True, "rtn", 11),
        ("rtnfwd_rtn", 64, 64, 64, RTN_ABSMAX, True, "rtn", 3),
        ("quest_rtn_noh", 64, 64, 96, QUEST, False, "rtn", 5),
        ("srfwd_sr", 64, 128, 96, SR_ABSMAX, True, "sr", 13, 99),
        ("srfwd_rtn_t256", 256, 96, 128, SR_ABSMAX, True, "rtn", 17, 2**64 - 3),
        # hadamard=False accepts ragged batch / d_out: ragged trailing groups in G, W_t, G_t, X_t
        ("quest_rtn_noh_ragged", 201, 64, 77, QUEST, False, "rtn", 5),
        ("quest_sr_noh_ragged", 72, 96, 40, QUEST, False, "sr", 9),
        ("rtnfwd_sr_noh_ragged", 45, 64, 33, RTN_ABSMAX, False, "sr", 21),
    ]
    for name, T, d_in, d_out, scheme, had, rounding, xi, *fseed in cases:
        if os.environ.get("GOLDEN_ONLY") and name not in os.environ["GOLDEN_ONLY"].split(","):
            continue
        seed = fseed[0] if fseed else None
        r = np.random.default_rng(zlib.crc32(name.encode()))
        x = bf16_values(r.normal(size=(T, d_in)).astype(np.float32))
        w = bf16_values((r.normal(size=(d_out, d_in)) / np.sqrt(d_in)).astype(np.float32))
        dy = bf16_values(r.normal(size=(T, d_out)).astype(np.float32))
        y, ctx = qlinear.forward(x, w, scheme=scheme, hadamard=had, seed=seed)
        dx, dw = qlinear.backward(dy, ctx, xi=xi, rounding=rounding)
        extra = {} if seed is None else {"seed": np.uint64(seed)}
        np.savez_compressed(
            os.path.join(HERE, f"qlinear_{name}.npz"), **extra,
            x=x, w=w, dy=dy, xi=np.uint64(xi), scheme=scheme.kind, hadamard=had,
            rounding=rounding, y=y, dx=dx, dw=dw,
            x_codes=ctx.x_q.codes, x_scales=ctx.x_q.scales,
            w_codes=ctx.w_q.codes, w_scales=ctx.w_q.scales,
            m_x=ctx.m_x, m_w=ctx.m_w,
        )

    # ------------------------------------------------------- MXF4 golden blob
    blob = codec.serialize(selftest._golden_tensor())
    with open(os.path.join(HERE, "golden.mxf4"), "wb") as f:
        f.write(blob)
    print("wrote fixtures to", HERE, "reference at", ref.__file__)


if __name__ == "__main__":
    main()
