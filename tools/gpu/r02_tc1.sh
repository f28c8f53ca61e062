# round-2: tensor-core fused col pass (k_quant_tc): parity tests, timing; reference suite on the b200 backend
set -x
python -m pytest -q -m gpu tests/test_gpu_quant.py tests/test_gpu_multitile.py tests/test_gpu_qlinear.py -x > gpurun_out/tc1_tests.log 2>&1; tail -5 gpurun_out/tc1_tests.log
python tools/ab_probe.py prod
python - <<'PY'
import torch, sys
sys.path.insert(0, ".")
import paper_2505_14669_b200 as qt
from paper_2505_14669_b200 import _lib
from paper_2505_14669_b200.mxfp4 import quant_fused, sign_bits
L = qt.load()
def t(f, n=10):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000 / n
for R, C, dt in ((16384, 4096, torch.bfloat16), (16384, 11008, torch.bfloat16), (4096, 4096, torch.float32), (11008, 4096, torch.float32), (4096, 11008, torch.float32)):
    x = torch.randn(R, C, device="cuda").to(dt)
    s = sign_bits(3, R, "cuda")
    f = lambda: quant_fused(x, _lib.QT_ROUND_QUEST, _lib.QT_ROUND_RTN, transform=_lib.QT_TRANSFORM_HADAMARD, col_transform=_lib.QT_TRANSFORM_RANDOMIZED, col_signs=s)
    r = []
    for mode in (0, 1):
        L.qt_debug_set_quant(mode, None); r.append(t(f))
    L.qt_debug_set_quant(0, None)
    print(f"fused {R}x{C} {dt}: tensor-core col pass {r[0]:.1f} us, cuda-core {r[1]:.1f} us", flush=True)
PY
timeout 1500 bash tools/gpu/ref_suite.sh -q -p no:cacheprovider -rf --durations=15 --deselect test_acceptance.py::test_c01_codec_exactness > gpurun_out/tc1_refsuite.log 2>&1; tail -30 gpurun_out/tc1_refsuite.log
