# round-2 A/B 5: two-team schedule of the tensor-core forward quantizer
set -x
QT_LIB_PATH=exp/teams/libquartet_b200.so python -m pytest -q -m gpu tests/test_gpu_quant.py tests/test_gpu_multitile.py tests/test_gpu_fullsize.py -k "tensor_core or fused or forward" > gpurun_out/ab5_tests.log 2>&1; tail -3 gpurun_out/ab5_tests.log
QT_LIB_PATH=exp/teams/libquartet_b200.so python tools/ab_probe.py teams
python tools/ab_probe.py lockstep
QT_LIB_PATH=exp/teams/libquartet_b200.so python tools/ab_probe.py teams-again
python tools/ab_probe.py lockstep-again
