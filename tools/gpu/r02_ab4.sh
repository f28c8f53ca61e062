# round-2 A/B 4: sleep between polls of the single-thread producer / MMA roles (tcq.cu, tcq_x.cu)
set -x
python -m pytest -q -m gpu tests/test_gpu_quant.py -k "tensor_core" > gpurun_out/ab4_tests.log 2>&1; tail -2 gpurun_out/ab4_tests.log
for v in nosleep sleep512; do QT_LIB_PATH=exp/$v/libquartet_b200.so python tools/ab_probe.py $v; done
python tools/ab_probe.py sleep128
QT_LIB_PATH=exp/nosleep/libquartet_b200.so python tools/ab_probe.py nosleep-again
python tools/ab_probe.py sleep128-again
