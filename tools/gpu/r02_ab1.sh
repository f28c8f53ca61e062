# round-2 A/B 1: mbarrier wait mode x checked-RTN bound; plus the new seam / diagnostics GPU tests
set -x
python -m pytest -q -m gpu tests/test_gpu_kernels_backend.py tests/test_gpu_diagnostics.py -x > gpurun_out/ab1_tests.log 2>&1; tail -3 gpurun_out/ab1_tests.log
for v in v0 v1 v2; do QT_LIB_PATH=exp/$v/libquartet_b200.so python tools/ab_probe.py $v; done
python tools/ab_probe.py prod
for v in v0 prod; do QT_LIB_PATH=$( [ $v = prod ] && echo "" || echo exp/$v/libquartet_b200.so ) python tools/ab_probe.py $v-again; done
