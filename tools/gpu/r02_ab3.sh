# round-2 A/B 3: warp-cooperative exact fallback in k_tcq_dual, L2 vs sqrt(32) max bound; parity; reference suite counts
set -x
python -m pytest -q -m gpu tests/test_gpu_quant.py tests/test_gpu_multitile.py tests/test_gpu_fullsize.py -k "dual" > gpurun_out/ab3_tests.log 2>&1; tail -3 gpurun_out/ab3_tests.log
QT_LIB_PATH=exp/amax/libquartet_b200.so python -m pytest -q -m gpu tests/test_gpu_quant.py tests/test_gpu_multitile.py tests/test_gpu_fullsize.py -k "dual" > gpurun_out/ab3_tests_amax.log 2>&1; tail -3 gpurun_out/ab3_tests_amax.log
python tools/ab_probe.py prod-l2
QT_LIB_PATH=exp/amax/libquartet_b200.so python tools/ab_probe.py amax
python tools/ab_probe.py prod-l2-again
QT_LIB_PATH=exp/amax/libquartet_b200.so python tools/ab_probe.py amax-again
timeout 1500 bash tools/gpu/ref_suite.sh -q -p no:cacheprovider -rf --deselect test_acceptance.py::test_c01_codec_exactness --junitxml=$GRAFT_REPO_ROOT/gpurun_out/refsuite.xml > gpurun_out/ab3_refsuite.log 2>&1; tail -4 gpurun_out/ab3_refsuite.log
