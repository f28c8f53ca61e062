set -x
python -m pytest -q -m gpu tests/test_gpu_diagnostics.py tests/test_gpu_quant.py -k "sr_fast or tensor_core" > gpurun_out/srf2_tests.log 2>&1; tail -2 gpurun_out/srf2_tests.log
python tools/ab_probe.py prod
python tools/ab_probe.py prod-again
