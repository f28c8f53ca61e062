# round-2: tensor-core forward quantizer with warp-cooperative fallbacks; dual with the new default bound
set -x
python -m pytest -q -m gpu tests/test_gpu_quant.py -k "tensor_core" > gpurun_out/xq_tests.log 2>&1; tail -3 gpurun_out/xq_tests.log
python tools/fwd_probe.py 4096
python tools/fwd_probe.py 11008
python tools/ab_probe.py prod
