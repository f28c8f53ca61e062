set -x
python -m pytest -q -m gpu tests/test_gpu_diagnostics.py tests/test_gpu_quant.py tests/test_gpu_multitile.py > gpurun_out/srf_tests.log 2>&1; tail -4 gpurun_out/srf_tests.log
python tools/ab_probe.py prod
python bench.py --steps 10 --warmup 3 > gpurun_out/srf_bench.json 2>gpurun_out/srf_bench.err; python -c "import json;d=json.loads(open('gpurun_out/srf_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['sr_backward']['ms_per_step'],d['sr_fast_backward']['ms_per_step'])"
