# round-2: full GPU suite + bench
set -x
python -m pytest -q -m gpu tests/test_gpu_dp_llama.py > gpurun_out/full_dp.log 2>&1; tail -3 gpurun_out/full_dp.log
python -m pytest -q -m gpu tests > gpurun_out/full_tests.log 2>&1; tail -5 gpurun_out/full_tests.log
python bench.py > gpurun_out/full_bench.json 2>gpurun_out/full_bench.err; python -c "import json;d=json.loads(open('gpurun_out/full_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['sr_backward'],d['e2e']['value'])"
