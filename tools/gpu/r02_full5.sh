set -x
python -m pytest -q -m gpu tests > gpurun_out/full5_tests.log 2>&1; tail -4 gpurun_out/full5_tests.log
python bench.py > gpurun_out/full5_bench.json 2>gpurun_out/full5_bench.err; python -c "import json;d=json.loads(open('gpurun_out/full5_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['sr_backward']['ms_per_step'],d['sr_fast_backward']['ms_per_step'],d['e2e']['value'],d['bf16_cublas']['speedup_ours'])"
