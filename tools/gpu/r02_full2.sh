set -x
python -m pytest -q -m gpu tests > gpurun_out/full2_tests.log 2>&1; tail -5 gpurun_out/full2_tests.log
python __graft_entry__.py > gpurun_out/full2_smoke.log 2>&1; tail -2 gpurun_out/full2_smoke.log
python bench.py > gpurun_out/full2_bench.json 2>gpurun_out/full2_bench.err; python -c "import json;d=json.loads(open('gpurun_out/full2_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['quantizer_roofline'],d['sr_backward'],d['e2e']['value'],d['bf16_cublas']['speedup_ours'])"
