set -x
python -m pytest -q -m gpu tests > gpurun_out/full4_tests.log 2>&1; tail -5 gpurun_out/full4_tests.log
python __graft_entry__.py > gpurun_out/full4_smoke.log 2>&1; tail -1 gpurun_out/full4_smoke.log
python bench.py > gpurun_out/full4_bench.json 2>gpurun_out/full4_bench.err; python -c "import json;d=json.loads(open('gpurun_out/full4_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['e2e']['value'],d['bf16_cublas']['speedup_ours']);print({k:(v.get('tokens_per_s'),v.get('speedup_vs_bf16'),v.get('launch')) for k,v in d['train'].items() if isinstance(v,dict)})"
