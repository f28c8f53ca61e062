set -x
python -m pytest -q -m gpu tests > gpurun_out/full9_tests.log 2>&1; tail -3 gpurun_out/full9_tests.log
python __graft_entry__.py > gpurun_out/full9_smoke.log 2>&1; tail -1 gpurun_out/full9_smoke.log
python bench.py > gpurun_out/full9_bench.json 2>gpurun_out/full9_bench.err; head -c 1500 gpurun_out/full9_bench.json; echo; python -c "import json;d=json.loads(open('gpurun_out/full9_bench.json').read().strip().splitlines()[-1]);print({k:(v.get('tokens_per_s'),v.get('speedup_vs_bf16')) for k,v in d['train'].items() if isinstance(v,dict)})"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02b.csv python tools/prof_step.py --all-shapes --iters 2 > /dev/null 2>&1
grep -c "k_zero_tiles" gpurun_out/launches_r02b.csv
