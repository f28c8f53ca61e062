set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant_tc -s 2 -c 1 -o gpurun_out/src_tc python tools/prof_fused.py 4096 > gpurun_out/src_tc.log 2>&1
tail -3 gpurun_out/src_tc.log
python -m pytest -q -m gpu tests/test_gpu_dp_llama.py tests/test_gpu_qlinear.py tests/test_gpu_quant.py -x > gpurun_out/tc2_tests.log 2>&1; tail -3 gpurun_out/tc2_tests.log
python bench.py --steps 10 --warmup 3 > gpurun_out/tc2_bench.json 2>gpurun_out/tc2_bench.err; python -c "import json;d=json.loads(open('gpurun_out/tc2_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['sr_backward'])"
