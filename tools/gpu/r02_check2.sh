# round-2: new GPU tests, the reference's own suite on the b200 backend, bench (SR backward), 2-rank gloo bench
set -x
python -m pytest -q -m gpu tests/test_gpu_named_abi.py -x > gpurun_out/c2_named.log 2>&1; tail -3 gpurun_out/c2_named.log
timeout 1200 bash tools/gpu/ref_suite.sh -x -q -p no:cacheprovider > gpurun_out/c2_refsuite.log 2>&1; tail -15 gpurun_out/c2_refsuite.log
python bench.py --steps 10 --warmup 3 > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; tail -c 600 gpurun_out/c2_bench.json; tail -3 gpurun_out/c2_bench.err
QT_BENCH_ONE_GPU=1 QT_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/c2_bench2.json 2> gpurun_out/c2_bench2.err; python -c "import json;d=json.loads(open('gpurun_out/c2_bench2.json').read().strip().splitlines()[-1]);print(d['value'],d['config']['launch'])"; tail -3 gpurun_out/c2_bench2.err
