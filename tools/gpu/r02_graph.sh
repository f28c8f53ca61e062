set -x
python -m pytest -q -m gpu tests/test_gpu_train_graph.py tests/test_gpu_nonfinite.py tests/test_gpu_llama.py -x > gpurun_out/graph_tests.log 2>&1; tail -5 gpurun_out/graph_tests.log
python tools/train_llama.py --preset 30m --batch 64 --steps 5 --warmup 3
python tools/train_llama.py --preset 30m --batch 64 --steps 5 --warmup 3 --linear bf16
python tools/train_llama.py --preset 200m --batch 64 --steps 5 --warmup 3
python tools/train_llama.py --preset 200m --batch 64 --steps 5 --warmup 3 --linear bf16
