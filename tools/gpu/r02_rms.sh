set -x
python -m pytest -q -m gpu tests/test_gpu_llama.py tests/test_gpu_train_graph.py > gpurun_out/rms_tests.log 2>&1; tail -3 gpurun_out/rms_tests.log
python tools/train_llama.py --preset 30m --batch 64 --steps 5 --warmup 3
python tools/train_llama.py --preset 30m --batch 64 --steps 5 --warmup 3 --linear bf16
