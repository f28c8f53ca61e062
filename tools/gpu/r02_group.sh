# group path (first member fused) : tests + Llama step times
timeout 900 python -m pytest tests/test_gpu_qlinear.py tests/test_gpu_llama.py tests/test_gpu_train_graph.py tests/test_gpu_nonfinite.py tests/test_gpu_dp_llama.py -x -q > gpurun_out/group_tests.log 2>&1
tail -3 gpurun_out/group_tests.log
for p in 200m 30m; do timeout 300 python tools/train_llama.py --preset $p --steps 10 --warmup 3 >> gpurun_out/group_llama.txt 2>&1; done
timeout 300 python tools/train_llama.py --preset 7b --block --batch 4 --steps 5 --warmup 3 >> gpurun_out/group_llama.txt 2>&1
cat gpurun_out/group_llama.txt | cut -c1-400
