python tools/prof_llama.py 200m > gpurun_out/prof200.txt 2>&1
