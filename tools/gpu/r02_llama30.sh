set -x
python tools/prof_llama.py 30m > gpurun_out/prof30.txt 2>&1; head -60 gpurun_out/prof30.txt | cut -c1-220
