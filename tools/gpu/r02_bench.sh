# round-2 GPU session: GPU suite + bench line + reference arm
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/r02_t.log 2>&1; tail -3 gpurun_out/r02_t.log
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; tail -c 3000 gpurun_out/r02_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_ref.json 2>gpurun_out/r02_ref.err; cat gpurun_out/r02_ref.json
