# round-2 final evidence: ncu launch list + full capture of one bench step (summaries written on the box),
# the bench line and the reference arm
set -x
mkdir -p gpurun_out/profiles
REP_DIR=/tmp bash tools/ncu_round.sh r02
OUT_DIR=gpurun_out/profiles REP_DIR=/tmp python tools/summarize_ncu.py r02 > gpurun_out/summarize_r02.log 2>&1; tail -3 gpurun_out/summarize_r02.log
cp gpurun_out/launches_r02.csv gpurun_out/profiles/ 2>/dev/null
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 400 gpurun_out/final_bench.json
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; cat gpurun_out/final_ref.json | tail -c 300
