# refreshed ncu evidence for the final round-2 kernels (launch list + full-set summary of one step)
mkdir -p gpurun_out/profiles
REP_DIR=/tmp bash tools/ncu_round.sh r02 > gpurun_out/ncu_round_r02.log 2>&1; tail -2 gpurun_out/ncu_round_r02.log
OUT_DIR=gpurun_out/profiles REP_DIR=/tmp python tools/summarize_ncu.py r02 > gpurun_out/summarize_r02.log 2>&1; tail -3 gpurun_out/summarize_r02.log
cp gpurun_out/launches_r02.csv gpurun_out/profiles/ 2>/dev/null
ls gpurun_out/profiles
