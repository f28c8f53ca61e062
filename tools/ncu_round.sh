#!/bin/bash
# Per-round ncu evidence (run under gpurun on ONE GPU). Outputs into gpurun_out/:
#   launches_<tag>.csv   every kernel launch of one bench step (gpu__time_duration, cold, serialised)
#   full_<tag>.ncu-rep   --set full of every hot-path kernel of one step (GEMMs + quantizers)
set -e
TAG=${1:-r01}
REP=${REP_DIR:-gpurun_out}   # large .ncu-rep files can go elsewhere (gpurun copies back <= 64 MiB)
cd "$(dirname "$0")/.."
# one warm-up step (6 matched launches/shape x 3 shapes: 2 fused forward quantizers, 1 dual, 3 GEMMs) is skipped
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python tools/prof_step.py --all-shapes --iters 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_quant|k_tcq" -s 18 -c 18 \
    -o ${REP}/full_${TAG} python tools/prof_step.py --all-shapes --iters 2 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
