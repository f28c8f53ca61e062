set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tcq_xq -s 2 -c 1 -o gpurun_out/src_xq python tools/prof_fused.py 4096 > gpurun_out/src_xq.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tcq_dual -s 2 -c 1 -o gpurun_out/src_dual2 python tools/prof_dual.py > gpurun_out/src_dual2.log 2>&1
tail -2 gpurun_out/src_xq.log gpurun_out/src_dual2.log
