# round-2: source-level ncu captures of the three quantizer kernels (dynamic SASS histograms)
set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 2 -c 1 -o gpurun_out/src_fx python tools/prof_fused.py 4096 > gpurun_out/src_fx.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 2 -c 1 -o gpurun_out/src_fw python tools/prof_fused.py 4096 f32 > gpurun_out/src_fw.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tcq_dual -s 2 -c 1 -o gpurun_out/src_dual python tools/prof_dual.py > gpurun_out/src_dual.log 2>&1
ls -la gpurun_out
