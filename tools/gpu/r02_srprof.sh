# source-level ncu capture of the exact-SR dual (CUDA-core k_quant)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 2 -c 1 -o gpurun_out/src_dsr python tools/prof_dual_sr.py > gpurun_out/src_dsr.log 2>&1
ncu -i gpurun_out/src_dsr.ncu-rep --page source --csv --print-source sass > gpurun_out/src_dsr.csv 2>/dev/null
ncu -i gpurun_out/src_dsr.ncu-rep --page details --csv > gpurun_out/src_dsr_details.csv 2>/dev/null
python tools/sass_hist.py gpurun_out/src_dsr.csv 67108864 | head -25
python tools/sass_stalls.py gpurun_out/src_dsr.csv | head -16
grep -i "Duration\|Registers Per\|Issue Slots Busy\|Local Memory\|Achieved Occupancy\|Theoretical Occupancy" gpurun_out/src_dsr_details.csv | head -12
