# round-2 (late): source-level ncu capture of the tensor-core forward quantizer k_tcq_xq (16384 x 4096 bf16)
set -x
python tools/fwd_probe.py 4096 > gpurun_out/xq_fwdprobe.txt 2>&1; cat gpurun_out/xq_fwdprobe.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tcq_xq -s 2 -c 1 -o gpurun_out/src_xq python tools/prof_fused.py 4096 > gpurun_out/src_xq.log 2>&1
tail -3 gpurun_out/src_xq.log
QT_PROF_QMODE=51 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tcq_xq -s 2 -c 1 -o gpurun_out/src_xqskel python tools/prof_fused.py 4096 > gpurun_out/src_xqskel.log 2>&1
tail -3 gpurun_out/src_xqskel.log
