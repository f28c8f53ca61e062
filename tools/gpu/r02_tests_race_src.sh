# round-2 GPU session: full GPU suite, racecheck on the grid-capped multi-tile tests, ncu source captures
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/t1.log 2>&1; tail -3 gpurun_out/t1.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python -m pytest -q -m gpu "tests/test_gpu_multitile.py::test_forward_fused_multitile" "tests/test_gpu_multitile.py::test_dual_multitile" "tests/test_gpu_multitile.py::test_requant_multitile" -k "grid3" > gpurun_out/race_mt.log 2>&1; tail -5 gpurun_out/race_mt.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tcq_dual -s 2 -c 1 -o gpurun_out/dual_src python tools/prof_dual.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_quant -s 2 -c 1 -o gpurun_out/fusedx_src python tools/prof_fused.py > /dev/null 2>&1
ls -la gpurun_out
