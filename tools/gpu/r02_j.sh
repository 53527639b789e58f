# ncu of the cfg2 (cutoff 1024) GEMM; engine tests; cfg2 probe on the new default.
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_f4 -c 1 -o gpurun_out/j_f4_cfg2 python tools/strassen_once.py 4096 1024 1 > gpurun_out/j_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/j_ncu.log
tail -1 gpurun_out/j_ncu.log
KERNELS=1 python tools/cfg2_probe.py "" "GF2_F4_DBG=2" "GF2_F4_DBG=1"
timeout 1200 python -m pytest tests/test_gpu_engines.py tests/test_gpu_parity.py -q -x > gpurun_out/j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j_pytest.log
tail -3 gpurun_out/j_pytest.log
