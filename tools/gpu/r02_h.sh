# Measured low-precision peaks; ncu --set full of k_umma_f4 (cfg3 step) on this build; full GPU tests.
mkdir -p gpurun_out
timeout 900 python tools/measure_lowp_peak.py gpurun_out/h_peaks_lowp.json > gpurun_out/h_peaks.log 2>&1; echo "peaks rc=$?" >> gpurun_out/h_peaks.log
tail -30 gpurun_out/h_peaks.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_f4 -c 1 -o gpurun_out/h_f4 python tools/strassen_once.py 16384 8192 1 > gpurun_out/h_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/h_ncu.log
tail -2 gpurun_out/h_ncu.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest.log
tail -3 gpurun_out/h_pytest.log
