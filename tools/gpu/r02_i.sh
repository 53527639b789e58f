# New GPU tests (reference binding, CLI), peaks rerun (cuBLAS MXFP4), default bench line with the measured-peak roofline.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_reference_binding.py tests/test_gpu_cli.py -q > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i_pytest.log
tail -25 gpurun_out/i_pytest.log
timeout 900 python tools/measure_lowp_peak.py gpurun_out/i_peaks_lowp.json > gpurun_out/i_peaks.log 2>&1; echo "peaks rc=$?" >> gpurun_out/i_peaks.log
grep -A8 mxf4_8192 gpurun_out/i_peaks.log | head -10; tail -8 gpurun_out/i_peaks.log
timeout 600 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; echo "bench rc=$?" >> gpurun_out/i_bench.err
tail -1 gpurun_out/i_bench.err
