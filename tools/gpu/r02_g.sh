# Full GPU tests + 5-minute parity fuzz on the new k_m4rm + default bench line.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g_pytest.log
tail -4 gpurun_out/g_pytest.log
timeout 420 python tools/fuzz.py 300 gpurun_out/g_fuzz.json > gpurun_out/g_fuzz.log 2>&1; echo "fuzz rc=$?" >> gpurun_out/g_fuzz.log
tail -3 gpurun_out/g_fuzz.log
timeout 600 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo "bench rc=$?" >> gpurun_out/g_bench.err
tail -1 gpurun_out/g_bench.err; cut -c1-300 gpurun_out/g_bench.json
