# New k_m4rm (BM 4096 x 256 columns, interleaved tables): parity, timing, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engines.py tests/test_gpu_api.py -q -x > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d_pytest.log
tail -5 gpurun_out/d_pytest.log
timeout 600 python tools/bench_configs.py --engine m4rm > gpurun_out/d_configs_m4rm.jsonl 2> gpurun_out/d_configs.err; echo "rc=$?" >> gpurun_out/d_configs.err
cat gpurun_out/d_configs_m4rm.jsonl | cut -c1-220
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_m4rm -c 1 -o gpurun_out/d_m4rm python tools/m4rm_once.py > gpurun_out/d_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/d_ncu.log
tail -3 gpurun_out/d_ncu.log
