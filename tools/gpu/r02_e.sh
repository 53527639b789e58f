# k_m4rm iteration: parity subset, M4RM timings (16384^3, cfg1, cfg4), ncu of 16384^3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "m4rm or cfg1 or golden or edge or window or triples" > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/e_pytest.log
tail -3 gpurun_out/e_pytest.log
timeout 300 python tools/m4rm_time.py > gpurun_out/e_time.jsonl 2> gpurun_out/e_time.err; echo "rc=$?" >> gpurun_out/e_time.err
cat gpurun_out/e_time.jsonl; tail -3 gpurun_out/e_time.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_m4rm -c 1 -o gpurun_out/e_m4rm python tools/m4rm_once.py > gpurun_out/e_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/e_ncu.log
tail -1 gpurun_out/e_ncu.log
