# TMEM-parked k_m4rm (BM 8192): full GPU tests, fuzz, M4RM timings, ncu.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/m_pytest.log
tail -3 gpurun_out/m_pytest.log
timeout 420 python tools/fuzz.py 300 gpurun_out/m_fuzz.json > gpurun_out/m_fuzz.log 2>&1; echo "fuzz rc=$?" >> gpurun_out/m_fuzz.log
tail -2 gpurun_out/m_fuzz.log
timeout 300 python tools/m4rm_time.py > gpurun_out/m_time.jsonl 2>&1; cut -c1-160 gpurun_out/m_time.jsonl
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_m4rm -c 1 -o gpurun_out/m_m4rm python tools/m4rm_once.py > gpurun_out/m_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/m_ncu.log
tail -1 gpurun_out/m_ncu.log
