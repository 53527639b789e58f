# Full GPU tests + small-call profile + configs on the current build.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/k_pytest.log
tail -4 gpurun_out/k_pytest.log
timeout 300 python tools/small_profile.py > gpurun_out/k_small.txt 2>&1; grep -v Warn gpurun_out/k_small.txt | grep -v _warn | head -60
timeout 600 python tools/bench_configs.py > gpurun_out/k_configs.jsonl 2> gpurun_out/k_configs.err; cut -c1-200 gpurun_out/k_configs.jsonl
timeout 300 python tools/m4rm_time.py > gpurun_out/k_m4rm_time.jsonl 2>&1; cut -c1-200 gpurun_out/k_m4rm_time.jsonl
