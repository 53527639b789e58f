# GPU check after an M4RM / host-path change: GPU tests, small-config
# profile, host breakdown, a short parity fuzz, all configs but cfg5.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b_pytest.log
timeout 300 python tools/small_profile.py > gpurun_out/b_small.txt 2>&1
timeout 300 python tools/host_breakdown.py > gpurun_out/b_host.txt 2>&1
timeout 400 python tools/fuzz.py 240 gpurun_out/b_fuzz.json 2>&1 | tail -c 20000 > gpurun_out/b_fuzz.log
timeout 600 python tools/bench_configs.py --skip-cfg5 > gpurun_out/b_configs.jsonl 2>&1
tail -3 gpurun_out/b_pytest.log; grep -v Warn gpurun_out/b_small.txt; cat gpurun_out/b_host.txt; tail -3 gpurun_out/b_fuzz.log; cat gpurun_out/b_configs.jsonl
