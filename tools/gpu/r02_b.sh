# Round 2, session 2 check: GPU tests on HEAD, smoke, default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/b_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/b_smoke.log
timeout 600 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "bench rc=$?" >> gpurun_out/b_bench.err
timeout 400 python tools/bench_configs.py > gpurun_out/b_configs.jsonl 2> gpurun_out/b_configs.err; echo "rc=$?" >> gpurun_out/b_configs.err
tail -3 gpurun_out/b_pytest.log; tail -2 gpurun_out/*.err gpurun_out/b_smoke.log
