# Full GPU tests, 5-min fuzz, default bench, configs on the leaf-depth-rule build.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l_pytest.log
tail -4 gpurun_out/l_pytest.log
timeout 420 python tools/fuzz.py 300 gpurun_out/l_fuzz.json > gpurun_out/l_fuzz.log 2>&1; echo "fuzz rc=$?" >> gpurun_out/l_fuzz.log
tail -2 gpurun_out/l_fuzz.log
timeout 600 python bench.py > gpurun_out/l_bench.json 2> gpurun_out/l_bench.err; echo "bench rc=$?" >> gpurun_out/l_bench.err
tail -1 gpurun_out/l_bench.err
timeout 600 python tools/bench_configs.py > gpurun_out/l_configs.jsonl 2> gpurun_out/l_configs.err; cut -c1-180 gpurun_out/l_configs.jsonl
