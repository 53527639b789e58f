# Quick GPU loop after a kernel change: GPU tests, small-config profile,
# cfg3 bench line without the CPU sample.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/q_pytest.log
timeout 300 python tools/small_profile.py 2>&1 | grep -v -i warn > gpurun_out/q_small.txt
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
tail -3 gpurun_out/q_pytest.log; cat gpurun_out/q_small.txt
python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print('BENCH ms',d['ms_per_step'],'frac',d['roofline']['frac'],'kern',d['roofline']['kernel_ms_per_step'],'e2e',d['e2e']['ms_per_step'],'ok',d['verified_sha256'])"
