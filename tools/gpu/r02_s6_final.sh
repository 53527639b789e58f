# Round 2, session 6 final build: GPU suite, both bench arms, launch list of the default bench, ncu of the top kernel.
mkdir -p gpurun_out/final6
python -m pytest tests -m gpu -x -q > gpurun_out/final6/gputest.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/final6/gputest.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final6/ref.json 2> gpurun_out/final6/ref.err; echo "ref arm rc=$?"
timeout 900 python bench.py > gpurun_out/final6/bench.json 2> gpurun_out/final6/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --engine m4rm --extra none --no-cpu-baseline > gpurun_out/final6/bench_m4rm.json 2>/dev/null; echo "bench m4rm rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final6/launches.csv python bench.py --steps 2 --warmup 1 --extra none --no-cpu-baseline --no-e2e > gpurun_out/final6/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_f4 -c 1 -o gpurun_out/final6/f4 python tools/strassen_once.py 16384 8192 1 > /dev/null 2>&1; echo "ncu f4 rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final6/smoke.log
