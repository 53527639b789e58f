# Round-2 final build: default bench line, M4RM-engine line, launch list of the default bench, ncu of the top kernel.
mkdir -p gpurun_out/final
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --engine m4rm --extra none --no-cpu-baseline > gpurun_out/final/bench_m4rm.json 2>/dev/null; echo "bench m4rm rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 1 --extra none --no-cpu-baseline --no-e2e > gpurun_out/final/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_umma_f4 -c 1 -o gpurun_out/final/f4 python tools/strassen_once.py 16384 8192 1 > /dev/null 2>&1; echo "ncu f4 rc=$?"
