# Long parity run on the final build: fuzzers + repetition stress (bounded logs).
mkdir -p gpurun_out/lf
timeout ${FT:-900} python tools/fuzz.py ${FS:-600} gpurun_out/lf/fuzz.json 2>&1 | tail -c 4000 > gpurun_out/lf/fuzz.log
timeout ${FT2:-1000} python tools/fuzz.py ${FS2:-600} gpurun_out/lf/fuzz_big.json --big 2>&1 | tail -c 4000 > gpurun_out/lf/fuzz_big.log
timeout 400 python tools/fuzz_ops.py 120 gpurun_out/lf/fuzz_ops.json 2>&1 | tail -c 4000 > gpurun_out/lf/fuzz_ops.log
timeout 900 python tools/stress.py 150 > gpurun_out/lf/stress.log 2>&1
for f in gpurun_out/lf/*.log; do echo "== $f"; tail -n 2 $f; done
