# Parity fuzzers after a kernel change (bounded logs).
mkdir -p gpurun_out
T=${1:-180}
timeout $((T+200)) python tools/fuzz.py $T gpurun_out/z_fuzz.json 2>&1 | tail -c 4000 > gpurun_out/z_fuzz.log
timeout $((T+300)) python tools/fuzz.py $T gpurun_out/z_fuzz_big.json --big 2>&1 | tail -c 4000 > gpurun_out/z_fuzz_big.log
timeout $((T+200)) python tools/fuzz_ops.py 60 gpurun_out/z_fuzz_ops.json 2>&1 | tail -c 4000 > gpurun_out/z_fuzz_ops.log
for f in gpurun_out/z_fuzz.log gpurun_out/z_fuzz_big.log gpurun_out/z_fuzz_ops.log; do tail -n 2 $f; done
