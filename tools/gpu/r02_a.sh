# Round 2, first GPU pass: GPU tests, the default bench line (cfg3 + cfg5
# extra), cfg5 as the primary workload, and the N=1 NCCL (--sharded) path
# on cfg5 (a world of one: mul_sharded + ShardedHostPipeline with C0 in).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 600 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; echo "bench rc=$?" >> gpurun_out/a_bench.err
timeout 600 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/a_bench_cfg5.json 2> gpurun_out/a_bench_cfg5.err; echo "rc=$?" >> gpurun_out/a_bench_cfg5.err
timeout 600 python bench.py --workload cfg5 --sharded --no-cpu-baseline --steps 5 > gpurun_out/a_bench_cfg5_sh.json 2> gpurun_out/a_bench_cfg5_sh.err; echo "rc=$?" >> gpurun_out/a_bench_cfg5_sh.err
timeout 300 python bench.py --gpus 2 > gpurun_out/a_bench_g2.json 2> gpurun_out/a_bench_g2.err; echo "rc=$?" >> gpurun_out/a_bench_g2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/a_ref.json 2> gpurun_out/a_ref.err; echo "rc=$?" >> gpurun_out/a_ref.err
tail -3 gpurun_out/a_pytest.log; tail -2 gpurun_out/*.err
