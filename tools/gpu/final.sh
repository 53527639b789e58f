# Round measurement suite: bench line (with the CPU sample), reference arm,
# all five configs, engine crossover, small-config profile, host costs,
# kernel timelines, the bench's ncu launch list and one full ncu capture of
# the GEMM. Everything lands in gpurun_out/ (copied to profiles/ by hand).
set -x
mkdir -p gpurun_out
O=gpurun_out/fin
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref.json 2> $O/ref.err
timeout 600 python bench.py --sharded --no-cpu-baseline > $O/sharded.json 2> $O/sharded.err
timeout 600 python tools/shard_estimate.py > $O/shard_estimate.txt 2>&1
timeout 1500 python tools/bench_configs.py > $O/configs.jsonl 2> $O/configs.err
timeout 300 python tools/engine_cross.py > $O/cross_default.txt 2>&1
GF2_TC_MIN_WORK=1e30 timeout 300 python tools/engine_cross.py > $O/cross_m4rm.txt 2>&1
GF2_TC_MIN_WORK=1 GF2_TC_MIN_LEAF=256 timeout 300 python tools/engine_cross.py > $O/cross_tensor.txt 2>&1
timeout 300 python tools/small_profile.py 2>&1 | grep -v -i warn > $O/small_profile.txt
timeout 300 python tools/host_breakdown.py > $O/host_breakdown.txt 2>&1
timeout 300 python tools/timeline.py --summary > $O/timeline_cfg3.txt 2>&1
timeout 600 python tools/timeline.py --size 65536 --addmul --summary --reps 1 > $O/timeline_cfg5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_umma_f4 -s 2 -c 1 -o $O/f4_bench \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-verify > $O/ncu_full.log 2>&1
cat $O/bench.json
