mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:k_combine -c 6 -o gpurun_out/comb5b python tools/cfg5_once.py > gpurun_out/comb5b.log 2>&1
timeout 300 python tools/cfg5_gap.py | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/small_profile.py 2>&1 | grep -E "^cfg2|combine"
