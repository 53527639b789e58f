mkdir -p gpurun_out
for w in 1e30 1; do GF2_TC_MIN_WORK=$w timeout 300 python tools/engine_cross.py; done
