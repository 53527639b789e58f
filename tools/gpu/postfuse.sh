mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_engines.py -m gpu -x -q -k "unfused or cfg2 or recursion" 2>&1 | tail -3
for k in 0 1025 2049 4097; do echo "== GF2_POST_FUSE_MIN_K=$k"; GF2_POST_FUSE_MIN_K=$k timeout 300 python tools/engine_cross.py | grep -E '"cutoff": [1-9]'; done
