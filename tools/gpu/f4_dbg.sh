mkdir -p gpurun_out
for d in 0 1 2; do echo "== GF2_F4_DBG=$d"; GF2_F4_DBG=$d timeout 300 python tools/small_profile.py 2>&1 | grep -E "^cfg|k_umma_f4"; done
