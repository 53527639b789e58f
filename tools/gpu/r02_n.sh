# k_m4rm_tm<NG> (NG = 2,3,4): parity, M4RM timings, engine configs, leaves at cutoff 4096.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "m4rm or cfg1 or golden or edge or window or triples" 2>&1 | tail -2
timeout 300 python tools/m4rm_time.py 2>&1 | cut -c1-150
GF2_M4RM_VERBOSE=1 timeout 300 python tools/bench_configs.py --engine m4rm 2>&1 | grep -v Warn | sort | uniq | cut -c1-170
