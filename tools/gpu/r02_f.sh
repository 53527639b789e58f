# k_m4rm timing experiments: normal, no rebuilds (1), no in-stage barriers (2), both (3).
mkdir -p gpurun_out
for d in 0 1 2 3; do
  GF2_M4RM_DBG=$d timeout 300 python tools/m4rm_time.py > gpurun_out/f_time_$d.jsonl 2>&1
  echo "dbg=$d"; cut -c1-140 gpurun_out/f_time_$d.jsonl
done
