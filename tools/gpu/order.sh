mkdir -p gpurun_out
for o in 0 1 4 8 32; do
  echo "== GF2_F4_ORDER=$o"
  GF2_F4_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --no-e2e | python -c "import json,sys;d=json.loads(sys.stdin.read());print('ms',round(d['ms_per_step'],4),'kern',round(d['roofline']['kernel_ms_per_step'],4),'ok',d['verified_sha256'])"
  GF2_F4_ORDER=$o timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_umma_f4 -c 1 python tools/strassen_once.py 16384 8192 1 2>&1 | grep -E "dram__|gpu__time"
done
