for o in 0 1000 0 1000; do
  echo "== order=$o"; GF2_F4_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('ms',round(d['ms_per_step'],4),'kern',round(d['roofline']['kernel_ms_per_step'],4),'ok',d['verified_sha256'])"
  GF2_F4_ORDER=$o timeout 300 python tools/small_profile.py 2>&1 | grep -E "^cfg[24] mul_strassen|k_umma"
done
