for r in 1 2 3; do for o in 0 1000 16; do
  echo -n "order=$o "; GF2_F4_ORDER=$o timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('ms',round(d['ms_per_step'],4),'kern',round(d['roofline']['kernel_ms_per_step'],4),'ok',d['verified_sha256'])"
done; done
for o in 0 1000; do echo "cfg5 order=$o"; GF2_F4_ORDER=$o timeout 300 python tools/cfg5_gap.py | tail -2; done
