# build the three trigger variants and time the small configs with each
set -e
for mode in 1 0 2; do
  make -s -C paper_0811_1714_b200/csrc clean >/dev/null
  make -s -j8 -C paper_0811_1714_b200/csrc NVFLAGS_EXTRA=-DGF2_PDL_TRIGGER=$mode >/dev/null 2>&1
  echo "== trigger mode $mode"
  timeout 300 python tools/engine_cross.py
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 20 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bench ms',round(d['ms_per_step'],4),'kern',round(d['roofline']['kernel_ms_per_step'],4),'ok',d['verified_sha256'])"
done
