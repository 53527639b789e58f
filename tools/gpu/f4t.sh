set -e
for w in 16 8; do
  make -s -C paper_0811_1714_b200/csrc clean >/dev/null
  make -s -j8 -C paper_0811_1714_b200/csrc NVFLAGS_EXTRA=-DGF2_F4T_WORDS=$w >/dev/null 2>&1
  echo "== F4T_WORDS=$w"
  for i in 1 2; do timeout 300 python tools/small_profile.py 2>&1 | grep -E "^cfg[24] mul_strassen|^cfg2 mul_strassen default|expand4_cols"; done
  timeout 600 python -m pytest tests -m gpu -x -q -k "engines or configs or cfg4" 2>&1 | tail -1
done
