for geom in "" "16,4" "16,5" "16,7" "16,8" "8,4" "8,2"; do
GF2_M4RM_GEOM=$geom python - <<'PY'
import os, sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0); g.set_engine("m4rm")
a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
f = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(2): g.mul_strassen(a, b)
ts = []
for _ in range(5):
    f.zero_(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); g.mul_strassen(a, b); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
print(os.environ.get("GF2_M4RM_GEOM") or "model", round(min(ts), 3))
PY
done
