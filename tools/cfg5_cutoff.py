"""cfg5 addmul at a given cutoff, digest-checked (exercises K-chunked FP4
leaves with the fused post-addition when cutoff >= 16384)."""
import json, sys, time, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
torch.cuda.set_device(0)
cutoff = int(sys.argv[1])
n = 65536
a, b, c = g.random(n, n, 51), g.random(n, n, 52), g.random(n, n, 53)
torch.cuda.synchronize()
t0 = time.perf_counter()
g.addmul(c, a, b, g.MulParams(cutoff=cutoff, k=8))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
want = json.load(open("tests/golden/digests.json"))["cfg5_addmul"]
print(f"cutoff {cutoff}: {dt*1e3:.1f} ms (first call, incl. workspace), digest ok: {O.digest(c.to_numpy()) == want}")
