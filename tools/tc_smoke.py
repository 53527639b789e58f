"""Minimal tensor-core engine smoke (debug aid)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
torch.cuda.set_device(0)
for eng in sys.argv[1:] or ["tc-i8", "tc-f8"]:
    g.set_engine(eng)
    for (m, l, n) in [(128, 128, 256), (128, 256, 256), (300, 500, 700), (1024, 1024, 1024)]:
        a, b = g.random(m, l, 1), g.random(l, n, 2)
        c = g.mul_direct(a, b)
        torch.cuda.synchronize()
        want = O.naive_product(O.random(m, l, 1), O.random(l, n, 2)).words
        got = c.to_numpy()
        ok = np.array_equal(got, want)
        print(eng, (m, l, n), "OK" if ok else "MISMATCH", flush=True)
        if not ok:
            d = O.unpack(O.HostMat(m, n, got)) ^ O.unpack(O.HostMat(m, n, want))
            print("  diff frac", d.mean(), "first", np.argwhere(d)[:5].tolist(), flush=True)
