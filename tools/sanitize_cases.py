"""Small cases touching every kernel, for compute-sanitizer runs."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
torch.cuda.set_device(0)
ok = True
for eng in ["m4rm", "tc-i8", "tc-f8"]:
    g.set_engine(eng)
    for (m, l, n) in [(1, 1, 1), (70, 130, 65), (300, 700, 260), (513, 1025, 600)]:
        a, b = g.random(m, l, 1), g.random(l, n, 2)
        want = O.naive_product(O.random(m, l, 1), O.random(l, n, 2)).words
        for c in (g.mul_direct(a, b), g.mul_m4rm(a, b, 8), g.mul_strassen(a, b, g.MulParams(cutoff=64))):
            ok &= bool(np.array_equal(c.to_numpy(), want))
    pa, pb = g.random(90, 640, 77), g.random(700, 512, 78)
    aw, bw = g.window(pa, 5, 64, 70, 385), g.window(pb, 11, 192, 385, 250)
    pc = g.random(80, 512, 79)
    g.addmul(g.window(pc, 3, 64, 70, 250), aw, bw, g.MulParams(cutoff=64))
    c0 = g.random(5, 70000, 3)
    g.mul_m4rm_into(c0, g.random(5, 64, 4), g.random(64, 70000, 5), 8)
    c1 = g.random(2, 3, 3)
    g.mul_m4rm_into(c1, g.random(2, 20000, 4), g.random(20000, 3, 5), 8)
x = g.random(100, 300, 9)
g.add_into(g.window(x, 1, 64, 50, 100), g.window(x, 50, 128, 50, 100), g.window(x, 0, 0, 50, 100))
g.bernoulli(33, 777, 4, p=0.1)
torch.cuda.synchronize()
print("sanitize cases ok" if ok else "MISMATCH")
