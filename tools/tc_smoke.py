"""Minimal tensor-core engine smoke (debug aid): small products against the
oracle, then (optionally) the 16384^3 Strassen step time."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
torch.cuda.set_device(0)
engines = [a for a in sys.argv[1:] if not a.startswith("--")] or ["tc-i8", "tc-f8"]
for eng in engines:
    g.set_engine(eng)
    for (m, l, n) in [(256, 256, 224), (128, 128, 256), (128, 256, 256), (300, 500, 700), (1024, 1024, 1024),
                      (512, 4096, 4096)]:
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
    if "--time" in sys.argv:
        a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
        for _ in range(3):
            c = g.mul_strassen(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            c = g.mul_strassen(a, b)
        e1.record()
        torch.cuda.synchronize()
        print(eng, "16384^3 strassen ms", e0.elapsed_time(e1) / 10,
              "digest", O.digest(c.to_numpy()), flush=True)
