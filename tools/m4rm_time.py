"""k_m4rm timings on the M4RM engine (tuning aid): 16384^3 mul_m4rm, cfg1
mul_m4rm 1024^3 and cfg4's mul_m4rm_into(C,A,B,8,512,8), each checked
against the config digest, CUDA events, L2 flushed, min and mean of 10."""
import hashlib
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0811_1714_b200 as g  # noqa: E402

torch.cuda.set_device(0)
g.set_engine("m4rm")
dig = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def sha(m):
    return hashlib.sha256(m.to_numpy().astype("<u8").tobytes()).hexdigest()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), sum(ts) / len(ts)


def line(name, m, l, n, ms, ok):
    print(json.dumps({"call": name, "m": m, "l": l, "n": n, "ms_min": ms[0], "ms_mean": ms[1],
                      "bitops_per_s": m * l * n / (ms[0] * 1e-3), "verified_sha256": ok,
                      "lookup_bound_ms": m * l * n / 64 / 37.2e12 * 1e3}), flush=True)


for (name, m, key, sa, sb) in [("mul_m4rm 16384^3", 16384, None, 31, 32), ("cfg1 mul_m4rm 1024^3", 1024, "cfg1", 11, 12)]:
    a, b = g.random(m, m, sa), g.random(m, m, sb)
    out = {}
    ms = timed(lambda: out.__setitem__("c", g.mul_m4rm(a, b, 8)))
    ok = sha(out["c"]) == dig[key] if key else sha(out["c"]) == dig["cfg3"]
    line(name, m, m, m, ms, ok)
    del a, b, out

m, l, n = 10000, 7001, 12345
a = g.bernoulli(m, l, 41, p=0.1)
b = g.bernoulli(l, n, 42, p=0.1)
c0 = g.random(m, n, 43)
c = g.copy_out(c0)
ms = timed(lambda: g.mul_m4rm_into(c, a, b, 8, 512, 8), reps=10)
g.copy_into(c, c0)
g.mul_m4rm_into(c, a, b, 8, 512, 8)
line("cfg4 mul_m4rm_into(C,A,B,8,512,8)", m, l, n, ms, sha(c) == dig.get("cfg4_addmul"))
