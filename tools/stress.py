"""Stress test (race detector by repetition): repeat products many times and
compare every result on the device with the first one (itself checked
against the reference digest / C port). Reports mismatch counts."""
import json, sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
from oracle import gf2_port as P
torch.cuda.set_device(0)
P.set_threads(P.max_threads())
dig = json.load(open("tests/golden/digests.json"))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
res = {}

def stress(name, fn, want_words=None, want_digest=None):
    first = fn()
    w = first.to_numpy()
    ok0 = (O.digest(w) == want_digest) if want_digest else bool((w == want_words).all())
    ref = first.storage.clone()
    bad = 0
    for _ in range(reps):
        c = fn()
        bad += int(not torch.equal(c.storage, ref))
    torch.cuda.synchronize()
    res[name] = {"first_correct": ok0, "reps": reps, "mismatches": bad}
    print(name, res[name], flush=True)

a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
for eng in ("tc-f4", "tc-i8"):
    g.set_engine(eng)
    stress(f"cfg3_{eng}", lambda: g.mul_strassen(a, b), want_digest=dig["cfg3"])
g.set_engine("tc-f4")
stress("cfg3_tc-f4_depth2", lambda: g.mul_strassen(a, b, g.MulParams(cutoff=4096)), want_digest=dig["cfg3"])
stress("cfg3_m4rm", lambda: g.mul_m4rm(a, b, 8), want_digest=dig["cfg3"])
m, l, n = 3001, 2750, 5003
x, y = g.random(m, l, 5), g.random(l, n, 6)
want = P.mul_strassen(O.random(m, l, 5), O.random(l, n, 6), cutoff=64).words
stress("odd_direct_tc-f4", lambda: g.mul_direct(x, y), want_words=want)
print(json.dumps(res))
