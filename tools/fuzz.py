"""Randomized parity fuzzer (GPU): engines x entry points x shapes x window
offsets x cutoffs, every result compared bit-exactly with the C port of the
reference algorithm (itself pinned to the reference's golden vectors by
tests/test_oracle.py). Runs for a time budget; writes a JSON summary.

    python tools/fuzz.py SECONDS [OUT.json] [--big]

--big: tensor engines only, shapes 512..9000, cutoffs 512..4096, so the
recursions run with tensor-core leaves (fewer, larger cases).
"""
import json, sys, time, traceback
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
from oracle import gf2_port as P

torch.cuda.set_device(0)
P.set_threads(P.max_threads())
args = [x for x in sys.argv[1:] if not x.startswith("--")]
BIG = "--big" in sys.argv
budget = float(args[0]) if args else 600
out = args[1] if len(args) > 1 else "gpurun_out/fuzz.json"
rng = np.random.default_rng(int(time.time()))
ENGINES = ["tc-i8", "tc-f8", "tc-f4"] if BIG else ["m4rm", "tc-i8", "tc-f8", "tc-f4"]
OPS = ["mul_m4rm", "mul_direct", "mul_strassen", "addmul", "addmul_direct", "mul_m4rm_into"]


def dim(big):
    if BIG:
        if rng.random() < 0.4:
            return max(512, 256 * int(rng.integers(2, 36)) + int(rng.integers(-2, 3)))
        return int(rng.integers(512, 9001))
    r = rng.random()
    hi = 6000 if big else 1500
    if r < 0.15:
        return int(rng.integers(1, 70))
    if r < 0.45:  # near a multiple of 64 (or of 64*2^d)
        base = 64 * int(rng.integers(1, hi // 64 + 1)) * int(rng.choice([1, 1, 2, 4]))
        return max(1, min(hi * 2, base + int(rng.integers(-2, 3))))
    return int(rng.integers(1, hi + 1))


def host_window(par, r0, wc, nr, nc):
    w = np.ascontiguousarray(par[r0:r0 + nr, wc:wc + O.words_per_row(nc)])
    if nc % 64 and w.shape[1]:
        w[:, -1] &= np.uint64(O.tail_mask(nc))
    return O.HostMat(nr, nc, w)


stats, failures = {}, []
t_end = time.time() + budget
n = 0
while time.time() < t_end:
    seed = int(rng.integers(1, 2**31))
    eng = str(rng.choice(ENGINES))
    op = str(rng.choice(OPS))
    big = rng.random() < 0.3
    m, l, nn = dim(big), dim(big), dim(big)
    case = dict(seed=seed, engine=eng, op=op, m=m, l=l, n=nn)
    try:
        g.set_engine(eng)
        win = rng.random() < 0.5
        ra, ca, rb, cb = (int(x) for x in rng.integers(0, 3, 4)) if win else (0, 0, 0, 0)
        pa = g.random(m + ra, l + 64 * ca + (7 if win else 0), seed)
        pb = g.random(l + rb, nn + 64 * cb + (5 if win else 0), seed + 1)
        a = g.window(pa, ra, 64 * ca, m, l) if win else pa
        b = g.window(pb, rb, 64 * cb, l, nn) if win else pb
        ha = host_window(pa.to_numpy(), ra, ca, m, l)
        hb = host_window(pb.to_numpy(), rb, cb, l, nn)
        want = P.mul_strassen(ha, hb, cutoff=64).words
        cutoff = int(rng.choice([512, 1024, 2048, 4096] if BIG else [64, 128, 256, 512, 1024, 2048]))
        case.update(window=win, cutoff=cutoff)
        if op in ("mul_m4rm", "mul_direct", "mul_strassen"):
            if op == "mul_m4rm":
                got = g.mul_m4rm(a, b, int(rng.integers(1, 17)))
            elif op == "mul_direct":
                got = g.mul_direct(a, b)
            else:
                got = g.mul_strassen(a, b, g.MulParams(cutoff=cutoff, k=8))
            ok = np.array_equal(got.to_numpy(), want) and g.trailing_bits_clean(got)
        else:
            c = g.random(m, nn, seed + 2)
            c0 = c.to_numpy()
            if op == "addmul":
                g.addmul(c, a, b, g.MulParams(cutoff=cutoff, k=8))
            elif op == "addmul_direct":
                g.addmul_direct(c, a, b)
            else:
                g.mul_m4rm_into(c, a, b, int(rng.integers(1, 17)), 512, int(rng.integers(1, 9)))
            ok = np.array_equal(c.to_numpy(), c0 ^ want)
    except Exception:
        ok = False
        case["error"] = traceback.format_exc()[-600:]
    key = f"{eng}/{op}"
    st = stats.setdefault(key, {"runs": 0, "fail": 0})
    st["runs"] += 1
    n += 1
    if not ok:
        st["fail"] += 1
        failures.append(case)
        print("FAIL", case, flush=True)
summary = {"seconds": budget, "cases": n, "failures": len(failures), "by_engine_op": stats,
           "failed_cases": failures[:50]}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({"cases": n, "failures": len(failures)}))
