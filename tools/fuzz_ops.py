"""Randomized fuzzer for the non-multiply operations of the path (GPU):
word ops on windows (add_into / copy_into / zero_into keep every bit outside
the target window), transpose, stack, augment (any column split), mul_cubic,
from_dense / to_dense, equal / first_difference -- each against NumPy on
dense 0/1 arrays. Runs for a time budget; writes a JSON summary.

    python tools/fuzz_ops.py SECONDS [OUT.json]
"""
import json, sys, time, traceback
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g

torch.cuda.set_device(0)
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/fuzz_ops.json"
rng = np.random.default_rng(int(time.time()))


def dim(hi=700):
    r = rng.random()
    if r < 0.2:
        return int(rng.integers(1, 70))
    if r < 0.5:
        return max(1, 64 * int(rng.integers(1, hi // 64 + 1)) + int(rng.integers(-2, 3)))
    return int(rng.integers(1, hi + 1))


def rand_dense(r, c):
    return (rng.random((r, c)) < 0.5).astype(np.uint8)


def parent_with_window(r, c):
    """A device parent with a window of r x c at a random 64-column offset,
    and the parent's dense copy and offsets."""
    ro, co = int(rng.integers(0, 4)), 64 * int(rng.integers(0, 3))
    pd = rand_dense(r + ro + int(rng.integers(0, 4)), c + co + int(rng.integers(0, 90)))
    par = g.from_dense(pd)
    return par, g.window(par, ro, co, r, c), pd, ro, co


OPS = ["add_into", "copy_into", "zero_into", "transpose", "stack", "augment", "mul_cubic",
       "dense_roundtrip", "equal_first_difference"]
stats, failures, n = {}, [], 0
t_end = time.time() + budget
while time.time() < t_end:
    op = str(rng.choice(OPS))
    r, c = dim(), dim()
    case = {"op": op, "r": r, "c": c}
    try:
        if op in ("add_into", "copy_into", "zero_into"):
            par, w, pd, ro, co = parent_with_window(r, c)
            a_d, b_d = rand_dense(r, c), rand_dense(r, c)
            a, b = g.from_dense(a_d), g.from_dense(b_d)
            exp = pd.copy()
            if op == "add_into":
                g.add_into(w, a, b)
                exp[ro:ro + r, co:co + c] = a_d ^ b_d
            elif op == "copy_into":
                g.copy_into(w, a)
                exp[ro:ro + r, co:co + c] = a_d
            else:
                g.zero_into(w)
                exp[ro:ro + r, co:co + c] = 0
            ok = np.array_equal(g.to_dense(par), exp) and g.trailing_bits_clean(par)
        elif op == "transpose":
            par, w, pd, ro, co = parent_with_window(r, c)
            t = g.transpose(w)
            ok = np.array_equal(g.to_dense(t), pd[ro:ro + r, co:co + c].T) and g.trailing_bits_clean(t)
        elif op == "stack":
            r2 = dim()
            a_d, b_d = rand_dense(r, c), rand_dense(r2, c)
            s = g.stack(g.from_dense(a_d), g.from_dense(b_d))
            ok = np.array_equal(g.to_dense(s), np.vstack([a_d, b_d])) and g.trailing_bits_clean(s)
        elif op == "augment":
            c2 = dim()
            a_d, b_d = rand_dense(r, c), rand_dense(r, c2)
            s = g.augment(g.from_dense(a_d), g.from_dense(b_d))
            ok = np.array_equal(g.to_dense(s), np.hstack([a_d, b_d])) and g.trailing_bits_clean(s)
        elif op == "mul_cubic":
            n2 = int(rng.integers(1, 80))
            a_d, b_d = rand_dense(r, c), rand_dense(c, n2)
            p = g.mul_cubic(g.from_dense(a_d), g.from_dense(b_d))
            want = (a_d.astype(np.int64) @ b_d.astype(np.int64)) & 1
            ok = np.array_equal(g.to_dense(p), want.astype(np.uint8))
        elif op == "dense_roundtrip":
            a_d = rand_dense(r, c)
            ok = np.array_equal(g.to_dense(g.from_dense(a_d)), a_d)
        else:
            a_d = rand_dense(r, c)
            b_d = a_d.copy()
            same = rng.random() < 0.3
            if not same:
                i, j = int(rng.integers(0, r)), int(rng.integers(0, c))
                b_d[i, j] ^= 1
            a, b = g.from_dense(a_d), g.from_dense(b_d)
            ok = g.equal(a, b) == same
            fd = g.first_difference(a, b)
            ok = ok and ((fd is None) if same else (tuple(fd) == (i, j)))
    except Exception:
        ok = False
        case["error"] = traceback.format_exc()[-600:]
    st = stats.setdefault(op, {"runs": 0, "fail": 0})
    st["runs"] += 1
    n += 1
    if not ok:
        st["fail"] += 1
        failures.append(case)
        print("FAIL", case, flush=True)
json.dump({"seconds": budget, "cases": n, "failures": len(failures), "by_op": stats,
           "failed_cases": failures[:50]}, open(out, "w"), indent=1)
print(json.dumps({"cases": n, "failures": len(failures)}))
