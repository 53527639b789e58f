"""Largest shapes one B200 holds comfortably, beyond BASELINE.json's cfg5:
the tensor-core recursion (tc-f4) and the M4RM engine must agree bit for bit
(two independent kernels), and both must pass the Freivalds check
C.X == A.(B.X) (a third kernel path: one-word M4RM tiles). Also reports the
time per multiply and the workspace high-water mark.

  python tools/max_size.py [OUT.json]            # 131072^3 and a ragged giant
  python tools/max_size.py OUT.json --huge       # also 262144^3 (8 GiB per matrix):
                                                 # the recursion is taken shallower
                                                 # so its workspace fits the device
"""
import json
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402
from paper_0811_1714_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
CASES = [("square 131072^3", 131072, 131072, 131072, False),
         ("ragged 100003 x 90001 x 120007, addmul", 100003, 90001, 120007, True)]


if "--only-huge" in sys.argv:
    sys.argv[sys.argv.index("--only-huge")] = "--huge"
    CASES.clear()
if "--huge" in sys.argv:
    sys.argv.remove("--huge")
    CASES.append(("square 262144^3 (depth limited by the workspace budget)",
                  262144, 262144, 262144, False))


def freivalds(c, a, b, c0=None, reps=2):
    for r in range(reps):
        x = g.random(b.ncols, 64, 900 + r)
        lhs = g.mul_m4rm(c, x, 8)
        rhs = g.mul_m4rm(a, g.mul_m4rm(b, x, 8), 8)
        if c0 is not None:
            rhs = g.add(rhs, g.mul_m4rm(c0, x, 8))
        if not g.equal(lhs, rhs):
            return False
    return True


def run(engine, a, b, c0):
    g.set_engine(engine)
    _lib.workspace_peak(reset=True)
    best = None
    for _ in range(2 if a.nrows < 200000 else 1):
        c = None
        c = g.copy_out(c0) if c0 is not None else None
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if c0 is not None:
            g.addmul(c, a, b)
        else:
            c = g.mul_strassen(a, b)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    peak = _lib.workspace_peak()
    g.release_workspace()
    return c, best, peak


out = []
ok_all = True
for name, m, l, n, addmul in CASES:
    a, b = g.random(m, l, 71), g.random(l, n, 72)
    c0 = g.random(m, n, 73) if addmul else None
    c_tc, t_tc, pk_tc = run("tc-f4", a, b, c0)
    c_lut, t_lut, pk_lut = run("m4rm", a, b, c0)
    g.set_engine("tc-f4")
    same = bool(g.equal(c_tc, c_lut))
    fr = freivalds(c_tc, a, b, c0)
    clean = bool(g.trailing_bits_clean(c_tc))
    w = float(m) * l * n
    rec = {"case": name, "m": m, "l": l, "n": n, "addmul": addmul,
           "engines_agree": same, "freivalds": fr, "trailing_bits_clean": clean,
           "tc_f4_ms": t_tc * 1e3, "tc_f4_bitops_per_s": w / t_tc,
           "m4rm_ms": t_lut * 1e3, "m4rm_bitops_per_s": w / t_lut,
           "workspace_peak_bytes": {"tc-f4": pk_tc, "m4rm": pk_lut}}
    print(json.dumps(rec), flush=True)
    out.append(rec)
    ok_all = ok_all and same and fr and clean
    del a, b, c0, c_tc, c_lut
    g.release_workspace()
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as fh:
        for rec in out:
            fh.write(json.dumps(rec) + "\n")
sys.exit(0 if ok_all else 1)
