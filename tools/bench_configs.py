"""Supplementary measurements for all five BASELINE.json configs (bench.py
reports the headline cfg3 line). Device-resident inputs, CUDA-event timing,
warm-up excluded, L2 flushed between reps, every result digest-verified.

    python tools/bench_configs.py [--reps R] [--engine tc-f4|tc-i8|tc-f8|m4rm]
                                  [--cutoff C]  (overrides the device default)
"""

import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_0811_1714_b200 as g  # noqa: E402


def digest(m):
    return hashlib.sha256(m.to_numpy().astype("<u8").tobytes()).hexdigest()


def timed(fn, reps, flush):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return out, min(ts), sum(ts) / len(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--engine", default="tc-f4")
    ap.add_argument("--cutoff", type=int, default=0)
    ap.add_argument("--skip-cfg5", action="store_true")
    args = ap.parse_args()
    g.set_engine(args.engine)
    if args.cutoff:
        g.strassen.GPU_CUTOFF = args.cutoff
    torch.cuda.set_device(0)
    dig = json.load(open(os.path.join(ROOT, "tests", "golden", "digests.json")))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    rows = []

    def rec(cfg, call, mln, fn, key, extra=None):
        out, tmin, tmean = timed(fn, args.reps, flush)
        m, l, n = mln
        d = {"cfg": cfg, "call": call, "m": m, "l": l, "n": n, "engine": args.engine,
             "gpu_cutoff": g.strassen.GPU_CUTOFF,
             "ms_min": tmin, "ms_mean": tmean, "bitops_per_s": m * l * n / (tmin * 1e-3),
             "verified_sha256": digest(out() if callable(out) else out) == dig[key]}
        if extra:
            d.update(extra)
        rows.append(d)
        print(json.dumps(d), flush=True)

    a, b = g.random(1024, 1024, 11), g.random(1024, 1024, 12)
    rec("cfg1", "mul_m4rm(A,B,8)", (1024,) * 3, lambda: g.mul_m4rm(a, b, 8), "cfg1")
    rec("cfg1", "mul_direct(A,B)", (1024,) * 3, lambda: g.mul_direct(a, b), "cfg1")
    a, b = g.random(4096, 4096, 21), g.random(4096, 4096, 22)
    p2 = g.MulParams(cutoff=1024, k=8)
    rec("cfg2", "mul_strassen(A,B,MulParams(cutoff=1024,k=8))", (4096,) * 3,
        lambda: g.mul_strassen(a, b, p2), "cfg2")
    rec("cfg2", "mul_strassen(A,B)", (4096,) * 3, lambda: g.mul_strassen(a, b), "cfg2")
    a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
    rec("cfg3", "mul_strassen(A,B)", (16384,) * 3, lambda: g.mul_strassen(a, b), "cfg3")
    rec("cfg3", "mul_m4rm(A,B,8)", (16384,) * 3, lambda: g.mul_m4rm(a, b, 8), "cfg3")
    del a, b
    a = g.bernoulli(10000, 7001, 41, p=0.1)
    b = g.bernoulli(7001, 12345, 42, p=0.1)
    rec("cfg4", "mul_strassen(A,B)", (10000, 7001, 12345), lambda: g.mul_strassen(a, b),
        "cfg4_product")
    c0 = g.random(10000, 12345, 43)
    c = g.create(10000, 12345)

    def addmul4():
        g.copy_into(c, c0)
        g.addmul(c, a, b)
        return c
    rec("cfg4", "C0 copy + addmul(C,A,B)", (10000, 7001, 12345), addmul4, "cfg4_addmul")

    def into4():
        g.copy_into(c, c0)
        g.mul_m4rm_into(c, a, b, 8, 512, 8)
        return c
    rec("cfg4", "C0 copy + mul_m4rm_into(C,A,B,8,512,8)", (10000, 7001, 12345), into4,
        "cfg4_addmul")
    del a, b, c, c0
    if not args.skip_cfg5:
        n = 65536
        a, b = g.random(n, n, 51), g.random(n, n, 52)
        c0 = g.random(n, n, 53)
        c = g.create(n, n)

        def addmul5():
            g.copy_into(c, c0)
            g.addmul(c, a, b)
            return c
        rec("cfg5", "C0 copy + addmul(C,A,B)", (n,) * 3, addmul5, "cfg5_addmul")
    out = os.path.join(ROOT, "gpurun_out", f"configs_{args.engine}_c{g.strassen.GPU_CUTOFF}.jsonl")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as fh:
        for r in rows:
            fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
