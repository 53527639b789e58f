"""Where the time goes in the small BASELINE configs (cfg1, cfg2 at the
reference's cutoff 1024, cfg4): per call, (a) CUDA-event time with the host
feeding the GPU just in time (what tools/bench_configs.py reports), (b) the
same call with the queue primed by a long kernel (device time only, host
latency hidden), (c) host enqueue time, and (d) the device time per kernel
(torch.profiler / CUPTI).

    python tools/small_profile.py [--reps 20]
"""
import argparse
import collections
import re
import sys
import time

import torch
from torch.profiler import profile, ProfilerActivity

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402


def ev_time(fn, reps, prime=None):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        if prime is not None:
            prime.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[0], ts[len(ts) // 2]


def host_time(fn, reps):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    ts.sort()
    return ts[len(ts) // 2] * 1e3


def kernels(fn, reps):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    tot = collections.defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        name = re.split(r"[(<]", e.name.replace("(anonymous namespace)::", "")
                        .replace("void ", ""))[0][:40]
        tot[name][0] += 1
        tot[name][1] += e.time_range.end - e.time_range.start
    return {k: (c / reps, us / reps) for k, (c, us) in tot.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    prime = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
    cases = []
    a1, b1 = g.random(1024, 1024, 11), g.random(1024, 1024, 12)
    cases.append(("cfg1 mul_m4rm(A,B,8) 1024^3", lambda: g.mul_m4rm(a1, b1, 8)))
    c1 = g.create(1024, 1024)
    plan1 = g.M4rmPlan(c1, a1, b1, 8)
    cases.append(("cfg1 M4rmPlan.run() 1024^3", plan1.run))
    a2, b2 = g.random(4096, 4096, 21), g.random(4096, 4096, 22)
    p2 = g.MulParams(cutoff=1024, k=8)
    cases.append(("cfg2 mul_strassen cutoff 1024", lambda: g.mul_strassen(a2, b2, p2)))
    cases.append(("cfg2 mul_strassen default", lambda: g.mul_strassen(a2, b2)))
    c2 = g.create(4096, 4096)
    plan2 = g.StrassenPlan(c2, a2, b2, p2)
    cases.append(("cfg2 StrassenPlan.run() cutoff 1024", plan2.run))
    a4 = g.bernoulli(10000, 7001, 41, 0.1)
    b4 = g.bernoulli(7001, 12345, 42, 0.1)
    c4 = g.random(10000, 12345, 43)
    cases.append(("cfg4 mul_strassen", lambda: g.mul_strassen(a4, b4)))
    cases.append(("cfg4 mul_m4rm_into(C,A,B,8,512,8)", lambda: g.mul_m4rm_into(c4, a4, b4, 8, 512, 8)))
    for name, fn in cases:
        for _ in range(3):
            fn()
        jit = ev_time(fn, args.reps)
        primed = ev_time(fn, args.reps, prime)
        host = host_time(fn, args.reps)
        ks = kernels(fn, 5)
        print(f"\n{name}: events just-in-time min {jit[0]*1e3:.1f} us med {jit[1]*1e3:.1f} us | "
              f"primed min {primed[0]*1e3:.1f} us med {primed[1]*1e3:.1f} us | host enqueue {host*1e3:.1f} us")
        for k, (cnt, us) in sorted(ks.items(), key=lambda kv: -kv[1][1]):
            print(f"    {us:9.1f} us  {cnt:5.1f} launches  {k}")


if __name__ == "__main__":
    main()
