"""Kernel timeline of one Strassen multiply (torch.profiler / CUPTI): start,
end and the idle gap before each kernel, to locate launch gaps in the step,
then the device time per kernel name.

  python tools/timeline.py                 # cfg3 16384^3 mul_strassen
  python tools/timeline.py --size 65536 --addmul --summary   # cfg5
  python tools/timeline.py --size 4096 --cutoff 1024          # cfg2
  python tools/timeline.py --cfg4 [--addmul]                  # cfg4
"""
import argparse
import collections
import re
import sys

import torch

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--addmul", action="store_true")
ap.add_argument("--cutoff", type=int, default=0, help="0 = device default")
ap.add_argument("--cfg4", action="store_true",
                help="cfg4: 10000x7001 . 7001x12345 Bernoulli(0.1), mul_strassen")
ap.add_argument("--summary", action="store_true",
                help="only the per-kernel totals, not every launch")
args = ap.parse_args()
n = args.size
torch.cuda.set_device(0)
a, b = g.random(n, n, 51 if n > 16384 else 31), g.random(n, n, 52 if n > 16384 else 32)
c = g.random(n, n, 53) if args.addmul else None
if args.cfg4:
    thr = (1 << 64) // 10
    a = g.bernoulli(10000, 7001, 41, threshold=thr)
    b = g.bernoulli(7001, 12345, 42, threshold=thr)
    c = g.random(10000, 12345, 43) if args.addmul else None


params = g.MulParams(cutoff=args.cutoff, k=8) if args.cutoff else None


def step():
    if args.addmul:
        g.addmul(c, a, b, params)
    else:
        g.mul_strassen(a, b, params)


for _ in range(2):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(args.reps):
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = None
busy = 0.0
tot = collections.defaultdict(lambda: [0, 0.0])
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0
    if not args.summary:
        print(f"{(s - t0):9.1f} us  dur {t - s:8.1f}  gap {gap:7.1f}  {e.name[:60]}")
    name = re.split(r"[(<]", e.name.replace("(anonymous namespace)::", "")
                    .replace("void ", ""))[0][:48]
    tot[name][0] += 1
    tot[name][1] += t - s
    if prev_end is None or s >= prev_end:
        busy += t - s
    elif t > prev_end:
        busy += t - prev_end
    prev_end = max(prev_end or 0, t)
span = prev_end - t0
print(f"\n{args.reps} x {'addmul' if args.addmul else 'mul_strassen'} {n}^3: "
      f"span {span / args.reps / 1e3:.3f} ms/rep, device busy "
      f"{busy / args.reps / 1e3:.3f} ms/rep")
for name, (cnt, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"  {us / args.reps / 1e3:9.3f} ms/rep  {cnt / args.reps:7.1f} launches/rep  {name}")
