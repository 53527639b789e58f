"""Kernel timeline of one cfg3 step (torch.profiler / CUPTI): start, end and
the idle gap before each kernel, to locate launch gaps in the step."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from torch.profiler import profile, ProfilerActivity
torch.cuda.set_device(0)
a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
for _ in range(3): g.mul_strassen(a, b)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        c = g.mul_strassen(a, b)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = None
for e in evs:
    s, t = e.time_range.start, e.time_range.end
    gap = (s - prev_end) if prev_end is not None else 0
    print(f"{(s - t0):9.1f} us  dur {t - s:8.1f}  gap {gap:7.1f}  {e.name[:60]}")
    prev_end = max(prev_end or 0, t)
