"""Crossover probe (design aid): M4RM vs the tc-f4 engine for one product
of size s^3 (device-resident, events, min of reps)."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
g.set_engine("tc-f4")
for s in (1024, 1536, 2048, 2560, 3072, 4096):
    a, b = g.random(s, s, 1), g.random(s, s, 2)
    tm = t(lambda: g.mul_m4rm(a, b, 8))
    tf = t(lambda: g.mul_direct(a, b))
    print(f"{s}^3 = 2^{(s**3).bit_length()-1}: m4rm {tm*1e3:.1f} us  tc-f4 {tf*1e3:.1f} us")
