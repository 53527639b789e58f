import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
prime = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
def t(fn, reps=10):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        prime.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1)*1e3)
    return min(ts)
for (m, l, n, cut) in [(3000, 3000, 3000, 512), (2048, 2048, 2048, 512), (4096, 4096, 4096, 512), (6000, 5000, 7000, 1024), (8192, 8192, 8192, 600)]:
    a, b = g.random(m, l, 1), g.random(l, n, 2)
    p = g.MulParams(cutoff=cut, k=8)
    print(m, l, n, cut, round(t(lambda: g.mul_strassen(a, b, p)), 1), flush=True)
