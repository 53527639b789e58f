"""Host-submission probe (design aid): CPU time to enqueue one 16384^3
mul_strassen, and device step time when the queue is (a) fed just in time
vs (b) primed by a long kernel so host latency cannot show."""
import sys, time, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
for _ in range(3): g.mul_strassen(a, b)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter(); c = g.mul_strassen(a, b); ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
print(f"host enqueue per call: min {min(ts)*1e6:.0f} us  median {sorted(ts)[10]*1e6:.0f} us")
big = torch.empty(4 << 30, dtype=torch.uint8, device='cuda')
for mode in ("just-in-time", "primed"):
    res = []
    for _ in range(10):
        torch.cuda.synchronize()
        if mode == "primed":
            big.zero_()                    # ~1 ms of GPU work queued ahead
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.mul_strassen(a, b); e1.record(); e1.synchronize()
        res.append(e0.elapsed_time(e1))
    print(mode, f"step ms min {min(res):.3f} median {sorted(res)[5]:.3f}")
