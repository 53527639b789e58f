"""Host-overhead probe: back-to-back eager mul_strassen vs StrassenPlan
replays (no L2 flush between, so host submission shows)."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
torch.cuda.set_device(0)
for n in (2048, 4096, 16384):
    a, b = g.random(n, n, 1), g.random(n, n, 2)
    c = g.create(n, n)
    plan = g.StrassenPlan(c, a, b)
    for mode in ("eager", "plan"):
        fn = (lambda: g.mul_strassen(a, b)) if mode == "eager" else plan.run
        for _ in range(5): fn()
        torch.cuda.synchronize()
        reps = 50 if n < 16384 else 10
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        print(f"{n}^3 {mode:5s}: {e0.elapsed_time(e1) / reps * 1e3:8.1f} us per multiply", flush=True)
