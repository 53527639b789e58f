"""cfg5 step accounting (design aid): CUDA-event time of one 65536^3 addmul
with the host feeding the GPU just in time vs the queue primed, the host
time of the call, and the device-busy time from the profiler."""
import sys
import time

import torch

sys.path.insert(0, '.')
import paper_0811_1714_b200 as g  # noqa: E402

torch.cuda.set_device(0)
n = 65536
a, b, c = g.random(n, n, 51), g.random(n, n, 52), g.random(n, n, 53)
prime = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
g.addmul(c, a, b)
torch.cuda.synchronize()
for mode in ("jit", "primed", "jit", "primed"):
    torch.cuda.synchronize()
    if mode == "primed":
        prime.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    g.addmul(c, a, b)
    th = time.perf_counter() - t0
    e1.record()
    e1.synchronize()
    print(f"{mode}: events {e0.elapsed_time(e1):.3f} ms, host call {th * 1e3:.3f} ms", flush=True)
