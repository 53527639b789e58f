"""Per-rank compute of the row-sharded multi-GPU path, measured on one GPU
(no NCCL: rank 0's shard, B already present): C_p += A_p[:, panel] .
B[panel, :] for each K-panel, as mul_sharded runs it. Estimates the compute
side of strong scaling at N GPUs; the broadcast of B (32 MiB) overlaps it."""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from paper_0811_1714_b200.sharded import k_panels, shard_rows
torch.cuda.set_device(0)
n = 16384
b = g.random(n, n, 32)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
def timed(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
t1 = timed(lambda: g.mul_strassen(g.random(n, n, 31), b) and None)
print(f"N=1 full multiply (incl. A generation) {t1:.3f} ms")
for world in (2, 4, 8):
    r0, r1 = shard_rows(n, world, 0)
    a_p = g.random(r1 - r0, n, 31, row_base=r0)
    for npanels in (1, 2, 4):
        panels = k_panels(n, npanels)
        def rank_work():
            c = g.create(r1 - r0, n)
            for k0, k1 in panels:
                g.addmul(c, g.window(a_p, 0, k0, r1 - r0, k1 - k0), g.window(b, k0, 0, k1 - k0, n))
        t = timed(rank_work)
        print(f"N={world} rows={r1-r0} npanels={npanels}: rank compute {t:.3f} ms  (ideal {t1/world:.3f})")
