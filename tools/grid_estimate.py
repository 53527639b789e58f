"""Per-rank compute of the sharded multi-GPU path on a pr x pc process grid,
measured on one GPU (no NCCL: rank (0, 0)'s block, its operands present):
C[rows_i, cols_j] += A[rows_i, :] . B[:, cols_j] in K-panels, as
mul_sharded runs it inside column group j. pc = 1 is the row-sharded layout
of north_star (e). Usage: grid_estimate.py [16384|65536] [npanels]"""
import sys, torch
sys.path.insert(0, '.')
import paper_0811_1714_b200 as g
from paper_0811_1714_b200.sharded import k_panels, shard_rows, shard_cols
torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
npanels = int(sys.argv[2]) if len(sys.argv) > 2 else 2
sa, sb = (31, 32) if n == 16384 else (51, 52)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=6):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


a_full, b_full = g.random(n, n, sa), g.random(n, n, sb)
c_full = g.create(n, n)
t1 = timed(lambda: g.addmul(c_full, a_full, b_full))
print(f"n={n} N=1 addmul {t1:.3f} ms")
del a_full, c_full
for world, grids in ((2, ((2, 1), (1, 2))), (4, ((4, 1), (2, 2), (1, 4))),
                     (8, ((8, 1), (4, 2), (2, 4)))):
    for pr, pc in grids:
        r0, r1 = shard_rows(n, pr, 0)
        c0, c1 = shard_cols(n, pc, 0)
        a_p = g.random(r1 - r0, n, sa, row_base=r0)
        b_p = g.copy_out(g.window(b_full, 0, c0, n, c1 - c0)) if pc > 1 else b_full
        c = g.create(r1 - r0, c1 - c0)
        panels = k_panels(n, npanels)

        def rank_work():
            for k0, k1 in panels:
                g.addmul(c, g.window(a_p, 0, k0, r1 - r0, k1 - k0),
                         g.window(b_p, k0, 0, k1 - k0, c1 - c0))
        t = timed(rank_work)
        print(f"N={world} grid {pr}x{pc} block {r1-r0}x{c1-c0} npanels={npanels}: "
              f"rank compute {t:.3f} ms (ideal {t1/world:.3f}, eff {t1/world/t:.2f})", flush=True)
        del a_p, c
        if pc > 1:
            del b_p
