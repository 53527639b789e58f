"""Multi-GPU C = A.B over GF(2) with the drop-in package: one process per GPU,
launched with torchrun.

    torchrun --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
        examples/sharded_mul.py --size 65536 [--grid auto|rows|PRxPC]

Layout `rows` (north_star (e)): C and A are row-sharded, B lives on rank 0 and
is broadcast over NVLink with NCCL in K-panels while the panels multiply.
Layout `PRxPC` / `auto`: a process grid; rank (i, j) owns C[rows_i, cols_j],
B's column block j is broadcast inside column group j only. Either way no
reduction is needed (K is never split across ranks), and the result is
bit-identical to the one-GPU product: every rank checks its block with
Freivalds' test (C.x == A.(B.x) for random 64-column x, B.x computed once
from the full B, which this example keeps on every rank just for the check).

`--backend gloo --one-gpu` runs all ranks on cuda:0 with gloo for the
collectives (NCCL cannot place two ranks on one GPU): a code-path check on a
one-GPU machine, not a measurement.
"""
import argparse
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_0811_1714_b200 as g  # noqa: E402
from paper_0811_1714_b200.sharded import (ProcessGrid, choose_grid, mul_sharded,  # noqa: E402
                                          mul_sharded_grid, shard_rows)

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=16384)
ap.add_argument("--grid", default="rows")
ap.add_argument("--npanels", type=int, default=2)
ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
ap.add_argument("--one-gpu", action="store_true")
args = ap.parse_args()

rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
local = 0 if args.one_gpu else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if args.backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
else:
    dist.init_process_group("gloo")

n = args.size
if args.grid == "rows":
    pr, pc = world, 1
elif args.grid == "auto":
    pr, pc = choose_grid(world, n, n)
else:
    pr, pc = (int(x) for x in args.grid.lower().split("x"))
grid = ProcessGrid(world, rank, pr, pc, make_groups=pc > 1)
(r0, r1), (c0, c1) = grid.rows(n), grid.cols(n)

a_i = g.random(r1 - r0, n, 1, row_base=r0)          # this rank's rows of A, generated in place
b_full = g.random(n, n, 2)                           # every rank, only for the check below
if pc == 1:
    b = b_full if rank == 0 else g.create(n, n)      # contents matter on rank 0 only
else:
    b = g.create(n, c1 - c0)                         # column block B_j, filled on grid row 0
    if grid.i == 0:
        g.copy_into(b, g.window(b_full, 0, c0, n, c1 - c0))


def multiply():
    if pc == 1:
        return mul_sharded(a_i, b, src=0, npanels=args.npanels)
    return mul_sharded_grid(a_i, b, grid, src_row=0, npanels=args.npanels)


c = multiply()                                       # warm-up (workspace pool, NCCL channels)
torch.cuda.synchronize()
dist.barrier()
t0 = time.perf_counter()
c = multiply()
torch.cuda.synchronize()
dist.barrier()
dt = time.perf_counter() - t0

# Freivalds on this rank's block: C[rows_i, cols_j] . x[cols_j] summed over j
# equals A[rows_i, :] . (B . x) -- so check per block with x supported on cols_j
x = g.create(n, 64)
g.copy_into(g.window(x, c0, 0, c1 - c0, 64), g.random(c1 - c0, 64, 3))
lhs = g.mul_m4rm(c, g.window(x, c0, 0, c1 - c0, 64), 8)
rhs = g.mul_m4rm(a_i, g.mul_m4rm(b_full, x, 8), 8)
ok = bool(g.equal(lhs, rhs))
flags = [None] * world
dist.all_gather_object(flags, ok)
if rank == 0:
    print(f"{n}^3 on {world} rank(s), layout {pr}x{pc}, {args.npanels} K-panels: "
          f"{dt * 1e3:.3f} ms wall, {float(n) ** 3 / dt:.3e} bit-ops/s, "
          f"Freivalds on every block: {all(flags)}")
dist.destroy_process_group()
sys.exit(0 if all(flags) else 1)
