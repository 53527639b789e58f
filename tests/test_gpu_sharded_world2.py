"""The multi-GPU path at world size 2 with its REAL device multiply: two
processes, gloo for the collective (NCCL cannot put two ranks on one GPU),
both ranks' matrices on cuda:0. `sharded.mul_sharded` runs exactly as under
NCCL -- A and C row-sharded and generated in place, B broadcast in K-panels
(from rank 0, or each rank's block of rows from that rank), each panel an
`addmul` on the B200 kernels -- and the gathered C must equal the
single-process product. (tests/test_sharding_gloo.py covers the same plan on
CPU with an injected multiply.) The ranks' kernels never wait on each other:
the only synchronisation is gloo's, on the host."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, l, n, npanels, src, accumulate, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_0811_1714_b200 as g
        from paper_0811_1714_b200.sharded import mul_sharded, owned_rows, shard_rows
        r0, r1 = shard_rows(m, world, rank)
        a_p = g.random(r1 - r0, l, 1, row_base=r0)  # this rank's rows of A
        b = g.create(l, n)
        full = g.random(l, n, 2)
        for k0, k1 in owned_rows(l, world, rank, src):  # only the rows this rank supplies
            g.copy_into(g.window(b, k0, 0, k1 - k0, n), g.window(full, k0, 0, k1 - k0, n))
        del full
        if accumulate:
            c_p = g.random(r1 - r0, n, 3, row_base=r0)
            mul_sharded(a_p, b, src=src, npanels=npanels, c=c_p, accumulate=True)
        else:
            c_p = mul_sharded(a_p, b, src=src, npanels=npanels)
        torch.cuda.synchronize()
        parts = [None] * world
        dist.all_gather_object(parts, c_p.to_numpy().tolist())
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("src", [0, None])
@pytest.mark.parametrize("m,l,n,npanels,accumulate", [(3000, 4100, 2500, 3, False),
                                                      (1100, 700, 1300, 2, True),
                                                      (129, 64, 65, 2, False)])
def test_mul_sharded_world2_device(m, l, n, npanels, accumulate, src):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_0811_1714_b200 as g
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, l, n, npanels, src, accumulate, q))
             for r in range(2)]
    for p in procs:
        p.start()
    try:
        parts = q.get(timeout=300)
    finally:
        for p in procs:
            p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    got = np.array([w for part in parts for w in part], dtype=np.uint64)
    a, b = g.random(m, l, 1), g.random(l, n, 2)
    want = g.mul_strassen(a, b).to_numpy()
    if accumulate:
        want = want ^ g.random(m, n, 3).to_numpy()
    assert np.array_equal(got.reshape(want.shape), want)
