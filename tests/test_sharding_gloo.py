"""World-size-2 run of the multi-GPU plan on CPU (gloo): A and C sharded by
row blocks, B broadcast in K-panels -- all from rank 0, or (src=None) each
rank's block of B's rows from that rank -- every rank accumulating its C
rows panel by panel. The local multiply is injected (here the CPU oracle,
as the checker); the gathered C must equal the single-process product."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, l, n, npanels, src, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import gf2_oracle as O
        from paper_0811_1714_b200.sharded import (k_panels, owned_rows,
                                                  pipelined_broadcast,
                                                  shard_rows)
        r0, r1 = shard_rows(m, world, rank)
        a_p = O.random(r1 - r0, l, 1, row_base=r0)    # generated in place
        wb = O.words_per_row(n)
        full_b = O.random(l, n, 2).words.view(np.int64)
        b_rows = torch.zeros((l, wb), dtype=torch.int64)
        for k0, k1 in owned_rows(l, world, rank, src):
            b_rows[k0:k1] = torch.from_numpy(full_b[k0:k1])   # only own rows
        c_p = np.zeros((r1 - r0, wb), dtype=np.uint64)

        def local(k0, k1):
            bw = b_rows[k0:k1].numpy().view(np.uint64)
            a_pan = O.view(a_p.words, 0, k0, r1 - r0, k1 - k0)
            c_p[:] ^= O.naive_product(a_pan, O.HostMat(k1 - k0, n, bw)).words

        pipelined_broadcast(b_rows, k_panels(l, npanels), local, src=src)
        sizes = [None] * world
        dist.all_gather_object(sizes, c_p.tolist())
        if rank == 0:
            q.put(sizes)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("src", [0, None])
@pytest.mark.parametrize("m,l,n,npanels", [(300, 700, 200, 3),
                                           (129, 64, 65, 2)])
def test_row_sharded_broadcast_pipeline_world2(m, l, n, npanels, src):
    from oracle import gf2_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, m, l, n, npanels, src, q))
             for r in range(2)]
    for p in procs:
        p.start()
    parts = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.array([w for part in parts for w in part], dtype=np.uint64)
    want = O.naive_product(O.random(m, l, 1), O.random(l, n, 2)).words
    assert np.array_equal(got.reshape(want.shape), want)
