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


def _grid_worker(rank, world, port, pr, pc, m, l, n, npanels, src_row, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import gf2_oracle as O
        from paper_0811_1714_b200.sharded import (ProcessGrid, gather_rows,
                                                  k_panels, owned_rows,
                                                  pipelined_broadcast,
                                                  shard_rows)
        grid = ProcessGrid(world, rank, pr, pc, make_groups=True)
        r0, r1 = grid.rows(m)
        c0, c1 = grid.cols(n)
        wa = O.words_per_row(l)
        # A_i: each rank of row group i holds 1/pc of its rows, gathered
        full_a = O.random(m, l, 1).words.view(np.int64)
        a_rows = torch.zeros((r1 - r0, wa), dtype=torch.int64)
        pieces = [shard_rows(r1 - r0, pc, j) for j in range(pc)]
        p0, p1 = pieces[grid.j]
        a_rows[p0:p1] = torch.from_numpy(full_a[r0 + p0:r0 + p1])
        gather_rows(a_rows, pieces, grid.row_ranks(grid.i), group=grid.row_group)
        assert np.array_equal(a_rows.numpy(), full_a[r0:r1])
        # B_j: the column block, rows supplied inside column group j
        bj = O.view(O.random(l, n, 2).words, 0, c0, l, c1 - c0)
        full_bj = O.masked(bj).view(np.int64)
        wb = full_bj.shape[1]
        b_rows = torch.zeros((l, wb), dtype=torch.int64)
        src = None if src_row is None else grid.col_ranks(grid.j)[src_row]
        for k0, k1 in owned_rows(l, pr, grid.i, None) if src is None else \
                owned_rows(l, world, rank, src):
            b_rows[k0:k1] = torch.from_numpy(full_bj[k0:k1])
        c_blk = np.zeros((r1 - r0, wb), dtype=np.uint64)
        a_p = O.HostMat(r1 - r0, l, a_rows.numpy().view(np.uint64))

        def local(k0, k1):
            bw = b_rows[k0:k1].numpy().view(np.uint64)
            a_pan = O.view(a_p.words, 0, k0, r1 - r0, k1 - k0)
            c_blk[:] ^= O.naive_product(a_pan, O.HostMat(k1 - k0, c1 - c0, bw)).words

        pipelined_broadcast(b_rows, k_panels(l, npanels), local, src=src,
                            group=grid.col_group)
        parts = [None] * world
        dist.all_gather_object(parts, (grid.block_of(rank, m, n), c_blk.tolist()))
        if rank == 0:
            q.put(parts)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("src_row", [0, None])
@pytest.mark.parametrize("pr,pc,m,l,n,npanels", [(2, 2, 300, 700, 520, 3),
                                                 (1, 2, 129, 64, 300, 2),
                                                 (2, 1, 200, 130, 65, 2)])
def test_process_grid_world(pr, pc, m, l, n, npanels, src_row):
    """pr x pc process grid on CPU (gloo): A_i gathered by rows inside the row
    group, B_j broadcast inside the column group, C blocks assembled."""
    from oracle import gf2_oracle as O
    world = pr * pc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grid_worker,
                         args=(r, world, port, pr, pc, m, l, n, npanels, src_row, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = O.naive_product(O.random(m, l, 1), O.random(l, n, 2)).words
    got = np.zeros_like(want)
    for (r0, r1, c0, c1), words in parts:
        blk = np.array(words, dtype=np.uint64).reshape(r1 - r0, -1)
        assert c0 % 64 == 0
        got[r0:r1, c0 // 64:c0 // 64 + blk.shape[1]] |= blk
    assert np.array_equal(got, want)


def test_grid_partition_properties():
    from paper_0811_1714_b200.sharded import ProcessGrid, choose_grid, shard_cols
    for world in (1, 2, 4, 6, 8):
        for m, n in ((16384, 16384), (10000, 12345), (65, 4000), (1, 1)):
            pr, pc = choose_grid(world, m, n)
            assert pr * pc == world
            cover = np.zeros((m, n), dtype=np.uint8) if m * n < 1 << 22 else None
            cells = 0
            for r in range(world):
                g = ProcessGrid(world, r, pr, pc)
                assert r in g.col_ranks(g.j) and r in g.row_ranks(g.i)
                assert len(g.col_ranks(g.j)) == pr and len(g.row_ranks(g.i)) == pc
                r0, r1, c0, c1 = g.block_of(r, m, n)
                assert (r0, r1) == g.rows(m) and (c0, c1) == g.cols(n)
                assert c0 % 128 == 0 or c0 == n or n < 128 * pc
                cells += (r1 - r0) * (c1 - c0)
                if cover is not None:
                    cover[r0:r1, c0:c1] += 1
            assert cells == m * n
            if cover is not None:
                assert (cover == 1).all()
    assert choose_grid(2, 16384, 16384) == (2, 1)      # ties keep row sharding
    assert choose_grid(8, 65536, 65536) == (2, 4)      # ties from 4 ranks on: more column blocks
    with pytest.raises(ValueError):
        ProcessGrid(4, 0, 3, 2)
    assert shard_cols(300, 2, 0) == (0, 256) and shard_cols(300, 2, 1) == (256, 300)
