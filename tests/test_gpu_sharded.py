"""The multi-GPU path (row-sharded C and A, B broadcast in K-panels over
NCCL) run for real on one GPU: a world-size-1 NCCL group exercises the
broadcast calls and the panel-by-panel addmul on the device; rank row
ranges of a larger world are emulated by generating each shard in place
(random(..., row_base=r0)) and checking every shard against the product."""

import os
import socket

import numpy as np
import pytest

from oracle import gf2_oracle as O

pytestmark = pytest.mark.gpu
g = pytest.importorskip("paper_0811_1714_b200")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("engine", ["tc-f4", "tc-i8", "m4rm"])
def test_sharded_shards_match_full_product(nccl_group, engine):
    from paper_0811_1714_b200.sharded import mul_sharded, shard_rows
    prev = g.get_engine()
    g.set_engine(engine)
    try:
        m, l, n, world = 3000, 2500, 1800, 4
        full = g.mul_strassen(g.random(m, l, 7), g.random(l, n, 8),
                              g.MulParams(cutoff=512)).to_numpy()
        b = g.random(l, n, 8)
        for rank in range(world):           # emulated ranks, one at a time
            r0, r1 = shard_rows(m, world, rank)
            a_p = g.random(r1 - r0, l, 7, row_base=r0)
            c_p = mul_sharded(a_p, b, g.MulParams(cutoff=512), npanels=3)
            assert np.array_equal(c_p.to_numpy(), full[r0:r1]), rank
    finally:
        g.set_engine(prev)


@pytest.mark.parametrize("pr,pc", [(2, 2), (1, 4), (4, 2)])
def test_grid_blocks_match_full_product(nccl_group, pr, pc):
    """Process grid pr x pc on the device, ranks emulated one at a time in
    the world-of-one NCCL group: rank (i, j) multiplies A's rows_i by the
    owned column block B_j (broadcast inside its column group: here the
    group of one) and must reproduce C[rows_i, cols_j], plain and
    accumulating, ragged right edge included."""
    from paper_0811_1714_b200.sharded import ProcessGrid, mul_sharded_grid
    m, l, n = 2900, 2300, 3001
    world = pr * pc
    params = g.MulParams(cutoff=512)
    a_full, b_full = g.random(m, l, 17), g.random(l, n, 18)
    c0_full = g.random(m, n, 19)
    full = g.mul_strassen(a_full, b_full, params).to_numpy()
    full_acc = full ^ c0_full.to_numpy()
    for rank in range(world):
        grid = ProcessGrid(world, rank, pr, pc)      # no groups: emulated
        (r0, r1), (c0, c1) = grid.rows(m), grid.cols(n)
        if r1 == r0 or c1 == c0:
            continue
        w0, w1 = c0 // 64, c0 // 64 + g.words_per_row(c1 - c0)
        a_blk = g.random(r1 - r0, l, 17, row_base=r0)
        b_blk = g.copy_out(g.window(b_full, 0, c0, l, c1 - c0))
        # src_row=None: this rank's own rows of B_j are the source (in the
        # world of one that is all of them; a grid-row root would name a
        # global rank that does not exist here)
        c_blk = mul_sharded_grid(a_blk, b_blk, grid, params, src_row=None, npanels=3)
        assert np.array_equal(c_blk.to_numpy(), full[r0:r1, w0:w1]), (rank, "plain")
        assert g.trailing_bits_clean(c_blk)
        c_acc = g.copy_out(g.window(c0_full, r0, c0, r1 - r0, c1 - c0))
        mul_sharded_grid(a_blk, b_blk, grid, params, src_row=None, npanels=2, c=c_acc)
        assert np.array_equal(c_acc.to_numpy(), full_acc[r0:r1, w0:w1]), (rank, "acc")


def test_sharded_cfg3_digest(nccl_group, digests):
    from paper_0811_1714_b200.sharded import mul_sharded
    a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
    c = mul_sharded(a, b, npanels=4)
    assert O.digest(c.to_numpy()) == digests["cfg3"]


def test_sharded_rotating_roots_accumulate(nccl_group):
    # src=None: panel i rooted at rank i % world (world 1 here: the same
    # broadcasts, the rotating-root code path); C0 + A.B into a given c
    from paper_0811_1714_b200.sharded import mul_sharded
    m, l, n = 1100, 3000, 900
    a, b = g.random(m, l, 3), g.random(l, n, 4)
    c = g.random(m, n, 5)
    mul_sharded(a, b, g.MulParams(cutoff=512), src=None, npanels=5, c=c)
    want = O.naive_product(O.random(m, l, 3), O.random(l, n, 4)).words ^ \
        O.random(m, n, 5).words
    assert np.array_equal(c.to_numpy(), want)


def test_host_pipeline_products():
    import torch
    from paper_0811_1714_b200.pipeline import HostPipeline
    m, l, n = 1500, 2100, 1300
    pipe = HostPipeline(m, l, n, g.MulParams(cutoff=256))
    ins, outs = [], []
    for i in range(5):
        a = torch.empty((m, g.words_per_row(l)), dtype=torch.int64, pin_memory=True)
        b = torch.empty((l, g.words_per_row(n)), dtype=torch.int64, pin_memory=True)
        av, bv = a.numpy().view(np.uint64), b.numpy().view(np.uint64)
        av[:] = O.random(m, l, 100 + i).words
        bv[:] = O.random(l, n, 200 + i).words
        c = np.zeros((m, g.words_per_row(n)), dtype=np.uint64)
        ins.append((a, b))
        outs.append(c)
        pipe.submit(av, bv, c)
    pipe.sync()
    for i, c in enumerate(outs):
        want = O.naive_product(O.random(m, l, 100 + i), O.random(l, n, 200 + i))
        assert np.array_equal(c, want.words), i


def test_sharded_host_pipeline_products(nccl_group):
    # world 1: this rank owns all of B; the pipeline's stream/event ordering
    # and the per-product broadcast + overwrite of C are what is exercised
    import torch
    from paper_0811_1714_b200.pipeline import ShardedHostPipeline
    m, l, n = 1300, 2200, 1100
    pipe = ShardedHostPipeline(m, l, n, g.MulParams(cutoff=256), npanels=3)
    ins, outs = [], []
    for i in range(5):
        a = torch.empty((m, g.words_per_row(l)), dtype=torch.int64, pin_memory=True)
        b = torch.empty((l, g.words_per_row(n)), dtype=torch.int64, pin_memory=True)
        av, bv = a.numpy().view(np.uint64), b.numpy().view(np.uint64)
        av[:] = O.random(m, l, 300 + i).words
        bv[:] = O.random(l, n, 400 + i).words
        c = np.full((m, g.words_per_row(n)), 7, dtype=np.uint64)
        ins.append((a, b))
        outs.append(c)
        pipe.submit(av, bv, c)
    pipe.sync()
    for i, c in enumerate(outs):
        want = O.naive_product(O.random(m, l, 300 + i), O.random(l, n, 400 + i))
        assert np.array_equal(c, want.words), i
