"""Multi-GPU C += A.B on one 8xB200 box (north_star (e)).

One process per GPU (torch.distributed, NCCL over NVLink 5 / NVSwitch).
C is sharded by row blocks and A is row-sharded the same way, so every rank
computes C_p (+)= A_p . B locally and NO reduction is needed (XOR
accumulation is shard-local). B lives on rank `src` and is broadcast once,
in K-panels: panel i+1 is on the wire (NCCL's stream) while panel i is
multiplied (this rank's stream), so the broadcast hides behind compute.
Bit-exactness across world sizes is automatic: the arithmetic is exact.

Process grid (`ProcessGrid`, pr x pc): rank (i, j) owns the block
C[rows_i, cols_j] = A[rows_i, :] . B[:, cols_j]. The column block B_j is an
owned l x n_j matrix on the pr ranks of column group j and is broadcast
inside that group only, exactly as the whole of B is in the row-sharded
layout -- which is the grid pr x 1. With pc > 1 a rank receives and expands
1/pc of B, and its block is squarer (more Winograd levels survive the
cutoff). Still no reduction: K is never split across ranks.

The plan/pipeline logic is backend-agnostic (tests drive it with gloo on
CPU tensors and an injected local multiply); `mul_sharded` binds it to the
device path.
"""

from __future__ import annotations

from typing import Callable, Sequence

_WORD = 64


def shard_rows(m: int, world: int, rank: int, align: int = _WORD):
    """Row range [r0, r1) of rank `rank`: the `align`-row blocks (so Strassen
    quadrants stay aligned) dealt out as evenly as possible, the first ranks
    taking one extra block; with fewer than `align` rows per rank, a plain
    balanced split."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    if m < align * world:
        per, extra = divmod(m, world)
        r0 = rank * per + min(rank, extra)
        return r0, r0 + per + (1 if rank < extra else 0)
    blocks = -(-m // align)
    per, extra = divmod(blocks, world)
    b0 = rank * per + min(rank, extra)
    b1 = b0 + per + (1 if rank < extra else 0)
    return min(m, b0 * align), min(m, b1 * align)


def shard_cols(n: int, parts: int, j: int, align: int = 2 * _WORD):
    """Column range [c0, c1) of column block j: 128-column (16-byte) aligned
    blocks, so that a block of C or B is a word-aligned window whose rows
    start on the vector boundary of the parent's rows."""
    return shard_rows(n, parts, j, align)


def choose_grid(world: int, m: int, n: int) -> tuple[int, int]:
    """pr x pc = world with the squarest C blocks (m/pr against n/pc). Two
    ranks keep the row-sharded layout; from 4 ranks on a tie goes to more
    COLUMN blocks: a rank then receives and expands less of B (the dearer
    side: it is transposed on the way), measured on one B200 at N = 8 as
    8.6 ms per cfg5 block on 2 x 4 against 10.1 ms on 4 x 2
    (profiles/r02_grid_rank_compute.txt)."""
    best = None
    for pr in range(1, world + 1):
        if world % pr:
            continue
        pc = world // pr
        h, w = -(-m // pr), -(-n // pc)
        key = (max(h, w) / max(1, min(h, w)), pc if world <= 2 else -pc)
        if best is None or key < best[0]:
            best = (key, (pr, pc))
    return best[1]


class ProcessGrid:
    """Ranks laid out row-major on pr x pc: rank = i * pc + j. `col_group`
    (the pr ranks sharing column block j: B_j is broadcast in it) and
    `row_group` (the pc ranks sharing row block i: they hold the same A_i)
    are torch.distributed groups when `make_groups` is set; every rank of
    the world must then construct the grid (new_group is collective)."""

    def __init__(self, world: int, rank: int, pr: int, pc: int,
                 make_groups: bool = False):
        if pr < 1 or pc < 1 or pr * pc != world:
            raise ValueError(f"grid {pr}x{pc} does not cover a world of {world}")
        if not 0 <= rank < world:
            raise ValueError(f"rank {rank} outside world {world}")
        self.world, self.rank, self.pr, self.pc = world, rank, pr, pc
        self.i, self.j = divmod(rank, pc)
        self.col_group = self.row_group = None
        if make_groups and world > 1:
            import torch.distributed as dist
            for j in range(pc):
                grp = dist.new_group(self.col_ranks(j))
                if j == self.j:
                    self.col_group = grp
            for i in range(pr):
                grp = dist.new_group(self.row_ranks(i))
                if i == self.i:
                    self.row_group = grp

    def col_ranks(self, j: int) -> list[int]:
        return [i * self.pc + j for i in range(self.pr)]

    def row_ranks(self, i: int) -> list[int]:
        return [i * self.pc + j for j in range(self.pc)]

    def rows(self, m: int) -> tuple[int, int]:
        return shard_rows(m, self.pr, self.i)

    def cols(self, n: int) -> tuple[int, int]:
        return shard_cols(n, self.pc, self.j)

    def block_of(self, rank: int, m: int, n: int):
        """(r0, r1, c0, c1) of any rank's C block (for gathering)."""
        i, j = divmod(rank, self.pc)
        return shard_rows(m, self.pr, i) + shard_cols(n, self.pc, j)


def k_panels(l: int, npanels: int) -> list[tuple[int, int]]:
    """Split the inner dimension into word-aligned panels [k0, k1)."""
    if l == 0:
        return []
    npanels = max(1, min(npanels, -(-l // _WORD)))
    words = -(-l // _WORD)
    per = -(-words // npanels)
    out = []
    for p in range(npanels):
        k0, k1 = p * per * _WORD, min(l, (p + 1) * per * _WORD)
        if k0 < k1:
            out.append((k0, k1))
    return out


def owned_rows(l: int, world: int, rank: int,
               src: int | None) -> list[tuple[int, int]]:
    """The rows [k0, k1) of B whose contents `rank` must supply: all of B on
    `src`, or with src=None the word-aligned block k_panels(l, world)[rank]
    (B's rows distributed over the ranks, e.g. each rank uploading its block
    from host memory over its own PCIe link)."""
    if src is not None:
        return [(0, l)] if rank == src and l > 0 else []
    blocks = k_panels(l, world)
    return [blocks[rank]] if rank < len(blocks) else []


def pipelined_broadcast(b_rows, panels: Sequence[tuple[int, int]],
                        local_addmul: Callable[[int, int], None],
                        src: int | None = 0, group=None) -> None:
    """Broadcast the rows of `b_rows` (a [l, pitch] tensor; rows = B's rows)
    asynchronously and run local_addmul(k0, k1) for each compute panel as
    soon as its rows have landed. src = a rank: one broadcast per panel from
    it. src = None: one broadcast per rank's block (owned_rows) from that
    rank; a panel waits for every block it overlaps."""
    import torch.distributed as dist
    if not panels:
        return
    if src is None:
        world = dist.get_world_size(group)
        pieces = k_panels(panels[-1][1], world)
        roots = list(range(len(pieces)))
        if group is not None:  # group ranks -> global ranks
            roots = [dist.get_global_rank(group, r) for r in roots]
    else:
        pieces, roots = list(panels), [src] * len(panels)
    works = [dist.broadcast(b_rows[k0:k1], src=r, group=group, async_op=True)
             for (k0, k1), r in zip(pieces, roots)]
    nxt = 0
    for k0, k1 in panels:
        while nxt < len(pieces) and pieces[nxt][0] < k1:
            works[nxt].wait()
            nxt += 1
        local_addmul(k0, k1)


def mul_sharded(a_shard, b, params=None, src: int | None = 0, group=None,
                npanels: int = 2, c=None, accumulate: bool = True):
    """C_p (+)= A_p . B on this rank. `b` is a BitMatrix of B's full shape
    on every rank; its contents matter only on `src` -- or, with src=None,
    only this rank's block of rows (`owned_rows`). If `c` is given the
    product is accumulated into it (addmul) -- or overwrites it with
    accumulate=False -- else a fresh C_p is returned."""
    from .core import BitMatrix, create, window, zero_into
    from .errors import DimensionError
    from .strassen import addmul

    if not isinstance(b, BitMatrix):
        # the broadcast moves whole rows of B's storage; a window's rows
        # would carry (and overwrite) its parent's columns on the receivers
        raise TypeError("mul_sharded broadcasts an owned BitMatrix B "
                        f"(got {type(b).__name__}; copy_out a window first)")
    if a_shard.ncols != b.nrows:
        raise DimensionError(
            f"inner dimensions {a_shard.ncols} and {b.nrows} differ")
    m, l, n = a_shard.nrows, a_shard.ncols, b.ncols
    if c is None:
        c = create(m, n, a_shard.device)
    elif not accumulate:
        zero_into(c)
    panels = k_panels(l, npanels)

    def local(k0: int, k1: int) -> None:
        addmul(c, window(a_shard, 0, k0, m, k1 - k0),
               window(b, k0, 0, k1 - k0, n), params)

    if not panels:
        return c
    pipelined_broadcast(b.storage, panels, local, src=src, group=group)
    return c


def mul_sharded_grid(a_block, b_block, grid: ProcessGrid, params=None,
                     src_row: int | None = None, npanels: int = 2, c=None,
                     accumulate: bool = True):
    """C[rows_i, cols_j] (+)= A[rows_i, :] . B[:, cols_j] on rank (i, j) of
    `grid`. `a_block` holds A's rows_i (every rank of row group i has them:
    generated in place, or gathered with `gather_rows`); `b_block` is the
    owned l x n_j matrix of column block j, filled on grid row `src_row` of
    the column group -- or, with src_row=None, only this rank's block of
    its rows (`owned_rows(l, pr, i, None)`). The broadcast runs inside the
    column group; everything else is `mul_sharded`."""
    src = None if src_row is None else grid.col_ranks(grid.j)[src_row]
    if grid.pr == 1:          # a column group of one: nothing to broadcast
        from .core import create, window, zero_into
        from .strassen import addmul
        m, l, n = a_block.nrows, a_block.ncols, b_block.ncols
        if c is None:
            c = create(m, n, a_block.device)
        elif not accumulate:
            zero_into(c)
        for k0, k1 in k_panels(l, npanels):
            addmul(c, window(a_block, 0, k0, m, k1 - k0),
                   window(b_block, k0, 0, k1 - k0, n), params)
        return c
    return mul_sharded(a_block, b_block, params, src=src, group=grid.col_group,
                       npanels=npanels, c=c, accumulate=accumulate)


def gather_rows(rows_tensor, pieces: Sequence[tuple[int, int]],
                roots: Sequence[int], group=None) -> None:
    """All-gather by rows: piece p = rows [r0, r1) of `rows_tensor` is
    broadcast from global rank roots[p] (each rank of a row group uploads
    1/pc of A_i over its own PCIe link and receives the rest over NVLink)."""
    import torch.distributed as dist
    works = [dist.broadcast(rows_tensor[r0:r1], src=r, group=group, async_op=True)
             for (r0, r1), r in zip(pieces, roots) if r1 > r0]
    for w in works:
        w.wait()


__all__ = ["shard_rows", "shard_cols", "choose_grid", "ProcessGrid", "k_panels",
           "owned_rows", "pipelined_broadcast", "mul_sharded",
           "mul_sharded_grid", "gather_rows"]
