"""Property-based checks of the host-side logic (CPU only): the native
peel_split against the oracle's restatement of strassen.py:66-84 (itself
pinned to the reference's KATs in test_oracle.py), and the multi-GPU
planning helpers' partition invariants."""

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import gf2_oracle as O
from paper_0811_1714_b200 import peel_split
from paper_0811_1714_b200.sharded import k_panels, owned_rows, shard_rows

dims = st.one_of(st.integers(1, 300), st.integers(1, 70000),
                 st.integers(1, 1100).map(lambda k: 64 * k),
                 st.integers(1, 1100).map(lambda k: 64 * k + 1))


@settings(max_examples=400, deadline=None)
@given(m=dims, l=dims, n=dims, cutoff=st.sampled_from([64, 128, 256, 1000, 1024, 2048, 4096, 8192]))
def test_native_peel_split_matches_oracle(m, l, n, cutoff):
    ps, want = peel_split(m, l, n, cutoff), O.peel_split(m, l, n, cutoff)
    assert (ps.m, ps.l, ps.n, ps.depth) == (want.m, want.l, want.n, want.depth)


@settings(max_examples=300, deadline=None)
@given(m=st.integers(0, 200000), world=st.integers(1, 16))
def test_shard_rows_partitions_every_row(m, world):
    spans = [shard_rows(m, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == m
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0 and a0 <= a1 and b0 <= b1
    if m >= 64 * world:
        assert all(r0 % 64 == 0 for r0, _ in spans)


@settings(max_examples=300, deadline=None)
@given(l=st.integers(0, 100000), npanels=st.integers(1, 64))
def test_k_panels_tile_k_on_word_boundaries(l, npanels):
    ps = k_panels(l, npanels)
    if l == 0:
        assert ps == []
        return
    assert ps[0][0] == 0 and ps[-1][1] == l and len(ps) <= npanels
    for (a0, a1), (b0, b1) in zip(ps, ps[1:]):
        assert a1 == b0 and a0 < a1
    assert all(k0 % 64 == 0 for k0, _ in ps)


@settings(max_examples=300, deadline=None)
@given(l=st.integers(0, 70000), world=st.integers(1, 8),
       src=st.one_of(st.none(), st.integers(0, 7)))
def test_owned_rows_partition_b(l, world, src):
    if src is not None and src >= world:
        src = world - 1
    owned = [owned_rows(l, world, r, src) for r in range(world)]
    spans = sorted(p for o in owned for p in o)
    assert spans == (k_panels(l, world) if src is None else ([(0, l)] if l else []))
    if src is not None:
        assert all(not o for r, o in enumerate(owned) if r != src)


def test_shard_rows_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard_rows(100, 4, 4)
