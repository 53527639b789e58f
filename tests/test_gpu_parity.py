"""Parity of the B200 path against the oracle (bit-exact, raw words).

Every test calls through the C ABI (paper_0811_1714_b200 -> libgf2b200.so)
on cuda:0 and compares with the CPU oracle restated from the reference
(oracle/), or with fixtures produced by the reference itself
(tests/golden/). Integer/bit work: the bar is bit-exact, including the
trailing (padding) bits of every row.
"""

import numpy as np
import pytest

from oracle import gf2_oracle as O
from oracle import gf2_port as P

pytestmark = pytest.mark.gpu

g = pytest.importorskip("paper_0811_1714_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    P.set_threads(P.max_threads())


def host(m):
    return O.HostMat(m.nrows, m.ncols, m.to_numpy())


def assert_words(dev, want: np.ndarray, ctx=""):
    got = dev.to_numpy()
    assert got.shape == want.shape, ctx
    if not np.array_equal(got, want):
        bad = np.argwhere(got != want)[0]
        raise AssertionError(f"{ctx}: first differing word at {tuple(bad)}")
    if isinstance(dev, g.BitMatrix):
        assert g.trailing_bits_clean(dev), ctx


# ------------------------------------------------------------- generators
def test_random_matches_reference_kats(golden):
    for key, args in [("kat_random_1x128_s0", (1, 128, 0)),
                      ("kat_random_2x65_s7", (2, 65, 7)),
                      ("kat_random_37x200_s123", (37, 200, 123))]:
        assert_words(g.random(*args), golden[key], key)


@pytest.mark.parametrize("shape", [(1, 1), (3, 63), (7, 64), (65, 65),
                                   (300, 1000), (1024, 1024), (10, 12345)])
def test_random_vs_oracle(shape):
    r, c = shape
    assert_words(g.random(r, c, 99), O.random(r, c, 99).words, str(shape))
    assert_words(g.random(r, c, 5, row_base=17),
                 O.random(r, c, 5, row_base=17).words, "row_base")


def test_bernoulli_vs_oracle():
    t = O.bernoulli_threshold(0.1)
    for (r, c, seed) in [(33, 7001, 41), (5, 65, 3), (70, 12345, 42)]:
        assert_words(g.bernoulli(r, c, seed, threshold=t),
                     O.bernoulli(r, c, seed, t).words, f"{r}x{c}")
    assert_words(g.bernoulli(9, 300, 2, p=0.1, row_base=40),
                 O.bernoulli(9, 300, 2, t, row_base=40).words, "row_base")


# ------------------------------------------------------------- word ops
def test_add_copy_zero_windows_preserve_edges():
    pa, pb, pc = g.random(40, 300, 1), g.random(40, 300, 2), g.random(40, 300, 3)
    ha, hb, hc = pa.to_numpy(), pb.to_numpy(), pc.to_numpy()
    # window at word offset 1, ragged width 150 (2.34 words)
    wa, wb, wc = (g.window(x, 5, 64, 30, 150) for x in (pa, pb, pc))
    g.add_into(wc, wa, wb)
    want = hc.copy()
    tm = np.uint64(O.tail_mask(150))
    seg_a, seg_b = ha[5:35, 1:4], hb[5:35, 1:4]
    want[5:35, 1:3] = seg_a[:, :2] ^ seg_b[:, :2]
    want[5:35, 3] = (hc[5:35, 3] & ~tm) | ((seg_a[:, 2] ^ seg_b[:, 2]) & tm)
    assert np.array_equal(pc.to_numpy(), want)
    g.copy_into(wc, wa)
    want[5:35, 1:3] = seg_a[:, :2]
    want[5:35, 3] = (hc[5:35, 3] & ~tm) | (seg_a[:, 2] & tm)
    assert np.array_equal(pc.to_numpy(), want)
    g.zero_into(wc)
    want[5:35, 1:3] = 0
    want[5:35, 3] = hc[5:35, 3] & ~tm
    assert np.array_equal(pc.to_numpy(), want)
    # aliasing add (out is an operand) and self-inverse
    a = g.random(9, 70, 4)
    g.add_into(a, a, a)
    assert g.equal(a, g.create(9, 70))
    # copy_out masks the tail of a window
    co = g.copy_out(g.window(pb, 0, 0, 3, 70))
    assert g.trailing_bits_clean(co)


def test_equal_first_difference():
    a = g.random(20, 130, 8)
    b = g.copy_out(a)
    assert g.equal(a, b) and a == b
    d = g.from_dense(g.to_dense(a) ^ np.eye(20, 130, k=3, dtype=np.uint8))
    assert not g.equal(a, d)
    assert g.first_difference(a, d) == (0, 3)


def test_host_roundtrip_dense():
    rng = np.random.default_rng(0)
    dense = rng.integers(0, 2, size=(37, 201), dtype=np.uint8)
    m = g.from_dense(dense)
    assert np.array_equal(g.to_dense(m), dense)
    assert np.array_equal(m.to_numpy(), O.pack_dense(dense))


# ------------------------------------------------------------- m4rm
def test_worked_two_by_two():
    # test_m4rm.py:58-62 / test_cubic.py:41-44
    a = g.from_dense([[1, 0], [1, 1]])
    b = g.from_dense([[0, 1], [1, 0]])
    assert g.to_dense(g.mul_m4rm(a, b, 1)).tolist() == [[0, 1], [1, 1]]


def test_identity_products():
    a = g.random(100, 100, 3)
    for k in (1, 4, 8, 16):
        assert g.equal(g.mul_m4rm(a, g.identity(100), k), a)
    i = g.identity(512)
    assert g.equal(g.mul_strassen(i, i, g.MulParams(cutoff=128)), i)


def test_golden_products_all_entry_points(golden):
    for i, m, l, n, sa, sb in golden["prod_cases"].tolist():
        want = golden[f"prod_{i}"]
        a, b = g.random(m, l, sa), g.random(l, n, sb)
        assert_words(g.mul_m4rm(a, b, 8), want, f"m4rm {m,l,n}")
        assert_words(g.mul_m4rm_blocked(a, b, 6, 17), want, "blocked")
        assert_words(g.mul_m4rm_multitable(a, b, 5, 8, 64), want, "multi")
        assert_words(g.mul_strassen(a, b, g.MulParams(cutoff=64)), want,
                     f"strassen {m,l,n}")
        assert_words(g.mul_strassen(a, b), want, "strassen default")


def test_window_operands_golden(golden):
    pa, pb = g.random(90, 640, 77), g.random(700, 512, 78)
    aw = g.window(pa, 5, 64, 70, 385)      # odd word offset, ragged
    bw = g.window(pb, 11, 192, 385, 250)   # odd word offset, ragged
    assert_words(g.mul_m4rm(aw, bw, 8), golden["win_product"], "m4rm win")
    assert_words(g.mul_strassen(aw, bw, g.MulParams(cutoff=64)),
                 golden["win_product"], "strassen win")
    pc = g.random(80, 512, 79)
    assert np.array_equal(pc.to_numpy(), golden["win_accum_parent_before"])
    g.addmul(g.window(pc, 3, 64, 70, 250), aw, bw, g.MulParams(cutoff=64))
    assert np.array_equal(pc.to_numpy(), golden["win_accum_parent"])


def test_mul_m4rm_into_golden(golden):
    a, b, c = g.random(150, 333, 91), g.random(333, 200, 92), \
        g.random(150, 200, 93)
    g.mul_m4rm_into(c, a, b, 8, 64, 4)
    assert_words(c, golden["into_result"], "into")


def test_random_triples_vs_oracle():
    # shape sweep like test_m4rm.py:141-157 / test_acceptance.py:40-70
    rng = np.random.default_rng(20260101)
    for trial in range(60):
        m, l, n = (int(x) for x in rng.integers(1, 1025, 3))
        a, b = g.random(m, l, trial * 7 + 1), g.random(l, n, trial * 7 + 2)
        want = O.naive_product(O.random(m, l, trial * 7 + 1),
                               O.random(l, n, trial * 7 + 2)).words
        assert_words(g.mul_m4rm(a, b, 8), want, f"m4rm {m,l,n}")
        assert_words(g.mul_strassen(a, b, g.MulParams(cutoff=128)), want,
                     f"strassen {m,l,n}")


@pytest.mark.parametrize("mln", [(1, 5000, 1), (2, 20000, 3), (64, 9000, 64),
                                 (700, 3000, 40), (5, 64, 70000),
                                 (3000, 1, 3000), (1, 1, 1)])
def test_edge_shapes_and_split_k(mln):
    m, l, n = mln
    a, b = g.random(m, l, 11), g.random(l, n, 12)
    want = P.mul_strassen(O.random(m, l, 11), O.random(l, n, 12), cutoff=64)
    assert_words(g.mul_m4rm(a, b, 8), want.words, str(mln))
    c0 = g.random(m, n, 13)
    g.mul_m4rm_into(c0, a, b, 8)
    want_acc = O.random(m, n, 13).words ^ want.words
    assert_words(c0, want_acc, "into " + str(mln))


def test_empty_and_degenerate():
    c = g.mul_m4rm(g.create(0, 5), g.create(5, 7), 3)
    assert c.shape == (0, 7)
    c = g.mul_m4rm(g.random(4, 0, 1), g.create(0, 7), 3)
    assert g.equal(c, g.create(4, 7))
    z = g.mul_strassen(g.create(4, 0), g.create(0, 7))
    assert g.equal(z, g.create(4, 7))
    assert g.mul_strassen(g.create(0, 5), g.create(5, 7)).shape == (0, 7)
    c = g.random(4, 7, 2)
    before = c.to_numpy()
    g.mul_m4rm_into(c, g.random(4, 0, 1), g.create(0, 7), 2)
    assert np.array_equal(c.to_numpy(), before)


def test_errors_match_reference():
    a = g.create(2, 3)
    with pytest.raises(g.DimensionError):
        g.mul_m4rm(a, g.create(4, 2), 4)
    with pytest.raises(g.ParameterError):
        g.mul_m4rm(g.create(2, 2), g.create(2, 2), 0)
    with pytest.raises(g.ParameterError):
        g.mul_m4rm(g.create(2, 2), g.create(2, 2), 17)
    with pytest.raises(g.ParameterError):
        g.mul_m4rm_multitable(g.create(2, 2), g.create(2, 2), 1, 9, 2)
    with pytest.raises(g.DimensionError):
        g.mul_strassen(g.create(2, 3), g.create(4, 2))
    with pytest.raises(AssertionError):
        p = g.create(8, 64)
        g.mul_m4rm_into(g.window(p, 0, 0, 8, 8), g.create(8, 8),
                        g.create(8, 8), 2)
    with pytest.raises(g.AlignmentError):
        g.window(g.create(4, 200), 0, 3, 2, 10)
    with pytest.raises(g.DimensionError):
        g.window(g.create(4, 200), 0, 64, 2, 200)
    with pytest.raises(g.DimensionError):
        g.add(g.create(2, 3), g.create(3, 2))
    with pytest.raises(g.ParameterError):
        g.MulParams(cutoff=32)
    # product target aliasing an operand is refused
    x = g.random(64, 64, 1)
    with pytest.raises(g.ParameterError):
        g.mul_m4rm_into(x, x, g.random(64, 64, 2), 8)


@pytest.fixture(params=["tc-f4", "m4rm"])
def engine(request):
    """tc-f4 (default: Winograd levels whose leaves would be shallower than
    2048 fold into direct products) and m4rm (the recursion at exactly the
    caller's cutoff, M4RM leaves and peel fix-ups, as the reference runs)."""
    prev = g.get_engine()
    g.set_engine(request.param)
    yield request.param
    g.set_engine(prev)


def test_peeling_pattern(engine):
    # test_strassen.py:175-180 (n = 2^10 - 1, 2^10, 2^10 + 1)
    for n in (1023, 1024, 1025):
        a, b = g.random(n, n, n), g.random(n, n, n + 1)
        want = O.naive_product(O.random(n, n, n), O.random(n, n, n + 1))
        assert_words(g.mul_strassen(a, b, g.MulParams(cutoff=128)),
                     want.words, str(n))


def test_strassen_random_triples_vs_port(engine):
    # test_strassen.py:207-216 shape range, deeper recursion via cutoff 64
    rng = np.random.default_rng(27)
    for trial in range(40):
        m, l, n = (int(x) for x in rng.integers(1, 2500, 3))
        a, b = g.random(m, l, trial + 3000), g.random(l, n, trial + 4000)
        want = P.mul_strassen(O.random(m, l, trial + 3000),
                              O.random(l, n, trial + 4000), cutoff=512)
        assert_words(g.mul_strassen(a, b, g.MulParams(cutoff=64)), want.words,
                     f"{m,l,n}")


def test_tensor_engine_folds_shallow_levels():
    """With a tensor engine, a cutoff whose leaves would be shallower than
    2048 does not buy Winograd levels: 1500^3 at cutoff 64
    runs as one product (a handful of launches) instead of a depth-4
    recursion; the m4rm engine keeps the reference's exact recursion. Same
    words either way."""
    a, b = g.random(1500, 1500, 1), g.random(1500, 1500, 2)
    p = g.MulParams(cutoff=64)
    prev = g.get_engine()
    try:
        g.set_engine("tc-f4")
        n0 = g.launch_count()
        c1 = g.mul_strassen(a, b, p)
        folded = g.launch_count() - n0
        g.set_engine("m4rm")
        n0 = g.launch_count()
        c2 = g.mul_strassen(a, b, p)
        exact = g.launch_count() - n0
    finally:
        g.set_engine(prev)
    assert folded <= 4 < exact
    assert g.equal(c1, c2)


def test_algebraic_laws():
    # test_acceptance.py:207-239: distributivity, associativity, transpose-free
    a, b, c = g.random(300, 500, 1), g.random(500, 400, 2), g.random(500, 400, 3)
    lhs = g.mul_strassen(a, g.add(b, c), g.MulParams(cutoff=64))
    rhs = g.add(g.mul_m4rm(a, b, 8), g.mul_m4rm(a, c, 8))
    assert g.equal(lhs, rhs)
    d = g.random(400, 200, 4)
    assert g.equal(g.mul_m4rm(g.mul_m4rm(a, b, 8), d, 8),
                   g.mul_m4rm(a, g.mul_m4rm(b, d, 8), 8))


# ------------------------------------------------------------- configs
def test_cfg1_digest(digests):
    a, b = g.random(1024, 1024, 11), g.random(1024, 1024, 12)
    assert O.digest(g.mul_m4rm(a, b, 8).to_numpy()) == digests["cfg1"]


def test_cfg2_digest(digests):
    a, b = g.random(4096, 4096, 21), g.random(4096, 4096, 22)
    c = g.mul_strassen(a, b, g.MulParams(cutoff=1024, k=8))
    assert O.digest(c.to_numpy()) == digests["cfg2"]
    assert g.trailing_bits_clean(c)


def test_cfg3_digest(digests):
    a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
    for params in (None, g.MulParams(), g.MulParams(cutoff=8192)):
        c = g.mul_strassen(a, b, params)
        assert O.digest(c.to_numpy()) == digests["cfg3"], params


def test_cfg4_digests(digests):
    t = O.bernoulli_threshold(0.1)
    a = g.bernoulli(10000, 7001, 41, threshold=t)
    b = g.bernoulli(7001, 12345, 42, threshold=t)
    c = g.mul_strassen(a, b)
    assert O.digest(c.to_numpy()) == digests["cfg4_product"]
    assert g.trailing_bits_clean(c)
    c0 = g.random(10000, 12345, 43)
    g.mul_m4rm_into(c0, a, b, 8, 512, 8)
    assert O.digest(c0.to_numpy()) == digests["cfg4_addmul"]
    c1 = g.random(10000, 12345, 43)
    g.addmul(c1, a, b)
    assert O.digest(c1.to_numpy()) == digests["cfg4_addmul"]
    assert g.trailing_bits_clean(c1)


def _freivalds(c, a, b, seed=7, reps=2):
    """C.X == A.(B.X) for random 64-column X: a size-independent check
    computed by the narrow (single-word) kernel path."""
    for r in range(reps):
        x = g.random(b.ncols, 64, seed + r)
        lhs = g.mul_m4rm(c, x, 8)
        rhs = g.mul_m4rm(a, g.mul_m4rm(b, x, 8), 8)
        if not g.equal(lhs, rhs):
            return False
    return True


def test_cfg5_addmul_digest(digests):
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < 16 << 30:
        pytest.skip("needs ~16 GB of free HBM")
    n = 65536
    a, b = g.random(n, n, 51), g.random(n, n, 52)
    c = g.mul_strassen(a, b)
    assert _freivalds(c, a, b)
    assert O.digest(c.to_numpy()) == digests["cfg5_product"]
    del c
    c0 = g.random(n, n, 53)
    g.addmul(c0, a, b)
    assert O.digest(c0.to_numpy()) == digests["cfg5_addmul"]
    # depth 1 with 32768^3 leaves: the tensor-core leaf launch splits K into
    # 8192-entry chunks while fusing the post-addition into C (red.xor)
    c0 = g.random(n, n, 53)
    g.addmul(c0, a, b, g.MulParams(cutoff=32768, k=8))
    assert O.digest(c0.to_numpy()) == digests["cfg5_addmul"]


def test_max_size_engines_agree():
    """Beyond cfg5 (the largest shapes one B200 holds comfortably, run by
    tools/max_size.py at 131072^3): here 98304 x 81920 x 90112 with a ragged
    twin, where the oracle cannot follow -- the tensor-core recursion and the
    M4RM engine (independent kernels) must agree bit for bit, and the result
    must pass Freivalds through a third path (one-word M4RM tiles)."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < 100 << 30:
        pytest.skip("needs ~100 GB of free HBM")
    prev = g.get_engine()
    try:
        for m, l, n in ((98304, 81920, 90112), (70001, 65537, 66003)):
            a, b = g.random(m, l, 81), g.random(l, n, 82)
            g.set_engine("tc-f4")
            c1 = g.mul_strassen(a, b)
            g.release_workspace()
            g.set_engine("m4rm")
            c2 = g.mul_strassen(a, b)
            g.release_workspace()
            g.set_engine("tc-f4")
            assert g.equal(c1, c2), (m, l, n)
            assert g.trailing_bits_clean(c1)
            assert _freivalds(c1, a, b)
            del a, b, c1, c2
    finally:
        g.set_engine(prev)
        g.release_workspace()


def test_freivalds_detects_fault():
    a, b = g.random(2048, 2048, 1), g.random(2048, 2048, 2)
    c = g.mul_strassen(a, b)
    assert _freivalds(c, a, b)
    d = g.to_dense(g.window(c, 0, 0, 1, 64))
    d[0, 0] ^= 1  # --inject-fault analogue (cli.py:199-200)
    g.copy_into(g.window(c, 0, 0, 1, 64), g.from_dense(d))
    assert not _freivalds(c, a, b)


def test_native_code_is_what_runs():
    before = g.launch_count()
    g.mul_m4rm(g.random(64, 64, 1), g.random(64, 64, 2), 8)
    assert g.launch_count() > before


M4RM_GEOM_CASE = r"""
import sys; sys.path.insert(0, %(root)r)
import numpy as np
import paper_0811_1714_b200 as g
from oracle import gf2_oracle as O
from oracle import gf2_port as P
P.set_threads(P.max_threads())
bad = []
for (m, l, n, seed) in [(1000, 1100, 1300, 1), (130, 2049, 777, 2), (2100, 640, 1024, 3), (64, 70, 65, 4)]:
    pa, pb = O.random(m, l, seed), O.random(l, n, seed + 100)
    want = P.mul_strassen(pa, pb, cutoff=1 << 20).words
    a, b = g.random(m, l, seed), g.random(l, n, seed + 100)
    if not np.array_equal(g.mul_m4rm(a, b, 8).to_numpy(), want):
        bad.append(("aligned", m, l, n))
    # odd word offsets: 8-byte staging instead of TMA
    big_a, big_b = g.random(m + 3, l + 128, seed + 7), g.random(l + 5, n + 128, seed + 8)
    aw, bw = g.window(big_a, 3, 64, m, l), g.window(big_b, 5, 64, l, n)
    ha, hb = big_a.to_numpy(), big_b.to_numpy()
    wa = O.HostMat(m, l, np.ascontiguousarray(ha[3:3 + m, 1:1 + O.words_per_row(l)]))
    wb = O.HostMat(l, n, np.ascontiguousarray(hb[5:5 + l, 1:1 + O.words_per_row(n)]))
    wa.words[:, -1] &= np.uint64(O.tail_mask(l))
    wb.words[:, -1] &= np.uint64(O.tail_mask(n))
    want_w = P.mul_strassen(wa, wb, cutoff=1 << 20).words
    c = g.random(m, n, seed + 9)
    c0 = c.to_numpy().copy()
    g.mul_m4rm_into(c, aw, bw, 8)
    if not np.array_equal(c.to_numpy(), c0 ^ want_w):
        bad.append(("window-accumulate", m, l, n))
    # mixed staging: A 16-byte aligned (TMA) with B at an odd word (8-byte
    # B loads), and A at an odd word with B aligned (16-byte B loads)
    aw2, bw2 = g.window(big_a, 3, 128, m, l), g.window(big_b, 5, 128, l, n)
    wa2 = O.HostMat(m, l, np.ascontiguousarray(ha[3:3 + m, 2:2 + O.words_per_row(l)]))
    wb2 = O.HostMat(l, n, np.ascontiguousarray(hb[5:5 + l, 2:2 + O.words_per_row(n)]))
    wa2.words[:, -1] &= np.uint64(O.tail_mask(l))
    wb2.words[:, -1] &= np.uint64(O.tail_mask(n))
    if not np.array_equal(g.mul_m4rm(aw2, bw, 8).to_numpy(), P.mul_strassen(wa2, wb, cutoff=1 << 20).words):
        bad.append(("tma-a/odd-b", m, l, n))
    if not np.array_equal(g.mul_m4rm(aw, bw2, 8).to_numpy(), P.mul_strassen(wa, wb2, cutoff=1 << 20).words):
        bad.append(("odd-a/aligned-b", m, l, n))
print("BAD", bad)
"""


@pytest.mark.parametrize("geom", ["16,1", "16,5", "12,2", "8,1", "8,3", "4,5", "2,16", "1,8", "1,16"])
def test_m4rm_every_geometry(geom):
    """Every k_m4rm tile height (RPT 16/12/8 -> 8192/6144/4096 rows with TMEM-parked groups, 4/2/1 -> 2048/1024/512) and
    K-split count, forced through GF2_M4RM_GEOM (read once per process,
    hence a subprocess), on ragged shapes with the TMA path (aligned
    operands), the 8-byte cp.async path (odd word offsets) and both mixes,
    plain and accumulating, against the C port."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GF2_M4RM_GEOM=geom)
    out = subprocess.run([sys.executable, "-c", M4RM_GEOM_CASE % {"root": root}], env=env,
                         cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "BAD []", out.stdout[-2000:]
