"""The drop-in surface beyond the multiply entries, on the device, against
fixtures generated from the reference (tests/golden/make_golden.py --api):
schedule_winograd (call order, result and scratch contents after the 22
steps), peel_fixup, make_table / CombinationTable, plus the mul_m4rm*
dispatch, the device guard and the owned-copy tail mask."""

import os

import numpy as np
import pytest

from oracle import gf2_oracle as O

pytestmark = pytest.mark.gpu
g = pytest.importorskip("paper_0811_1714_b200")
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return np.load(os.path.join(HERE, "golden", "golden_api.npz"))


def _upload(words, ncols):
    return g.from_numpy(np.ascontiguousarray(words, dtype=np.uint64), ncols)


def test_schedule_winograd_matches_reference(api):
    for i, (m, l, n, sa, sb, m2, l2, n2) in enumerate(api["sched_cases"].tolist()):
        a, b = g.random(m, l, sa), g.random(l, n, sb)
        c = g.random(m, n, 100 + i)
        x, y = g.random(m2, max(l2, n2), 200 + i), g.random(l2, n2, 300 + i)
        a0, b0 = a.to_numpy().copy(), b.to_numpy().copy()
        names = {id(c): 0, id(x): 1, id(a): 2, id(b): 3, id(y): 4}
        calls = []

        def mult(cc, aa, bb):
            rec = []
            for w in (cc, aa, bb):
                p = w.parent if isinstance(w, g.MatrixWindow) else w
                ro = w.row_offset if isinstance(w, g.MatrixWindow) else 0
                co = w.col_offset if isinstance(w, g.MatrixWindow) else 0
                rec += [names[id(p)], ro, co, w.nrows, w.ncols]
            calls.append(rec)
            g.copy_into(cc, g.mul_cubic(aa, bb))

        g.schedule_winograd(a, b, c, (x, y), mult)
        assert calls == api[f"sched{i}_calls"].tolist()
        assert np.array_equal(c.to_numpy(), api[f"sched{i}_c"])
        assert np.array_equal(x.to_numpy(), api[f"sched{i}_x"])
        assert np.array_equal(y.to_numpy(), api[f"sched{i}_y"])
        assert np.array_equal(a.to_numpy(), a0) and np.array_equal(b.to_numpy(), b0)


def test_schedule_winograd_device_multiplier_and_errors():
    """A device multiplier (mul_direct on the tensor engine) on quadrant
    windows of an offset window, and the reference's shape errors."""
    big_a, big_b = g.random(600, 700, 1), g.random(700, 600, 2)
    a = g.window(big_a, 3, 64, 512, 512)
    b = g.window(big_b, 5, 128, 512, 384)
    c = g.create(512, 384)
    x, y = g.create(256, 256), g.create(256, 192)
    g.schedule_winograd(a, b, c, (x, y), lambda cc, aa, bb: g.copy_into(cc, g.mul_direct(aa, bb)))
    want = O.naive_product(O.HostMat(512, 512, g.copy_out(a).to_numpy()),
                           O.HostMat(512, 384, g.copy_out(b).to_numpy()))
    assert np.array_equal(c.to_numpy(), want.words)
    with pytest.raises(g.DimensionError):
        g.schedule_winograd(g.random(127, 128, 8), g.random(128, 128, 9), g.create(127, 128),
                            (g.create(64, 64), g.create(64, 64)), lambda *a: None)
    with pytest.raises(g.DimensionError):
        g.schedule_winograd(g.random(128, 128, 8), g.random(128, 128, 9), g.create(128, 64),
                            (g.create(64, 64), g.create(64, 64)), lambda *a: None)


def test_peel_fixup_matches_reference(api):
    for i, (m, l, n, sa, sb, m2, l2, n2) in enumerate(api["peel_cases"].tolist()):
        a, b = g.random(m, l, sa), g.random(l, n, sb)
        c = _upload(api[f"peel{i}_before"], n)
        g.peel_fixup(c, a, b, m2, l2, n2, g.MulParams(cutoff=64))
        assert np.array_equal(c.to_numpy(), api[f"peel{i}_c"]), i
        assert g.trailing_bits_clean(c)
    a = g.random(10, 10, 20)
    with pytest.raises(g.DimensionError):
        g.peel_fixup(g.create(10, 10), a, a, 11, 10, 10, g.MulParams(cutoff=64))
    with pytest.raises(g.DimensionError):
        g.peel_fixup(g.create(10, 11), a, a, 10, 10, 10)


def test_peel_fixup_after_device_strassen():
    """peel_fixup completing a device-computed block of a peeled shape
    (the reference's own composition: recursion on the block, then fix-ups)."""
    m, l, n = 1100, 1030, 1500
    ps = g.peel_split(m, l, n, 256)
    a, b = g.random(m, l, 5), g.random(l, n, 6)
    c = g.random(m, n, 7)
    g.copy_into(g.window(c, 0, 0, ps.m, ps.n),
                g.mul_strassen(g.window(a, 0, 0, ps.m, ps.l), g.window(b, 0, 0, ps.l, ps.n),
                               g.MulParams(cutoff=256)))
    g.peel_fixup(c, a, b, ps.m, ps.l, ps.n)
    want = O.naive_product(O.random(m, l, 5), O.random(l, n, 6))
    assert np.array_equal(c.to_numpy(), want.words)


def test_make_table_matches_reference(api, golden):
    parent = g.random(6, 192, 8)
    t = g.CombinationTable(4, 70)
    g.make_table(g.window(parent, 0, 64, 6, 70), 1, 4, t)
    assert np.array_equal(t.matrix.to_numpy(), api["table_win_k4"])
    assert g.trailing_bits_clean(t.matrix)
    b = g.random(8, 64, 6)
    t = g.CombinationTable(8, 64)
    g.make_table(b, 0, 8, t)
    g.make_table(b, 0, 3, t)
    assert t.k == 3 and tuple(t.rows.shape) == (8, 1)
    assert np.array_equal(t.matrix.to_numpy(), api["table_refill_matrix"])
    pb = g.random(40, 1000, 9)
    t = g.CombinationTable(12, 777)
    g.make_table(g.window(pb, 5, 128, 20, 777), 3, 12, t)
    assert np.array_equal(t.matrix.to_numpy(), api["table_win_k12"])
    # the round-1 fixtures: k = 3 and 8 from a window at word offset 1
    pb = g.random(40, 256, 5)
    w = g.window(pb, 3, 64, 9, 130)
    for k in (3, 8):
        t = g.CombinationTable(k, 130)
        g.make_table(w, 1, k, t)
        assert np.array_equal(t.matrix.to_numpy()[:1 << k], golden[f"table_k{k}"])
        assert not t.matrix.to_numpy()[0].any()


def test_make_table_k16_linearity_and_errors():
    b = g.random(20, 300, 11)
    t = g.CombinationTable(16, 300)
    g.make_table(b, 2, 16, t)
    tab = t.matrix.to_numpy()
    src = b.to_numpy()[2:18]
    rng = np.random.default_rng(3)
    for _ in range(200):
        x, y = (int(v) for v in rng.integers(0, 1 << 16, 2))
        assert np.array_equal(tab[x ^ y], tab[x] ^ tab[y])
    for i in range(16):   # unit slots are the source rows (big-endian)
        assert np.array_equal(tab[1 << (15 - i)], src[i])
    bb = g.random(4, 50, 9)
    t = g.CombinationTable(4, 50)
    with pytest.raises(g.DimensionError):
        g.make_table(bb, 2, 4, t)
    with pytest.raises(g.DimensionError):
        g.make_table(g.random(4, 51, 10), 0, 4, t)
    with pytest.raises(g.ParameterError):
        g.make_table(bb, 0, 5, t)
    with pytest.raises(g.ParameterError):
        g.CombinationTable(17, 50)


def test_mul_m4rm_dispatch():
    """mul_m4rm* products past the crossover run on the tensor engine (no
    M4RM launch), small ones on the M4RM kernel; set_engine("m4rm") forces
    the M4RM kernel. Same words either way."""
    from paper_0811_1714_b200 import _lib
    prev = g.get_engine()
    try:
        g.set_engine("tc-f4")
        a, b = g.random(2048, 2048, 1), g.random(2048, 4096, 2)
        k0, n0 = _lib.m4rm_launch_count(), g.launch_count()
        c_tc = g.mul_m4rm(a, b, 8)
        assert _lib.m4rm_launch_count() == k0 and g.launch_count() - n0 >= 3
        s1, s2 = g.random(200, 300, 3), g.random(300, 100, 4)
        k0 = _lib.m4rm_launch_count()
        g.mul_m4rm(s1, s2, 8)
        assert _lib.m4rm_launch_count() - k0 == 1
        g.set_engine("m4rm")
        k0 = _lib.m4rm_launch_count()
        c_m = g.mul_m4rm(a, b, 8)
        assert _lib.m4rm_launch_count() - k0 == 1
        assert np.array_equal(c_tc.to_numpy(), c_m.to_numpy())
        c0 = g.random(2048, 4096, 5)
        c1 = g.copy_out(c0)
        g.set_engine("tc-f4")
        g.mul_m4rm_into(c1, a, b, 8, 512, 8)
        assert np.array_equal(c1.to_numpy(), c0.to_numpy() ^ c_m.to_numpy())
    finally:
        g.set_engine(prev)


def test_device_guard(monkeypatch):
    """Operations refuse matrices of another device than the current one
    (they would launch device-1 pointers on device 0)."""
    from paper_0811_1714_b200 import core
    a = g.random(64, 64, 1)
    monkeypatch.setattr(core, "_cur_dev", lambda: 1)
    with pytest.raises(g.DimensionError, match="current device"):
        g.add(a, a)
    with pytest.raises(g.DimensionError, match="current device"):
        g.mul_strassen(a, a)
    with pytest.raises(g.DimensionError, match="current device"):
        a.to_numpy()


def test_to_host_masks_window_tail():
    parent = g.random(20, 130, 3)
    w = g.window(parent, 2, 0, 10, 66)       # right edge mid-parent, live bits beyond
    h = w.to_host()
    words = np.asarray(h.words)
    assert words.shape == (10, 2)
    assert not (words[:, -1] & np.uint64(~g.tail_mask(66) & 0xFFFFFFFFFFFFFFFF)).any()
    assert np.array_equal(g.from_host(h).to_numpy(), g.copy_out(w).to_numpy())
