"""Device transpose / augment / stack / mul_cubic and GF2M file I/O against
fixtures produced by the reference (tests/golden) and the oracle."""

import numpy as np
import pytest

from oracle import gf2_oracle as O

pytestmark = pytest.mark.gpu
g = pytest.importorskip("paper_0811_1714_b200")


@pytest.fixture(autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_reference_fixtures(golden):
    a, b = g.random(70, 130, 61), g.random(70, 77, 62)
    assert np.array_equal(g.augment(a, b).to_numpy(), golden["augment_ragged"])
    assert np.array_equal(g.augment(g.random(70, 128, 63), b).to_numpy(),
                          golden["augment_aligned"])
    assert np.array_equal(g.stack(g.random(30, 130, 64), g.random(41, 130, 65)).to_numpy(),
                          golden["stack"])
    t = g.transpose(a)
    assert np.array_equal(t.to_numpy(), golden["transpose_70x130"])
    assert g.trailing_bits_clean(t)
    c = g.mul_cubic(g.random(200, 300, 66), g.random(300, 57, 67))
    assert np.array_equal(c.to_numpy(), golden["cubic_200x300x57"])


@pytest.mark.parametrize("shape", [(1, 1), (64, 64), (65, 63), (300, 1000),
                                   (1000, 130), (4096, 4096)])
def test_transpose_vs_dense(shape):
    r, c = shape
    a = g.random(r, c, 5)
    dense = O.unpack(O.random(r, c, 5))
    assert np.array_equal(g.to_dense(g.transpose(a)), dense.T)
    assert g.equal(g.transpose(g.transpose(a)), a)


def test_transpose_window_and_law():
    p = g.random(300, 700, 8)
    w = g.window(p, 7, 128, 200, 333)
    assert np.array_equal(g.to_dense(g.transpose(w)), g.to_dense(w).T)
    # acceptance criterion 8 (test_acceptance.py:224-227): (AB)^T = B^T A^T
    a, b = g.random(300, 500, 1), g.random(500, 200, 2)
    assert g.equal(g.transpose(g.mul_strassen(a, b, g.MulParams(cutoff=64))),
                   g.mul_m4rm(g.transpose(b), g.transpose(a), 8))


def test_augment_stack_offsets():
    rng = np.random.default_rng(3)
    for _ in range(20):
        r = int(rng.integers(1, 60))
        ca, cb = (int(x) for x in rng.integers(1, 300, 2))
        a, b = g.random(r, ca, 1), g.random(r, cb, 2)
        want = np.hstack([g.to_dense(a), g.to_dense(b)])
        got = g.augment(a, b)
        assert np.array_equal(g.to_dense(got), want), (r, ca, cb)
        assert g.trailing_bits_clean(got)
        s = g.stack(g.random(r, ca, 3), g.random(r + 1, ca, 4))
        assert np.array_equal(g.to_dense(s), np.vstack([g.to_dense(g.random(r, ca, 3)),
                                                        g.to_dense(g.random(r + 1, ca, 4))]))
    with pytest.raises(g.DimensionError):
        g.augment(g.create(2, 3), g.create(3, 3))
    with pytest.raises(g.DimensionError):
        g.stack(g.create(2, 3), g.create(2, 4))


def test_mul_cubic_vs_oracle():
    for (m, l, n) in [(1, 1, 1), (9984, 701, 57), (100, 7001, 63), (64, 64, 200)]:
        a, b = g.random(m, l, 11), g.random(l, n, 12)
        want = O.naive_product(O.random(m, l, 11), O.random(l, n, 12)).words
        assert np.array_equal(g.mul_cubic(a, b).to_numpy(), want), (m, l, n)


def test_gf2m_roundtrip_and_reference_bytes(golden, tmp_path):
    fp = tmp_path / "m.gf2m"
    g.save(g.random(37, 200, 5), fp)
    assert np.array_equal(np.frombuffer(fp.read_bytes(), dtype=np.uint8),
                          golden["gf2m_37x200_s5"])
    g.save(g.window(g.random(9, 300, 6), 2, 64, 5, 130), fp)
    assert np.array_equal(np.frombuffer(fp.read_bytes(), dtype=np.uint8),
                          golden["gf2m_window"])
    fp.write_bytes(golden["gf2m_37x200_s5"].tobytes())
    m = g.load(fp)
    assert g.equal(m, g.random(37, 200, 5)) and m.shape == (37, 200)
    big = g.random(3000, 4097, 9)
    g.save(big, fp)
    assert g.equal(g.load(fp), big)


def test_to_host_returns_reference_matrix_when_gf2mat_is_imported(monkeypatch):
    """to_host() hands back the reference's own BitMatrix type
    when the caller has gf2mat imported (stand-in module here: the
    reference is not present on the GPU box), else a HostMatrix."""
    import sys
    import types

    class StubBitMatrix:  # the reference's constructor shape (core.py:71-80)
        def __init__(self, nrows, ncols):
            self.nrows, self.ncols = nrows, ncols
            self.width = (ncols + 63) // 64
            self.data = np.zeros(nrows * self.width, dtype=np.uint64)
            self.words = self.data.reshape(nrows, self.width)

    stub = types.ModuleType("gf2mat")
    stub.create = StubBitMatrix
    monkeypatch.setitem(sys.modules, "gf2mat", stub)
    a = g.random(100, 130, 5)
    h = a.to_host()
    assert isinstance(h, StubBitMatrix)
    assert np.array_equal(h.words, a.to_numpy())
    w = g.window(a, 3, 64, 50, 66)
    hw = w.to_host()
    assert isinstance(hw, StubBitMatrix) and np.array_equal(hw.words, w.to_numpy())
    monkeypatch.delitem(sys.modules, "gf2mat")
    assert isinstance(a.to_host(), g.HostMatrix)


def test_release_workspace_returns_pool_memory():
    """gf2_release_workspace: the stream-ordered pool's cached workspace goes
    back to the system and later products still run."""
    import torch
    a, b = g.random(8192, 8192, 1), g.random(8192, 8192, 2)
    c = g.mul_strassen(a, b, g.MulParams(cutoff=4096))
    torch.cuda.synchronize()
    before = torch.cuda.mem_get_info()[0]
    g.release_workspace()
    after = torch.cuda.mem_get_info()[0]
    assert after >= before
    assert g.equal(g.mul_strassen(a, b, g.MulParams(cutoff=4096)), c)
