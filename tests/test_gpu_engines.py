"""Parity of the tcgen05 tensor-core engines (kind::i8, kind::f8f6f4, kind::mxf4) with
the oracle: the same product as M4RM, bit-exact including trailing bits."""

import numpy as np
import pytest

from oracle import gf2_oracle as O
from oracle import gf2_port as P

pytestmark = pytest.mark.gpu
g = pytest.importorskip("paper_0811_1714_b200")

ENGINES = ["m4rm", "tc-i8", "tc-f8", "tc-f4"]


@pytest.fixture(autouse=True)
def _engine_reset():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    P.set_threads(P.max_threads())
    prev = g.get_engine()
    yield
    g.set_engine(prev)


def words(m):
    return m.to_numpy()


@pytest.mark.parametrize("engine", ENGINES)
def test_small_and_ragged(engine):
    g.set_engine(engine)
    rng = np.random.default_rng(5)
    for trial in range(25):
        m, l, n = (int(x) for x in rng.integers(1, 700, 3))
        a, b = g.random(m, l, trial + 1), g.random(l, n, trial + 2)
        want = O.naive_product(O.random(m, l, trial + 1), O.random(l, n, trial + 2))
        c = g.mul_direct(a, b)
        assert np.array_equal(words(c), want.words), (engine, m, l, n)
        assert g.trailing_bits_clean(c)


@pytest.mark.parametrize("engine", ENGINES)
def test_golden_and_windows(engine, golden):
    g.set_engine(engine)
    for i, m, l, n, sa, sb in golden["prod_cases"].tolist():
        a, b = g.random(m, l, sa), g.random(l, n, sb)
        assert np.array_equal(words(g.mul_direct(a, b)), golden[f"prod_{i}"])
        assert np.array_equal(words(g.mul_strassen(a, b, g.MulParams(cutoff=64))),
                              golden[f"prod_{i}"])
    pa, pb = g.random(90, 640, 77), g.random(700, 512, 78)
    aw = g.window(pa, 5, 64, 70, 385)
    bw = g.window(pb, 11, 192, 385, 250)
    assert np.array_equal(words(g.mul_direct(aw, bw)), golden["win_product"])
    pc = g.random(80, 512, 79)
    g.addmul(g.window(pc, 3, 64, 70, 250), aw, bw, g.MulParams(cutoff=64))
    assert np.array_equal(words(pc), golden["win_accum_parent"])
    a, b, c = g.random(150, 333, 91), g.random(333, 200, 92), g.random(150, 200, 93)
    g.addmul_direct(c, a, b)
    assert np.array_equal(words(c), golden["into_result"])


@pytest.mark.parametrize("engine", ENGINES)
def test_adversarial_large_sums(engine):
    """Rows of ones against columns of odd popcount near K: the f8 path's
    fp32 partial sums are as large as possible (K chunked at 8192)."""
    g.set_engine(engine)
    for l in (4096, 8192, 20000):
        ones = np.full((128, O.words_per_row(l)), np.uint64(0xFFFFFFFFFFFFFFFF))
        ones[:, -1] &= np.uint64(O.tail_mask(l))
        a = g.from_numpy(ones, l)
        dense_b = np.ones((l, 300), dtype=np.uint8)
        dense_b[0, ::2] = 0
        dense_b[5, ::3] = 0
        b = g.from_dense(dense_b)
        want = dense_b.sum(0) & 1
        got = g.to_dense(g.mul_direct(a, b))
        assert np.array_equal(got, np.tile(want, (128, 1))), (engine, l)


@pytest.mark.parametrize("engine", ENGINES)
def test_configs(engine, digests):
    g.set_engine(engine)
    a, b = g.random(1024, 1024, 11), g.random(1024, 1024, 12)
    assert O.digest(words(g.mul_direct(a, b))) == digests["cfg1"]
    a, b = g.random(4096, 4096, 21), g.random(4096, 4096, 22)
    assert O.digest(words(g.mul_strassen(a, b, g.MulParams(cutoff=1024, k=8)))) == digests["cfg2"]
    a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
    assert O.digest(words(g.mul_strassen(a, b))) == digests["cfg3"]
    assert O.digest(words(g.mul_direct(a, b))) == digests["cfg3"]
    t = O.bernoulli_threshold(0.1)
    a = g.bernoulli(10000, 7001, 41, threshold=t)
    b = g.bernoulli(7001, 12345, 42, threshold=t)
    assert O.digest(words(g.mul_strassen(a, b))) == digests["cfg4_product"]
    c0 = g.random(10000, 12345, 43)
    g.addmul(c0, a, b)
    assert O.digest(words(c0)) == digests["cfg4_addmul"]


def test_engine_switch_validation():
    with pytest.raises(ValueError):
        g.set_engine("nope")
    g.set_engine("tc-f8")
    assert g.get_engine() == "tc-f8"


def test_small_mul_m4rm_runs_m4rm():
    """Below the crossover mul_m4rm is one M4RM launch on every engine
    (large products dispatch to the tensor engine: test_gpu_api.py)."""
    g.set_engine("tc-i8")
    a, b = g.random(200, 300, 1), g.random(300, 100, 2)
    g._lib.timer_enable(True)
    g.mul_m4rm(a, b, 8)
    ms, ops, n = g._lib.timer_read()
    g._lib.timer_enable(False)
    assert n == 1 and ops == 200 * 300 * 100


@pytest.mark.parametrize("engine", ["tc-f4", "tc-i8"])
@pytest.mark.parametrize("cutoff", [2048, 4096, 16384])
def test_cfg3_every_depth(engine, cutoff, digests):
    """The 16384^3 product at recursion depths 3, 2 and 0 (the default
    cutoff 8192 = depth 1 is in test_configs): exercises the one-pass
    addition levels and, on tc-f4, the level-0 B pre-addition that writes
    its outputs transposed."""
    g.set_engine(engine)
    a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)
    c = g.mul_strassen(a, b, g.MulParams(cutoff=cutoff, k=8))
    assert O.digest(words(c)) == digests["cfg3"]


@pytest.mark.parametrize("engine", ["tc-f4", "tc-i8"])
def test_large_peeled_tensor_recursion_vs_port(engine):
    """Odd sizes, depth 2 with peeling, tensor-core leaves (2240x2048x2112,
    above the M4RM crossover), ragged column tiles and odd word counts in the
    transposed pre-addition; product and C += A.B against the C port."""
    g.set_engine(engine)
    m, l, n = 9000, 8300, 8500
    pa, pb = O.random(m, l, 61), O.random(l, n, 62)
    want = P.mul_strassen(pa, pb, cutoff=2048).words
    a, b = g.random(m, l, 61), g.random(l, n, 62)
    got = g.mul_strassen(a, b, g.MulParams(cutoff=2048, k=8))
    assert np.array_equal(words(got), want)
    assert g.trailing_bits_clean(got)
    c = g.random(m, n, 63)
    c0 = words(c)
    g.addmul(c, a, b, g.MulParams(cutoff=2048, k=8))
    assert np.array_equal(words(c), c0 ^ want)


@pytest.mark.parametrize("engine", ["tc-f4", "tc-i8"])
def test_tensor_recursion_on_windows_vs_port(engine):
    """Windows (odd word offsets, pitch != width) through the tensor-core
    recursion: depth 1 at cutoff 2048 with FP4/i8 leaves; product into a
    fresh matrix and C += A.B into a window of a larger C, whose bits
    outside the window must not change."""
    g.set_engine(engine)
    pa, pb, pc = g.random(5200, 4700, 71), g.random(4700, 5000, 72), g.random(5300, 5100, 73)
    aw = g.window(pa, 37, 64, 5100, 4500)          # word offset 1
    bw = g.window(pb, 101, 192, 4500, 4700)        # word offset 3
    cw = g.window(pc, 55, 128, 5100, 4700)         # word offset 2
    ha, hb = words(pa), words(pb)
    sub_a = O.HostMat(5100, 4500, np.ascontiguousarray(ha[37:37 + 5100, 1:1 + 71]))
    sub_b = O.HostMat(4500, 4700, np.ascontiguousarray(hb[101:101 + 4500, 3:3 + 74]))
    sub_a.words[:, -1] &= np.uint64(O.tail_mask(4500))
    sub_b.words[:, -1] &= np.uint64(O.tail_mask(4700))
    want = P.mul_strassen(sub_a, sub_b, cutoff=2048).words
    got = g.mul_strassen(aw, bw, g.MulParams(cutoff=2048, k=8))
    assert np.array_equal(words(got), want)
    before = words(pc).copy()
    g.addmul(cw, aw, bw, g.MulParams(cutoff=2048, k=8))
    after = words(pc)
    region = before[55:55 + 5100, 2:2 + 74].copy()
    # the window's last word holds 4700 - 73*64 = 28 columns; bits past them belong to the parent
    keep = np.uint64(~O.tail_mask(4700) & 0xFFFFFFFFFFFFFFFF)
    exp = region ^ want
    exp[:, -1] = (exp[:, -1] & ~keep) | (region[:, -1] & keep)
    assert np.array_equal(after[55:55 + 5100, 2:2 + 74], exp)
    outside = before.copy()
    outside[55:55 + 5100, 2:2 + 74] = after[55:55 + 5100, 2:2 + 74]
    assert np.array_equal(after, outside)


def test_f4_direct_random_windows_vs_port():
    """tc-f4 single products (no recursion: transposing B expansion, several
    row and column tiles, ragged tile widths) on random shapes and window
    offsets, plain and accumulating into a window."""
    g.set_engine("tc-f4")
    rng = np.random.default_rng(17)
    for trial in range(6):
        m, l, n = (int(x) for x in rng.integers(300, 2600, 3))
        ra, ca, rb, cb = (int(x) for x in rng.integers(0, 4, 4))
        pa = g.random(m + ra + 3, l + 64 * ca + 70, 100 + trial)
        pb = g.random(l + rb + 5, n + 64 * cb + 90, 200 + trial)
        aw, bw = g.window(pa, ra, 64 * ca, m, l), g.window(pb, rb, 64 * cb, l, n)
        wa, wb = words(pa), words(pb)
        sa = np.ascontiguousarray(wa[ra:ra + m, ca:ca + O.words_per_row(l)])
        sb = np.ascontiguousarray(wb[rb:rb + l, cb:cb + O.words_per_row(n)])
        sa[:, -1] &= np.uint64(O.tail_mask(l))
        sb[:, -1] &= np.uint64(O.tail_mask(n))
        want = P.mul_strassen(O.HostMat(m, l, sa), O.HostMat(l, n, sb), cutoff=64).words
        got = g.mul_direct(aw, bw)
        assert np.array_equal(words(got), want), (m, l, n)
        c = g.random(m, n, 300 + trial)
        c0 = words(c)
        g.addmul_direct(c, aw, bw)
        assert np.array_equal(words(c), c0 ^ want), (m, l, n)


@pytest.mark.parametrize("engine", ["tc-f4", "tc-i8"])
def test_two_fused_levels_option(engine, digests):
    """GF2_FUSE_LEVELS=2 (read once per process, hence a subprocess): both
    Strassen levels of a depth-2 product folded into the operand expansion
    (up to 16 source blocks per word; on tc-f4 the B side gathers from B^T
    with swapped quadrant masks at both levels)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_0811_1714_b200 as g\n"
        "from oracle import gf2_oracle as O\n"
        "g.set_engine(%r)\n"
        "a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)\n"
        "print(O.digest(g.mul_strassen(a, b, g.MulParams(cutoff=4096)).to_numpy()))\n"
    ) % (root, engine)
    env = dict(os.environ, GF2_FUSE_LEVELS="2")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == digests["cfg3"]


@pytest.mark.parametrize("engine", ["tc-f4", "tc-i8"])
@pytest.mark.parametrize("min_k", ["1000000", "0"])
def test_unfused_post_additions(engine, min_k, digests):
    """GF2_POST_FUSE_MIN_K (read once per process, hence a subprocess) above
    the leaf depth: the leaf products are stored plainly into their own
    level and one more combine pass folds them up (the default for
    1024-deep leaves); 0: the GEMM epilogue XORs each product into its
    destination quadrants (the default elsewhere). cfg2 at the reference's
    cutoff (depth 2) and an accumulate into a window."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "import paper_0811_1714_b200 as g\n"
        "from oracle import gf2_oracle as O\n"
        "g.set_engine(%r)\n"
        "a, b = g.random(4096, 4096, 21), g.random(4096, 4096, 22)\n"
        "print(O.digest(g.mul_strassen(a, b, g.MulParams(cutoff=1024, k=8)).to_numpy()))\n"
        "big = g.random(4200, 4300, 5)\n"
        "before = big.to_numpy().copy()\n"
        "w = g.window(big, 7, 64, 4096, 4096)\n"
        "g.addmul(w, a, b, g.MulParams(cutoff=1024, k=8))\n"
        "ref = g.mul_strassen(a, b).to_numpy()\n"
        "after = big.to_numpy()\n"
        "exp = before.copy(); exp[7:7 + 4096, 1:1 + 64] ^= ref\n"
        "print(bool((after == exp).all()))\n"
    ) % (root, engine)
    # GF2_TC_MIN_LEAF_K=0: keep the reference's depth 2 (1024-deep tensor
    # leaves), which the default leaf-depth rule would fold to depth 1
    env = dict(os.environ, GF2_POST_FUSE_MIN_K=min_k, GF2_TC_MIN_LEAF_K="0")
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-2] == digests["cfg2"]
    assert lines[-1] == "True"


@pytest.mark.parametrize("env", [{"GF2_PDL": "0"}, {"GF2_F4_ORDER": "0"}, {"GF2_F4_ORDER": "3"}])
def test_launch_and_raster_options(env, digests):
    """The same results with programmatic dependent launch off (every kernel
    then starts after its predecessor completes) and with the FP4 GEMM's
    other tile rasters (column tiles fastest; blocks of 3 row tiles, a
    ragged last block): cfg2 at cutoff 1024, cfg3 and a ragged addmul.
    Options are read once per process, hence a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "import paper_0811_1714_b200 as g\n"
        "from oracle import gf2_oracle as O\n"
        "from oracle import gf2_port as P\n"
        "a, b = g.random(4096, 4096, 21), g.random(4096, 4096, 22)\n"
        "print(O.digest(g.mul_strassen(a, b, g.MulParams(cutoff=1024, k=8)).to_numpy()))\n"
        "a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)\n"
        "print(O.digest(g.mul_strassen(a, b).to_numpy()))\n"
        "m, l, n = 5000, 4700, 5300\n"
        "c = g.random(m, n, 3)\n"
        "c0 = c.to_numpy().copy()\n"
        "g.addmul(c, g.random(m, l, 1), g.random(l, n, 2), g.MulParams(cutoff=2048))\n"
        "P.set_threads(P.max_threads())\n"
        "want = P.mul_strassen(P.random(m, l, 1), P.random(l, n, 2), cutoff=2048).words\n"
        "print(bool((c.to_numpy() == (c0 ^ want)).all()))\n"
    ) % (root,)
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-3] == digests["cfg2"]
    assert lines[-2] == digests["cfg3"]
    assert lines[-1] == "True"


@pytest.mark.parametrize("engine,n,cutoff,limit", [("m4rm", 4096, 512, 20e6), ("tc-f4", 8192, 1024, 150e6)])
def test_workspace_limit_takes_a_shallower_recursion(engine, n, cutoff, limit):
    """A recursion whose level buffers would not fit the device is run one or
    more levels shallower instead of failing with out-of-memory (fit_depth in
    csrc/gf2_strassen.cu). GF2_WS_LIMIT (bytes; read once per process, hence
    a subprocess) stands in for a full device: the unconstrained recursions
    here ask for 61 MiB (M4RM engine, depth 3) and 238 MiB (tc-f4, depth 2);
    under the limit both run at depth 1, stay inside it and give the same
    product."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_0811_1714_b200 as g\n"
        "from paper_0811_1714_b200 import _lib\n"
        "from oracle import gf2_port as P\n"
        "g.set_engine(%r)\n"
        "n, cutoff = %d, %d\n"
        "a, b = g.random(n, n, 5), g.random(n, n, 6)\n"
        "_lib.workspace_peak(reset=True)\n"
        "c = g.mul_strassen(a, b, g.MulParams(cutoff=cutoff, k=8))\n"
        "print(_lib.workspace_peak())\n"
        "P.set_threads(P.max_threads())\n"
        "want = P.mul_strassen(P.random(n, n, 5), P.random(n, n, 6), cutoff=cutoff).words\n"
        "print(bool((c.to_numpy() == want).all()))\n"
    ) % (root, engine, n, cutoff)
    peaks = {}
    for name, env in (("free", {}), ("limited", {"GF2_WS_LIMIT": str(int(limit))})):
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), cwd=root,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        lines = out.stdout.strip().splitlines()
        assert lines[-1] == "True", name
        peaks[name] = int(lines[-2])
    assert peaks["free"] > limit          # the unconstrained recursion would not have fit
    assert peaks["limited"] <= limit


@pytest.mark.parametrize("engine", ["m4rm", "tc-f4"])
def test_deep_recursion_many_leaves(engine):
    """Fuzzer regression: cutoff 64 on 4546x12000x12000 recurses to depth 6
    (7^6 = 117649 leaves), more problems than one launch's gridDim.z holds;
    leaves run in chunks (tiny leaves go to M4RM on every engine)."""
    g.set_engine(engine)
    m, l, n = 4546, 12000, 12000
    want = P.mul_strassen(O.random(m, l, 3), O.random(l, n, 4), cutoff=64).words
    got = g.mul_strassen(g.random(m, l, 3), g.random(l, n, 4), g.MulParams(cutoff=64, k=8))
    assert np.array_equal(words(got), want)


@pytest.mark.parametrize("engine,fuse", [("tc-f4", "1"), ("tc-i8", "1"), ("tc-f4", "2"),
                                         ("tc-i8", "2")])
def test_cfg3_depth6_tensor_leaves_chunked(engine, fuse, digests):
    """cfg3 at cutoff 256: depth 6, 117649 tensor-core leaves of 256^3 --
    the tensor job runs in chunks of source problems. Leaves below 640 go
    to M4RM by default, so GF2_TC_MIN_LEAF=256 (read once per process,
    hence a subprocess) forces them onto the tensor engine. With
    GF2_FUSE_LEVELS=2 each source problem feeds 49 leaves and owns 7 C
    problems, so the chunks (<= 1337 of the 2401 sources) must advance C by
    7 blocks per source (it advanced by one)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_0811_1714_b200 as g\n"
        "from oracle import gf2_oracle as O\n"
        "g.set_engine(%r)\n"
        "a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)\n"
        "print(O.digest(g.mul_strassen(a, b, g.MulParams(cutoff=256, k=8)).to_numpy()))\n"
    ) % (root, engine)
    env = dict(os.environ, GF2_TC_MIN_LEAF="256", GF2_TC_MIN_LEAF_K="0", GF2_FUSE_LEVELS=fuse)
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == digests["cfg3"]


@pytest.mark.parametrize("engine", ["tc-i8", "tc-f8"])
def test_single_cta_umma_tiles(engine, digests):
    """GF2_UMMA_CG=1 (read once per process, hence a subprocess): the 8-bit
    GEMM on single-CTA 128 x 256 tiles (tcgen05.mma.cta_group::1) instead of
    CTA pairs -- cfg2 at cutoff 1024, cfg3, and a ragged direct addmul on
    windows against the C port."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_0811_1714_b200 as g\n"
        "from oracle import gf2_oracle as O\n"
        "from oracle import gf2_port as P\n"
        "g.set_engine(%r)\n"
        "a, b = g.random(4096, 4096, 21), g.random(4096, 4096, 22)\n"
        "print(O.digest(g.mul_strassen(a, b, g.MulParams(cutoff=1024, k=8)).to_numpy()))\n"
        "a, b = g.random(16384, 16384, 31), g.random(16384, 16384, 32)\n"
        "print(O.digest(g.mul_strassen(a, b).to_numpy()))\n"
        "pa, pb = g.random(1300, 2000, 1), g.random(1900, 1500, 2)\n"
        "aw, bw = g.window(pa, 7, 64, 1201, 1777), g.window(pb, 3, 128, 1777, 1301)\n"
        "c = g.random(1201, 1301, 3)\n"
        "c0 = c.to_numpy().copy()\n"
        "g.addmul_direct(c, aw, bw)\n"
        "P.set_threads(P.max_threads())\n"
        "want = P.mul_strassen(O.HostMat(1201, 1777, g.copy_out(aw).to_numpy()),\n"
        "                      O.HostMat(1777, 1301, g.copy_out(bw).to_numpy()), cutoff=64).words\n"
        "print(bool((c.to_numpy() == (c0 ^ want)).all()))\n"
    ) % (root, engine)
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, GF2_UMMA_CG="1"),
                         cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert lines[-3] == digests["cfg2"]
    assert lines[-2] == digests["cfg3"]
    assert lines[-1] == "True"


@pytest.mark.parametrize("engine", ["tc-f4", "m4rm"])
def test_strassen_plan_graph_replay(engine, digests):
    """StrassenPlan (CUDA graph of one multiply): replays equal the eager
    result, read the operands' current contents, and accumulate correctly."""
    import torch
    g.set_engine(engine)
    n = 4096
    a, b = g.random(n, n, 21), g.random(n, n, 22)
    c = g.create(n, n)
    plan = g.StrassenPlan(c, a, b, g.MulParams(cutoff=1024, k=8))
    for _ in range(3):
        plan.run()
    torch.cuda.synchronize()
    assert O.digest(words(c)) == digests["cfg2"]
    g.copy_into(a, g.random(n, n, 99))          # refill in place, replay
    plan.run()
    assert g.equal(c, g.mul_strassen(a, b, g.MulParams(cutoff=1024, k=8)))
    acc = g.random(n, n, 5)
    acc0 = words(acc)
    p2 = g.StrassenPlan(acc, a, b, g.MulParams(cutoff=2048), accumulate=True)
    p2.run()
    p2.run()                                    # C + AB + AB = C
    assert np.array_equal(words(acc), acc0)
    del plan, p2


@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (200, 300, 130), (2048, 2048, 4096)])
def test_m4rm_plan_graph_replay(shape, digests):
    """M4rmPlan (CUDA graph of one mul_m4rm / mul_m4rm_into): replays equal
    the eager product (cfg1's digest at 1024^3; the 2048x2048x4096 product
    is past the crossover, so the graph holds the tensor-core path), read
    the operands' current contents, and accumulate (C + AB + AB = C)."""
    import torch
    m, l, n = shape
    seed = 11 if shape == (1024, 1024, 1024) else 3
    a, b = g.random(m, l, seed), g.random(l, n, seed + 1)
    c = g.create(m, n)
    plan = g.M4rmPlan(c, a, b, 8)
    for _ in range(3):
        plan.run()
    torch.cuda.synchronize()
    if shape == (1024, 1024, 1024):
        assert O.digest(words(c)) == digests["cfg1"]
    assert g.equal(c, g.mul_m4rm(a, b, 8))
    g.copy_into(a, g.random(m, l, 99))
    plan.run()
    assert g.equal(c, g.mul_m4rm(a, b, 8))
    acc = g.random(m, n, 5)
    acc0 = words(acc)
    p2 = g.M4rmPlan(acc, a, b, 8, accumulate=True)
    p2.run()
    p2.run()
    assert np.array_equal(words(acc), acc0)
    with pytest.raises(g.DimensionError):
        g.M4rmPlan(g.create(m + 1, n), a, b, 8)
    del plan, p2
