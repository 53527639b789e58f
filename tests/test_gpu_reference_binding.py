"""The INTEGRATION.md binding (examples/gf2mat_b200.py) run against the
UNMODIFIED reference package: gf2mat 0.1.0 installed under baseline/_ref
(or the source tree named by GF2_REF_SRC). gf2mat's own BitMatrix objects go
in and come out; the products are checked against the config digests
 and against gf2mat's own algorithms, and the reference CLI
runs `check` with the "b200" algorithm registered in its `_algorithm` table
(cli.py:65-94). Skipped, with the reason, where the reference is absent."""

import contextlib
import hashlib
import importlib.util
import io
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _ref_path():
    src = os.environ.get("GF2_REF_SRC")
    if src and os.path.isdir(os.path.join(src, "gf2mat")):
        return src
    p = os.path.join(ROOT, "baseline", "_ref")
    return p if os.path.isdir(os.path.join(p, "gf2mat")) else None


@pytest.fixture(scope="module")
def ref():
    path = _ref_path()
    if path is None:
        pytest.skip("reference gf2mat not installed (baseline/_ref absent, GF2_REF_SRC unset)")
    saved = {k: v for k, v in sys.modules.items() if k == "gf2mat" or k.startswith("gf2mat.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, path)
    try:
        import gf2mat
        import gf2mat.cli  # noqa: F401
        spec = importlib.util.spec_from_file_location("gf2mat_b200", os.path.join(ROOT, "examples", "gf2mat_b200.py"))
        b200 = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(b200)
        yield gf2mat, b200
    finally:
        sys.path.remove(path)
        for k in [k for k in sys.modules if k == "gf2mat" or k.startswith("gf2mat.")]:
            del sys.modules[k]
        sys.modules.update(saved)


@pytest.fixture(scope="module")
def digests():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "digests.json")) as fh:
        return json.load(fh)


def dig(m):
    return hashlib.sha256(np.ascontiguousarray(m.words, dtype="<u8").tobytes()).hexdigest()


def test_reference_is_the_stock_package(ref):
    gf2mat, _ = ref
    assert gf2mat.__version__ == "0.1.0"
    assert os.path.realpath(gf2mat.__file__).startswith(os.path.realpath(_ref_path()))


def test_cfg1_cfg2_cfg3_through_the_binding(ref, digests):
    """cfg1 mul_m4rm(A,B,8), cfg2 mul_strassen(A,B,MulParams(cutoff=1024,k=8))
    and cfg3 mul_strassen(A,B) on gf2mat.random inputs, gf2mat.BitMatrix out."""
    gf2mat, b200 = ref
    a, b = gf2mat.random(1024, 1024, 11), gf2mat.random(1024, 1024, 12)
    c = b200.mul_m4rm(a, b, 8)
    assert isinstance(c, gf2mat.BitMatrix) and dig(c) == digests["cfg1"]
    assert gf2mat.equal(c, gf2mat.mul_m4rm(a, b, 8))  # the reference's own M4RM
    a, b = gf2mat.random(4096, 4096, 21), gf2mat.random(4096, 4096, 22)
    assert dig(b200.mul_strassen(a, b, gf2mat.MulParams(cutoff=1024, k=8))) == digests["cfg2"]
    a, b = gf2mat.random(16384, 16384, 31), gf2mat.random(16384, 16384, 32)
    assert dig(b200.mul_strassen(a, b)) == digests["cfg3"]


def test_cfg4_through_the_binding(ref, digests):
    """cfg4: Bernoulli(0.1) operands (the reference has no
    Bernoulli generator, so the oracle's packs them into gf2mat matrices),
    the product and both addmul spellings."""
    gf2mat, b200 = ref
    from oracle import gf2_oracle as O
    t = O.bernoulli_threshold(0.1)

    def to_ref(h):
        m = gf2mat.create(h.nrows, h.ncols)
        m.words[...] = h.words
        return m

    a = to_ref(O.bernoulli(10000, 7001, 41, t))
    b = to_ref(O.bernoulli(7001, 12345, 42, t))
    assert dig(b200.mul_strassen(a, b)) == digests["cfg4_product"]
    c = gf2mat.random(10000, 12345, 43)
    b200.mul_m4rm_into(c, a, b, 8, 512, 8)
    assert dig(c) == digests["cfg4_addmul"]
    c = gf2mat.random(10000, 12345, 43)
    b200.addmul(c, a, b)
    assert dig(c) == digests["cfg4_addmul"]


def test_windows_and_errors_through_the_binding(ref):
    """gf2mat MatrixWindow operands and targets (ragged edges: the parent's
    bits beyond the window survive), and gf2mat's own exception classes."""
    gf2mat, b200 = ref
    pa, pb = gf2mat.random(300, 400, 1), gf2mat.random(500, 700, 2)
    a = gf2mat.window(pa, 10, 64, 200, 300)
    b = gf2mat.window(pb, 5, 128, 300, 450)
    want = gf2mat.mul_cubic(a, b)
    assert gf2mat.equal(b200.mul_strassen(a, b, gf2mat.MulParams(cutoff=64)), want)
    assert gf2mat.equal(b200.mul_m4rm(a, b, 8), want)
    parent = gf2mat.random(260, 600, 3)
    before = parent.words.copy()
    cw = gf2mat.window(parent, 30, 64, 200, 450)
    c0 = gf2mat.copy_out(cw)
    b200.mul_m4rm_into(cw, a, b, 8)
    assert gf2mat.equal(cw, gf2mat.add(c0, want))
    outside = np.ones(parent.words.shape, dtype=bool)
    outside[30:230, 1:1 + cw.width] = False
    assert np.array_equal(parent.words[outside], before[outside])
    tm = gf2mat.core.tail_mask(450)  # bits of the last window word beyond column 450+64
    assert np.array_equal(parent.words[30:230, cw.width] & ~tm, before[30:230, cw.width] & ~tm)
    with pytest.raises(gf2mat.DimensionError):
        b200.mul_strassen(gf2mat.random(10, 20, 1), gf2mat.random(21, 5, 2))


def test_reference_cli_check_with_b200_registered(ref):
    """`gf2mat check --algo b200 --algo strassen` (cli.py:181-211: every
    variant against the naive-product oracle and mul_cubic) passes, and
    --inject-fault on the B200 result is caught (exit 1)."""
    gf2mat, b200 = ref
    cli = gf2mat.cli
    orig = b200.register(cli)
    try:
        out = io.StringIO()
        with contextlib.redirect_stdout(out):
            rc = cli.main(["check", "--dims", "130x200x70", "--dims", "700x640x1100", "--algo", "b200",
                           "--algo", "strassen", "--cutoff", "128"])
        assert rc == 0, out.getvalue()
        assert "b200:ok" in out.getvalue() and "check: PASS" in out.getvalue()
        out = io.StringIO()
        with contextlib.redirect_stdout(out):
            rc = cli.main(["check", "--dims", "64x64x64", "--algo", "b200", "--inject-fault"])
        assert rc == 1 and "b200:FAIL" in out.getvalue()
    finally:
        cli._algorithm = orig
