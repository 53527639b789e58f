"""The device CLI (cli.py-compatible front end): gen / mul / check / bench /
params, exit codes, fault injection (cli.py:181-211, test_cli.py)."""

import csv

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
g = pytest.importorskip("paper_0811_1714_b200")


@pytest.fixture(autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(*argv):
    from paper_0811_1714_b200.cli import main
    return main(list(argv))


def test_gen_mul_roundtrip(tmp_path, capsys, golden):
    a, b, c = (str(tmp_path / x) for x in ("a.gf2m", "b.gf2m", "c.gf2m"))
    assert run("gen", "--dims", "37x200", "--seed", "5", "--out", a) == 0
    assert np.array_equal(np.fromfile(a, dtype=np.uint8), golden["gf2m_37x200_s5"])
    assert run("gen", "--dims", "200x90", "--seed", "6", "--out", b) == 0
    for algo in ("auto", "m4rm", "cubic", "m4rm-t8"):
        assert run("mul", a, b, c, "--algo", algo) == 0
        want = g.mul_cubic(g.random(37, 200, 5), g.random(200, 90, 6))
        assert g.equal(g.load(c), want)


def test_check_oracle_is_host_naive_product():
    """check's oracle is a host product of the downloaded operands,
    independent of every device kernel (cli.py:181-211 uses
    _reference.naive_product the same way)."""
    from paper_0811_1714_b200 import cli
    a, b = g.random(70, 130, 1), g.random(130, 90, 2)
    want = cli.naive_product(a, b)
    assert np.array_equal(g.to_dense(g.mul_cubic(a, b)), want)
    assert cli._first_mismatch(g.mul_strassen(a, b), want) is None
    bad = want.copy()
    bad[3, 77] ^= 1
    assert cli._first_mismatch(g.mul_strassen(a, b), bad) == (3, 77)


def test_check_pass_and_fault(capsys):
    assert run("check", "--dims", "300x200x100", "--dims", "65x64x1") == 0
    assert "check: PASS" in capsys.readouterr().out
    assert run("check", "--dims", "64x64x64", "--inject-fault") == 1
    assert "FAIL(0, 0)" in capsys.readouterr().out


def test_bench_csv_and_errors(tmp_path, capsys):
    out = tmp_path / "b.csv"
    assert run("bench", "--dims", "1024x1024x1024", "--reps", "2",
               "--algo", "m4rm", "--algo", "strassen", "--out", str(out)) == 0
    # the reference's BenchRecord header, byte for byte (cli.py:97-129)
    assert open(out).readline().strip() == ("algorithm,m,l,n,k,t,bs,cutoff,reps,wall_s,mean_s,"
                                            "min_s,peak_mem_bytes")
    rows = list(csv.DictReader(open(out)))
    assert [r["algorithm"] for r in rows] == ["m4rm", "strassen"]
    assert all(float(r["min_s"]) <= float(r["mean_s"]) for r in rows)
    assert all(int(r["peak_mem_bytes"]) > 0 for r in rows)  # each rep allocates its product
    assert run("mul", str(tmp_path / "missing"), str(out), str(out)) == 2
    assert run("check", "--dims", "2x2x2", "--algo", "nope") == 2
    prev = g.get_engine()
    assert run("params", "--engine", "tc-f8") == 0
    assert "engine=tc-f8" in capsys.readouterr().out
    g.set_engine(prev)
