"""Pin the CPU oracle (NumPy restatement + C port) to the reference.

Fixtures in tests/golden/ were produced by importing the reference itself
(tests/golden/make_golden.py); digests match SURVEY.md §8(c). CPU only.
"""

import numpy as np
import pytest

from oracle import gf2_oracle as O
from oracle import gf2_port as P


def test_random_kats(golden):
    # SURVEY.md §8(c) literal KATs
    assert O.random(1, 128, 0).words.tolist() == [[0xe220a8397b1dcdaf,
                                                   0x6e789e6aa1b965f4]]
    assert O.random(2, 65, 7).words.tolist() == [
        [0x63cbe1e459320dd7, 0x0], [0xe6984080bab12a02, 0x8000000000000000]]
    for key, args in [("kat_random_1x128_s0", (1, 128, 0)),
                      ("kat_random_2x65_s7", (2, 65, 7)),
                      ("kat_random_37x200_s123", (37, 200, 123))]:
        assert np.array_equal(O.random(*args).words, golden[key])
        assert np.array_equal(P.random(*args).words, golden[key])


def test_random_row_base_slices():
    full = O.random(50, 333, 9)
    part = O.random(20, 333, 9, row_base=17)
    assert np.array_equal(full.words[17:37], part.words)
    assert np.array_equal(P.random(20, 333, 9, row_base=17).words, part.words)


def test_gray_codes(golden):
    # Fig. 1 of the paper / graycode.py:38-48
    for k in range(1, 6):
        code, changed = O.build_gray(k)
        assert code == golden[f"gray_code_k{k}"].tolist()
        assert changed[1:] == golden[f"gray_changed_k{k}"].tolist()[1:]
    assert O.build_gray(3)[0] == [0, 1, 3, 2, 6, 7, 5, 4]


def test_make_table(golden):
    pb = O.random(40, 256, 5)
    w = O.view(pb.words, 3, 64, 9, 130)
    src = O.masked(w)
    for k in (3, 8):
        tbl = O.make_table(src[1:1 + k], k)
        assert np.array_equal(tbl, golden[f"table_k{k}"])


def test_read_bits(golden):
    rb = O.random(3, 256, 7)
    for r, sc, k, v in golden["read_bits_kat"].tolist():
        assert int(O.read_bits_rows(rb.words[r:r + 1], sc, k)[0]) == v


def test_peel_split(golden):
    for row in golden["peel_split_kat"].tolist():
        m, l, n, cut = row[:4]
        assert O.peel_split(m, l, n, cut).astuple() == tuple(row[4:])
        assert P.peel_split(m, l, n, cut) == tuple(row[4:])


def _prod_cases(golden):
    for i, m, l, n, sa, sb in golden["prod_cases"].tolist():
        yield i, m, l, n, O.random(m, l, sa), O.random(l, n, sb)


def test_naive_and_m4rm_vs_reference_products(golden):
    for i, m, l, n, a, b in _prod_cases(golden):
        want = golden[f"prod_{i}"]
        assert np.array_equal(O.naive_product(a, b).words, want), (m, l, n)
        c = O.zeros(m, n).words
        O.m4rm_mul_into(c, a, b, k=min(8, max(1, l)), b_s=37, t=3)
        assert np.array_equal(c, want), (m, l, n)


def test_port_vs_reference_products(golden):
    for i, m, l, n, a, b in _prod_cases(golden):
        want = golden[f"prod_{i}"]
        got = P.mul_strassen(a, b, cutoff=64)
        assert np.array_equal(got.words, want), (m, l, n)
        c = O.zeros(m, n)
        P.m4rm_mul_into(c, a, b, k=5, b_s=17, t=3)
        assert np.array_equal(c.words, want), (m, l, n)


def test_window_products(golden):
    pa, pb, pc = O.random(90, 640, 77), O.random(700, 512, 78), \
        O.random(80, 512, 79)
    aw = O.view(pa.words, 5, 64, 70, 385)
    bw = O.view(pb.words, 11, 192, 385, 250)
    assert np.array_equal(O.naive_product(aw, bw).words, golden["win_product"])
    got = P.mul_strassen(aw, bw, cutoff=64)
    assert np.array_equal(got.words, golden["win_product"])
    assert np.array_equal(pc.words, golden["win_accum_parent_before"])
    cw = O.view(pc.words, 3, 64, 70, 250)
    P.mul_strassen(aw, bw, cutoff=64, c=cw, accumulate=True)
    assert np.array_equal(pc.words, golden["win_accum_parent"])


def test_into_variant(golden):
    a, b, c = O.random(150, 333, 91), O.random(333, 200, 92), \
        O.random(150, 200, 93)
    O.m4rm_mul_into(c.words, a, b, 8, 64, 4)
    assert np.array_equal(c.words, golden["into_result"])


def test_slow_oracle_agrees():
    a, b = O.random(7, 70, 3), O.random(70, 9, 4)
    assert np.array_equal(O.unpack(O.naive_product(a, b)),
                          O.naive_product_slow(a, b))


def test_cfg1_digest(digests):
    a, b = O.random(1024, 1024, 11), O.random(1024, 1024, 12)
    assert O.digest(O.naive_product(a, b).words) == digests["cfg1"]
    c = O.zeros(1024, 1024)
    P.m4rm_mul_into(c, a, b, 8)
    assert O.digest(c.words) == digests["cfg1"]


def test_bernoulli_generator():
    t = O.bernoulli_threshold(0.1)
    assert t == (1 << 64) // 10 == 0x1999999999999999
    a = O.bernoulli(64, 7001, 41, t)
    assert O.trailing_bits_clean(a)
    dens = O.unpack(a).mean()
    assert 0.09 < dens < 0.11
    assert np.array_equal(P.bernoulli(64, 7001, 41, t).words, a.words)
    part = O.bernoulli(10, 7001, 41, t, row_base=30)
    assert np.array_equal(part.words, a.words[30:40])


@pytest.mark.slow
def test_cfg4_digests_port(digests):
    t = O.bernoulli_threshold(0.1)
    P.set_threads(P.max_threads())
    a = P.bernoulli(10000, 7001, 41, t)
    b = P.bernoulli(7001, 12345, 42, t)
    c = P.mul_strassen(a, b)
    assert O.digest(c.words) == digests["cfg4_product"]
    c0 = P.random(10000, 12345, 43)
    P.mul_strassen(a, b, c=c0, accumulate=True)
    assert O.digest(c0.words) == digests["cfg4_addmul"]
