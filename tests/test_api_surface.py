"""The drop-in surface on CPU (no device work): every public name of the
reference that the hot path touches exists here, and the host-side pieces
of that surface (Gray codes, the tuning rules behind default_params) match
fixtures generated from the reference itself (tests/golden/make_golden.py
--api)."""

import json
import os

import numpy as np
import pytest

import paper_0811_1714_b200 as g
from paper_0811_1714_b200 import strassen as S

HERE = os.path.dirname(os.path.abspath(__file__))

# OUT OF SCOPE -- element ops (core.py:211-275), the scalar
# XOR switch (core.py:32), cubic's public parity helpers (cubic.py:19-59)
# and the tuning config layer (tuning.py:68-123).
OUT_OF_SCOPE = {"get_bit", "set_bit", "read_bits", "row_add", "set_scalar_xor",
                "parity64", "parity_accumulate", "load_config", "resolve_params"}


@pytest.fixture(scope="module")
def api():
    return np.load(os.path.join(HERE, "golden", "golden_api.npz"))


def test_reference_names_present():
    with open(os.path.join(HERE, "golden", "reference_api.json")) as fh:
        ref = json.load(fh)
    missing = set(ref["__all__"]) - set(g.__all__)
    assert missing <= OUT_OF_SCOPE, sorted(missing - OUT_OF_SCOPE)
    for name in g.__all__:
        assert hasattr(g, name), name


def test_gray_codes_up_to_16(api):
    for k in (6, 9, 12, 16):
        gc = g.build_gray(k)
        assert gc.k == k
        assert list(gc.code) == api[f"gray_code_k{k}"].tolist()
        assert list(gc.changed_bit)[1:] == api[f"gray_changed_k{k}"].tolist()[1:]
    assert g.build_gray(3).code == (0, 1, 3, 2, 6, 7, 5, 4)        # Fig. 1
    for bad in (0, 17):
        with pytest.raises(g.ParameterError):
            g.build_gray(bad)


def test_default_params_kats(api):
    for l1, l2, cutoff, b_s, k, t in api["default_params_kat"].tolist():
        if cutoff < 0:
            with pytest.raises(g.ParameterError):
                g.default_params(l1, l2)
            continue
        p = g.default_params(l1, l2)
        assert (p.cutoff, p.b_s, p.k, p.t, p.l1_bytes, p.l2_bytes) == \
            (cutoff, b_s, k, t, l1, l2)
    for bs, l1, t, nc, k in api["choose_k_kat"].tolist():
        assert S.choose_k(bs, l1, t, nc if nc else None) == k
    with pytest.raises(g.ParameterError):
        g.default_params(0, 1 << 20)
    p = g.default_params()                 # device defaults (no cache sizes)
    assert p.cutoff == g.GPU_CUTOFF and 1 <= p.b_s <= p.cutoff


def test_winograd_schedule_shape():
    """22 steps: 15 additions, 7 products, each product target a C quadrant
    or the P scratch, as in strassen.py:183-204."""
    steps = S._WINOGRAD_STEPS
    assert len(steps) == 22
    assert sum(op == "+" for op, *_ in steps) == 15
    prods = [s for s in steps if s[0] == "*"]
    assert len(prods) == 7
    assert {d for _, d, _, _ in prods} <= {"C11", "C12", "C21", "C22", "P"}
