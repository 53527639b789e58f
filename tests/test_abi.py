"""The C-ABI library loads and exports every symbol include/gf2b200.h
declares; host-only entry points work without a GPU. CPU only."""

import ctypes
import os
import re

import pytest

from paper_0811_1714_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gf2b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gf2_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for name in syms:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.py"


def test_version_and_pitch():
    lib = _lib.load()
    assert b"sm_100a" in lib.gf2_version()
    assert lib.gf2_pitch_words(1) == 2
    assert lib.gf2_pitch_words(64) == 2
    assert lib.gf2_pitch_words(65) == 2
    assert lib.gf2_pitch_words(129) == 4
    assert lib.gf2_pitch_words(1024) == 16
    assert lib.gf2_pitch_words(12345) == 208
    assert lib.gf2_pitch_words(16384) == 256


def test_peel_split_through_abi(golden):
    from paper_0811_1714_b200 import peel_split
    for row in golden["peel_split_kat"].tolist():
        m, l, n, cut = row[:4]
        assert tuple(peel_split(m, l, n, cut)) == tuple(row[4:])


def test_validation_without_device():
    """Parameter / dimension checks happen before any CUDA call and map
    to the reference's exception classes."""
    lib = _lib.load()
    v = _lib.Gf2View(None, 1, 0, 0)
    rc = lib.gf2_m4rm(ctypes.byref(v), ctypes.byref(v), ctypes.byref(v), 0,
                      0, None)
    assert rc == _lib.GF2_ERR_PARAMETER
    assert b"k=0 outside 1..16" in lib.gf2_last_error()
    with pytest.raises(_lib.ParameterError):
        _lib.check(rc)
    a = _lib.Gf2View(None, 1, 0, 3)
    b = _lib.Gf2View(None, 1, 4, 0)
    rc = lib.gf2_m4rm(ctypes.byref(v), ctypes.byref(a), ctypes.byref(b), 8,
                      0, None)
    assert rc == _lib.GF2_ERR_DIMENSION
    assert b"inner dimensions 3 and 4 differ" in lib.gf2_last_error()
    rc = lib.gf2_strassen(ctypes.byref(v), ctypes.byref(v), ctypes.byref(v),
                          32, 0, 0, None)
    assert rc == _lib.GF2_ERR_PARAMETER
    odd = _lib.Gf2View(12, 1, 1, 64)  # misaligned pointer
    rc = lib.gf2_zero(ctypes.byref(odd), None)
    assert rc == _lib.GF2_ERR_ALIGNMENT


def test_no_cpu_fallback():
    """Without a GPU the product path raises instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_0811_1714_b200 as g
    with pytest.raises(g.NativeUnavailable):
        g.random(4, 4, 1)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_0811_1714_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(
                    r"^\s*(from|import)\s+oracle|gf2_oracle|gf2_port|"
                    r"libgf2oracle|sys\.path.*oracle", text, re.M), f
