"""ctypes wrapper for oracle/libgf2oracle.so -- TEST / BASELINE ONLY.

The C port (gf2_oracle.c) restates the reference's M4RM + Strassen-Winograd
path (see that file's header for the file:line map). tests/ use it as a
fast checker; bench.py times it as the CPU baseline ("kind": "port").
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import gf2_oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libgf2oracle.so")


class _OMat(ctypes.Structure):
    _fields_ = [("w", ctypes.c_void_p), ("pitch", ctypes.c_int64),
                ("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64)]


_lib = None


def build() -> None:
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER(_OMat)
        L.oracle_m4rm_mul_into.argtypes = [P, P, P, ctypes.c_int,
                                           ctypes.c_int64, ctypes.c_int]
        L.oracle_mul_strassen.argtypes = [P, P, P, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_int]
        L.oracle_random.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                    ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_uint64, ctypes.c_int64]
        L.oracle_bernoulli.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_int64]
        L.oracle_peel_split.argtypes = [ctypes.c_int64] * 4 + [
            ctypes.POINTER(ctypes.c_int64)]
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _omat(words: np.ndarray, nrows: int, ncols: int) -> _OMat:
    assert words.dtype == np.uint64
    if words.ndim == 2 and words.shape[0] > 1:
        pitch = words.strides[0] // 8
    else:
        pitch = O.words_per_row(ncols)
    return _OMat(words.ctypes.data if words.size else None, pitch, nrows,
                 ncols)


def random(nrows: int, ncols: int, seed: int, row_base: int = 0) -> O.HostMat:
    m = O.zeros(nrows, ncols)
    if m.words.size:
        lib().oracle_random(m.words.ctypes.data, m.width, nrows, ncols,
                            seed & 0xFFFFFFFFFFFFFFFF, row_base)
    return m


def bernoulli(nrows: int, ncols: int, seed: int, threshold: int,
              row_base: int = 0) -> O.HostMat:
    m = O.zeros(nrows, ncols)
    if m.words.size:
        lib().oracle_bernoulli(m.words.ctypes.data, m.width, nrows, ncols,
                               seed & 0xFFFFFFFFFFFFFFFF, threshold, row_base)
    return m


def m4rm_mul_into(c: O.HostMat, a: O.HostMat, b: O.HostMat, k: int = 8,
                  b_s: int = 0, t: int = 1) -> None:
    ca, aa, bb = (_omat(c.words, c.nrows, c.ncols),
                  _omat(a.words, a.nrows, a.ncols),
                  _omat(b.words, b.nrows, b.ncols))
    rc = lib().oracle_m4rm_mul_into(ctypes.byref(ca), ctypes.byref(aa),
                                    ctypes.byref(bb), k, b_s, t)
    if rc:
        raise ValueError("oracle_m4rm_mul_into: bad dimensions")


def mul_strassen(a: O.HostMat, b: O.HostMat, cutoff: int = 2048,
                 b_s: int = 0, k: int = 0, t: int = 8,
                 c: O.HostMat | None = None,
                 accumulate: bool = False) -> O.HostMat:
    if c is None:
        c = O.zeros(a.nrows, b.ncols)
    ca, aa, bb = (_omat(c.words, c.nrows, c.ncols),
                  _omat(a.words, a.nrows, a.ncols),
                  _omat(b.words, b.nrows, b.ncols))
    rc = lib().oracle_mul_strassen(ctypes.byref(ca), ctypes.byref(aa),
                                   ctypes.byref(bb), cutoff, b_s, k, t,
                                   int(accumulate))
    if rc:
        raise ValueError("oracle_mul_strassen: bad dimensions")
    return c


def peel_split(m: int, l: int, n: int, cutoff: int):
    out = (ctypes.c_int64 * 4)()
    lib().oracle_peel_split(m, l, n, cutoff, out)
    return tuple(out)
