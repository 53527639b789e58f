"""gf2mat backend for the B200 path: the module a gf2mat maintainer would add
as `gf2mat/_b200.py`. Host `BitMatrix` / `MatrixWindow`
objects stay the reference's own (core.py:57-170); each product uploads the
operands into device matrices allocated by the library, runs the B200
kernels through the C ABI (include/gf2b200.h) and downloads the result.
Nothing here but ctypes and numpy: no torch, no CUDA headers.

    import gf2mat, gf2mat_b200 as b200
    c = b200.mul_strassen(a, b)              # strassen.py:257-282
    b200.mul_m4rm_into(c, a, b, 8)           # m4rm.py:150-155
    b200.register(gf2mat.cli)                # `gf2mat check --algo b200`

`tests/test_gpu_reference_binding.py` runs this module against the
unmodified gf2mat package installed under baseline/_ref.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("GF2B200_LIB", os.path.join(_HERE, "..", "paper_0811_1714_b200", "libgf2b200.so"))
_lib = ctypes.CDLL(_LIB_PATH)


class _View(ctypes.Structure):  # gf2b200.h `gf2_view`
    _fields_ = [("data", ctypes.c_void_p), ("pitch", ctypes.c_int64),
                ("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64)]


_P = ctypes.POINTER(_View)
_U64P = ctypes.POINTER(ctypes.c_uint64)
for _name, _args in {
    "gf2_alloc": [ctypes.c_int64, ctypes.c_int64, _P, ctypes.c_void_p],
    "gf2_free": [_P, ctypes.c_void_p],
    "gf2_upload": [_P, _U64P, ctypes.c_int64, ctypes.c_void_p],
    "gf2_download": [_P, _U64P, ctypes.c_int64, ctypes.c_void_p],
    "gf2_strassen": [_P, _P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p],
    "gf2_mul_base": [_P, _P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_void_p],
    "gf2_stream_sync": [ctypes.c_void_p],
}.items():
    getattr(_lib, _name).argtypes = _args
    getattr(_lib, _name).restype = ctypes.c_int
_lib.gf2_last_error.restype = ctypes.c_char_p

GPU_CUTOFF = 8192  # the library's device default (MulParams.cutoff 0 or None)


def _errors():
    from gf2mat.errors import AlignmentError, DimensionError, GF2MatError, ParameterError
    return {1: DimensionError, 2: AlignmentError, 3: ParameterError}, GF2MatError


def _check(rc):
    if rc:
        table, base = _errors()
        raise table.get(rc, base)(_lib.gf2_last_error().decode())


def _tail(ncols):
    rem = ncols % 64
    return np.uint64(0xFFFFFFFFFFFFFFFF) if rem == 0 else np.uint64((0xFFFFFFFFFFFFFFFF << (64 - rem)) & 0xFFFFFFFFFFFFFFFF)


class _Dev:
    """A device matrix with the host matrix's shape (and optionally words)."""

    def __init__(self, m, upload=True):
        self.v = _View()
        _check(_lib.gf2_alloc(m.nrows, m.ncols, ctypes.byref(self.v), None))
        if upload and m.nrows and m.width:
            w = np.ascontiguousarray(m.words, dtype=np.uint64)
            if m.ncols % 64:
                w[:, -1] &= _tail(m.ncols)  # a window's parent bits stay behind
            _check(_lib.gf2_upload(ctypes.byref(self.v), w.ctypes.data_as(_U64P), w.shape[1], None))

    def download_into(self, m):
        """Write the device words back into host matrix `m` (bits of a
        window's parent beyond its right edge are preserved)."""
        if not (m.nrows and m.width):
            return
        w = np.empty((m.nrows, m.width), dtype=np.uint64)
        _check(_lib.gf2_download(ctypes.byref(self.v), w.ctypes.data_as(_U64P), m.width, None))
        _check(_lib.gf2_stream_sync(None))
        if m.ncols % 64:
            t = _tail(m.ncols)
            w[:, -1] = (m.words[:, -1] & ~t) | (w[:, -1] & t)
        m.words[...] = w

    def __del__(self):
        try:
            _lib.gf2_free(ctypes.byref(self.v), None)
        except Exception:
            pass


def _shape_check(c, a, b):
    from gf2mat.errors import DimensionError
    if a.ncols != b.nrows:
        raise DimensionError(f"inner dimensions {a.ncols} and {b.nrows} differ")
    if c is not None and (c.nrows != a.nrows or c.ncols != b.ncols):
        raise DimensionError(f"target {c.nrows}x{c.ncols} != {a.nrows}x{b.ncols}")


def mul_strassen(a, b, params=None):
    """strassen.py:257-282 on the B200 (tensor-core leaves)."""
    from gf2mat import core
    _shape_check(None, a, b)
    c = core.create(a.nrows, b.ncols)
    cutoff = (params.cutoff if params is not None and params.cutoff else GPU_CUTOFF)
    k = params.k if params is not None and params.k else 8
    da, db, dc = _Dev(a), _Dev(b), _Dev(c, upload=False)
    _check(_lib.gf2_strassen(ctypes.byref(dc.v), ctypes.byref(da.v), ctypes.byref(db.v), cutoff, k, 0, None))
    dc.download_into(c)
    return c


def addmul(c, a, b, params=None):
    """C += A.B in place: add_into(C, C, mul_strassen(A, B)) (core.py:278-300)."""
    _shape_check(c, a, b)
    cutoff = (params.cutoff if params is not None and params.cutoff else GPU_CUTOFF)
    da, db, dc = _Dev(a), _Dev(b), _Dev(c)
    _check(_lib.gf2_strassen(ctypes.byref(dc.v), ctypes.byref(da.v), ctypes.byref(db.v), cutoff, 8, 1, None))
    dc.download_into(c)
    return c


def mul_m4rm(a, b, k=8):
    """m4rm.py:124-131 on the B200."""
    from gf2mat import core
    _shape_check(None, a, b)
    c = core.create(a.nrows, b.ncols)
    da, db, dc = _Dev(a), _Dev(b), _Dev(c, upload=False)
    _check(_lib.gf2_mul_base(ctypes.byref(dc.v), ctypes.byref(da.v), ctypes.byref(db.v), k, 0, None))
    dc.download_into(c)
    return c


def mul_m4rm_into(c, a, b, k=8, b_s=0, t=1):
    """m4rm.py:150-155 (C ^= A.B) on the B200; b_s / t do not change the
    device tiling (results are independent of them)."""
    _shape_check(c, a, b)
    da, db, dc = _Dev(a), _Dev(b), _Dev(c)
    _check(_lib.gf2_mul_base(ctypes.byref(dc.v), ctypes.byref(da.v), ctypes.byref(db.v), k, 1, None))
    dc.download_into(c)
    return c


def register(cli):
    """One-line registration in the reference CLI's algorithm table
    (cli.py:65-94 `_algorithm`): the name "b200" runs mul_strassen here."""
    orig = cli._algorithm

    def _algorithm(name, params):
        if name == "b200":
            return (lambda a, b: mul_strassen(a, b, params)), (params.k, params.t, params.b_s, params.cutoff)
        return orig(name, params)

    cli._algorithm = _algorithm
    return orig
