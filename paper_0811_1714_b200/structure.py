"""Structural operations and the narrow-B cubic product on device
(SURVEY.md §8(f) #3-#4): transpose (core.py:374-376), augment / stack
(core.py:344-371), mul_cubic (cubic.py:76-102)."""

from __future__ import annotations

from . import _lib
from .core import (BitMatrix, Mat, _check_cuda_dev, _stream, copy_into,
                   create, window)
from .errors import DimensionError


def transpose(a: Mat) -> BitMatrix:
    """core.py:374-376 -- new matrix with result[j, i] == a[i, j]
    (bit transpose in 64x64 blocks per warp)."""
    out = create(a.ncols, a.nrows, a.device)
    if a.nrows and a.ncols:
        _lib.check(_lib.lib_cuda().gf2_transpose(out._view(), a._view(),
                                                 _stream()))
    return out


def stack(a: Mat, b: Mat) -> BitMatrix:
    """core.py:361-371 -- rows of a above rows of b."""
    if a.ncols != b.ncols:
        raise DimensionError(
            f"stack column counts {a.ncols} and {b.ncols} differ")
    out = create(a.nrows + b.nrows, a.ncols, a.device)
    if a.nrows and a.ncols:
        copy_into(window(out, 0, 0, a.nrows, a.ncols), a)
    if b.nrows and b.ncols:
        copy_into(window(out, a.nrows, 0, b.nrows, b.ncols), b)
    return out


def augment(a: Mat, b: Mat) -> BitMatrix:
    """core.py:344-358 -- columns of a followed by columns of b; b lands at
    any bit offset (the reference densifies when a.ncols % 64 != 0; here a
    funnel-shift column copy does it in place)."""
    if a.nrows != b.nrows:
        raise DimensionError(
            f"augment row counts {a.nrows} and {b.nrows} differ")
    out = create(a.nrows, a.ncols + b.ncols, a.device)
    if a.nrows and a.ncols:
        copy_into(window(out, 0, 0, a.nrows, a.ncols), a)
    if a.nrows and b.ncols:
        _check_cuda_dev(out, b)
        _lib.check(_lib.lib_cuda().gf2_copy_cols(out._view(), a.ncols,
                                                 b._view(), _stream()))
    return out


def mul_cubic(a: Mat, b: Mat) -> BitMatrix:
    """cubic.py:76-102 -- AND + XOR-fold + parity against B^T; the
    reference's base case for narrow B (n < 64)."""
    if a.ncols != b.nrows:
        raise DimensionError(
            f"inner dimensions {a.ncols} and {b.nrows} differ")
    c = create(a.nrows, b.ncols, a.device)
    if a.nrows and b.ncols and a.ncols:
        _check_cuda_dev(c, a, b)
        _lib.check(_lib.lib_cuda().gf2_cubic(c._view(), a._view(), b._view(),
                                             0, _stream()))
    return c
