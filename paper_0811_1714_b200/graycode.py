"""Gray codes and tables of row combinations -- the reference's public
graycode API (graycode.py:26-156) over device matrices.

`build_gray` / `GrayCode` are a tiny host-side sequence (the reflect-and-
prefix construction); the drop-in keeps them so callers that inspect the
table order keep working. `CombinationTable` holds its 2^k rows in HBM and
`make_table` fills them with one kernel launch (`gf2_make_table`:
csrc/gf2_kernels.cu k_make_table, a Gray walk per word column). The M4RM
multiply itself never goes through these objects: it builds its tables in
shared memory inside the kernel (csrc/gf2_m4rm.cu).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

from . import _lib
from .core import Mat, _check_cuda_dev, _stream, create, window
from .errors import DimensionError, ParameterError

MAX_K = 16


@dataclass(frozen=True)
class GrayCode:
    """graycode.py:26-35 -- the code sequence (code[0] = 0) and, per step,
    the index of the bit that flipped (bit 0 = least significant;
    changed_bit[0] is unused)."""

    k: int
    code: tuple[int, ...]
    changed_bit: tuple[int, ...]


def build_gray(k: int) -> GrayCode:
    """graycode.py:38-48 -- k-bit reflected Gray code. Value j of the
    reflect-and-prefix sequence is j ^ (j >> 1); between steps j-1 and j
    the flipped bit is the lowest set bit of j."""
    if not 1 <= k <= MAX_K:
        raise ParameterError(f"gray code width {k} outside 1..{MAX_K}")
    n = 1 << k
    code = tuple(j ^ (j >> 1) for j in range(n))
    changed = (0,) + tuple((j & -j).bit_length() - 1 for j in range(1, n))
    return GrayCode(k, code, changed)


@lru_cache(maxsize=None)
def gray_code(k: int) -> GrayCode:
    """graycode.py:55-60 -- cached accessor (codes are immutable)."""
    return build_gray(k)


class CombinationTable:
    """graycode.py:78-105 -- direct-indexed table of the 2^k XOR
    combinations of k source rows, in device memory. Index bit k-1 is the
    FIRST source row; slot 0 is the zero row. `k` is the width of the most
    recent fill and may be below `capacity`."""

    def __init__(self, k: int, ncols: int, device=None):
        if not 1 <= k <= MAX_K:
            raise ParameterError(f"table width {k} outside 1..{MAX_K}")
        self.capacity = k
        self.k = k
        self.ncols = ncols
        self.matrix = create(1 << k, ncols, device)

    @property
    def words(self):
        """(2^capacity, width) int64 device view of the table words."""
        return self.matrix.words

    @property
    def rows(self):
        """The 2^k rows of the last fill; rows[x] is combination x."""
        return self.matrix.words[:1 << self.k]

    def row(self, x: int):
        return self.matrix.words[x]


def make_table(b: Mat, start_row: int, k: int, table: CombinationTable) -> None:
    """graycode.py:108-156 -- fill `table` with all combinations of rows
    [start_row, start_row + k) of `b` on the device (same checks, in the
    same order, and the same errors as the reference). Bits of a window
    source beyond its right edge are masked, so the table rows stay clean."""
    if not 1 <= k <= table.capacity:
        raise ParameterError(
            f"table fill width {k} outside 1..{table.capacity}")
    if start_row < 0 or start_row + k > b.nrows:
        raise DimensionError(
            f"rows [{start_row},{start_row + k}) outside 0..{b.nrows}")
    if table.ncols != b.ncols:
        raise DimensionError(
            f"table width {table.ncols} != source width {b.ncols}")
    table.k = k
    if table.ncols == 0:
        return
    src = window(b, start_row, 0, k, b.ncols)
    _check_cuda_dev(table.matrix, src)
    _lib.check(_lib.lib_cuda().gf2_make_table(table.matrix._view(), src._view(),
                                              int(k), _stream()))


__all__ = ["MAX_K", "GrayCode", "build_gray", "gray_code", "CombinationTable",
           "make_table"]
