"""Strassen-Winograd with peeling on B200 -- the reference's entry points
(strassen.py:27-84, 257-282) with the same signatures and validation.

The recursion itself runs natively (csrc/gf2_strassen.cu): the same peel
rule and the same depth as the reference for the given cutoff, but each
recursion level is one batched device launch (all 7^s sub-products at
once) instead of a depth-first walk with two scratch quadrants.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Callable, NamedTuple

from . import _lib
from .core import (BitMatrix, Mat, _check_cuda_dev, _stream, add_into, window,
                   words_per_row)
from .errors import DimensionError, ParameterError

_WORD = 64

# Crossover chosen for the B200 with the tc-f4 base case (DESIGN.md §4.3,
# tools/bench_configs.py --cutoff): leaves of 8192 keep the FP4 GEMM at ~0.94
# of its peak; another level (4096 leaves) costs more in additions and
# expansion than its 1/8 fewer MACs save (cfg3 1.08 vs 1.15 ms, cfg5 57 vs 67).
GPU_CUTOFF = 8192


@dataclass
class MulParams:
    """strassen.py:27-56 -- same fields, defaults and invariants.

    On the device, `cutoff` sets the recursion depth exactly as in the
    reference (peel_split); `k`, `t`, `b_s`, `l1_bytes`, `l2_bytes` are
    validated and recorded (the kernel picks its own tiling).
    """

    cutoff: int = 2048
    b_s: int | None = None
    k: int = 0
    t: int = 8
    l1_bytes: int = 32768
    l2_bytes: int = 1 << 20

    def __post_init__(self):
        if self.b_s is None:
            self.b_s = max(self.cutoff // 2, 1)
        if self.cutoff < 64:
            raise ParameterError(f"cutoff {self.cutoff} < 64")
        if not 1 <= self.t <= 8:
            raise ParameterError(f"t={self.t} outside 1..8")
        if not 0 <= self.k <= 16:
            raise ParameterError(f"k={self.k} outside 0..16")
        if not 1 <= self.b_s <= self.cutoff:
            raise ParameterError(
                f"block size {self.b_s} outside 1..cutoff={self.cutoff}")


class PeelSplit(NamedTuple):
    m: int
    l: int
    n: int
    depth: int


def peel_split(m: int, l: int, n: int, cutoff: int) -> PeelSplit:
    """strassen.py:66-84 (evaluated by the native library)."""
    out = (ctypes.c_int64 * 4)()
    _lib.check(_lib.load().gf2_peel_split(m, l, n, cutoff, out))
    return PeelSplit(*(int(x) for x in out))


DEFAULT_L1_BYTES = 32 * 1024      # tuning.py:23-24
DEFAULT_L2_BYTES = 1 << 20


def choose_k(b_s: int, l1_bytes: int, t: int = 8,
             ncols: int | None = None) -> int:
    """tuning.py:29-44 -- the reference's Gray-table width rule: about
    0.75 log2(b_s) - 2, one narrower when that makes t tables of ncols-bit
    rows fit in L1. Recorded in MulParams; the device kernel's tables do
    not depend on it."""
    if b_s < 2:
        raise ParameterError(f"block size {b_s} < 2")
    k = max(1, min(16, math.floor(0.75 * math.log2(b_s)) - 2))
    if ncols is not None and k > 1:
        row_bytes = 8 * words_per_row(ncols)
        if t * (row_bytes << k) > l1_bytes >= t * (row_bytes << (k - 1)):
            k -= 1
    return k


def default_params(l1_bytes: int | None = None,
                   l2_bytes: int | None = None) -> MulParams:
    """Device defaults with no arguments: recursion above GPU_CUTOFF, the
    selected base-case engine below (tcgen05 kind::mxf4 by default; small
    leaves run M4RM). Given cache sizes, the reference's own derivation
    (tuning.py:47-65): the largest multiple-of-64 cutoff whose two square
    operands fit in L2, b_s = cutoff / 2, t = 8, k = choose_k -- the same
    MulParams the reference returns (the product does not depend on them)."""
    if l1_bytes is None and l2_bytes is None:
        return MulParams(cutoff=GPU_CUTOFF, k=8, t=8)
    l1 = DEFAULT_L1_BYTES if l1_bytes is None else l1_bytes
    l2 = DEFAULT_L2_BYTES if l2_bytes is None else l2_bytes
    if l1 <= 0 or l2 <= 0:
        raise ParameterError(
            f"cache sizes must be positive, got L1={l1} L2={l2}")
    cutoff = math.isqrt(4 * l2) // 64 * 64
    if cutoff < 64:
        raise ParameterError(f"L2 of {l2} bytes is too small to tune")
    b_s = cutoff // 2
    return MulParams(cutoff=cutoff, b_s=b_s, k=choose_k(b_s, l1, 8, cutoff),
                     t=8, l1_bytes=l1, l2_bytes=l2)


# strassen.py:183-204 -- one Winograd level as data: 15 additions ("+",
# out = u XOR v) and 7 products ("*", out = u . v) in the reference's order,
# over the quadrants of A, B, C and the scratch windows X (A-shaped sums),
# P (X holding the A11.B11 product) and Y (B-shaped sums). Over GF(2) every
# subtraction of the published schedule is an XOR.
_WINOGRAD_STEPS = (
    ("+", "X", "A11", "A21"), ("+", "Y", "B22", "B12"), ("*", "C21", "X", "Y"),
    ("+", "X", "A21", "A22"), ("+", "Y", "B12", "B11"), ("*", "C22", "X", "Y"),
    ("+", "X", "X", "A11"), ("+", "Y", "B22", "Y"), ("*", "C12", "X", "Y"),
    ("+", "X", "A12", "X"), ("*", "C11", "X", "B22"), ("*", "P", "A11", "B11"),
    ("+", "C12", "P", "C12"), ("+", "C21", "C12", "C21"),
    ("+", "C12", "C12", "C22"), ("+", "C22", "C21", "C22"),
    ("+", "C12", "C12", "C11"), ("+", "Y", "Y", "B21"),
    ("*", "C11", "A22", "Y"), ("+", "C21", "C21", "C11"),
    ("*", "C11", "A12", "B21"), ("+", "C11", "P", "C11"),
)


def schedule_winograd(a: Mat, b: Mat, c: Mat, temps: tuple,
                      multiply: Callable[[Mat, Mat, Mat], None]) -> None:
    """strassen.py:141-204 -- one recursion level on device windows:
    c = a . b with 7 calls multiply(dst, u, v) and 15 device additions, in
    the reference's order. `temps` = (X, Y) scratch matrices, at least
    (m/2) x max(l/2, n/2) and (l/2) x (n/2); c must not alias a or b. The
    library's own recursion (mul_strassen) runs this schedule as batched
    launches instead (csrc/gf2_strassen.cu); this entry serves callers that
    drive the levels themselves."""
    m, l, n = a.nrows, a.ncols, b.ncols
    if c.nrows != m or c.ncols != n:
        raise DimensionError(f"target {c.shape} != product {m}x{n}")
    if m % 2 or l % 128 or n % 128:
        raise DimensionError(
            f"dimensions {m}x{l}x{n} not halvable on word boundaries")
    m2, l2, n2 = m // 2, l // 2, n // 2
    xbuf, ybuf = temps
    q = {"X": window(xbuf, 0, 0, m2, l2), "P": window(xbuf, 0, 0, m2, n2),
         "Y": window(ybuf, 0, 0, l2, n2)}
    for name, mat, rows, cols in (("A", a, m2, l2), ("B", b, l2, n2),
                                  ("C", c, m2, n2)):
        for i in (0, 1):
            for j in (0, 1):
                q[f"{name}{i + 1}{j + 1}"] = window(mat, i * rows, j * cols,
                                                    rows, cols)
    for op, out, u, v in _WINOGRAD_STEPS:
        if op == "+":
            add_into(q[out], q[u], q[v])
        else:
            multiply(q[out], q[u], q[v])


def peel_fixup(c: Mat, a: Mat, b: Mat, m2: int, l2: int, n2: int,
               params: MulParams | None = None) -> None:
    """strassen.py:219-249 -- complete c = a . b given that c[:m2, :n2]
    already holds a[:m2, :l2] . b[:l2, :n2]: the inner remainder is
    accumulated into that block, then the remaining rows, then the
    remaining columns, each one base-case product on the device
    (gf2_peel_fixup; never the recursion). `params` is accepted like the
    reference's (the device base case does not depend on it)."""
    m, l, n = a.nrows, a.ncols, b.ncols
    if c.nrows != m or c.ncols != n:
        raise DimensionError(f"target {c.shape} != product {m}x{n}")
    if not (0 <= m2 <= m and 0 <= l2 <= l and 0 <= n2 <= n):
        raise DimensionError(
            f"peel dims ({m2},{l2},{n2}) exceed ({m},{l},{n})")
    if a.ncols != b.nrows:
        raise DimensionError(
            f"inner dimensions {a.ncols} and {b.nrows} differ")
    _check_cuda_dev(c, a, b)
    _lib.check(_lib.lib_cuda().gf2_peel_fixup(
        c._view(), a._view(), b._view(), int(m2), int(l2), int(n2), _stream()))


def _strassen(c: Mat, a: Mat, b: Mat, params: MulParams,
              accumulate: bool) -> None:
    _check_cuda_dev(c, a, b)
    _lib.check(_lib.lib_cuda().gf2_strassen(
        c._view(), a._view(), b._view(), int(params.cutoff), int(params.k),
        int(accumulate), _stream()))


def mul_strassen(a: Mat, b: Mat, params: MulParams | None = None) -> BitMatrix:
    """strassen.py:257-282 -- full dispatch: peel, Strassen-Winograd
    recursion, leaves on the base-case engine (set_engine), peel fix-ups."""
    if a.ncols != b.nrows:
        raise DimensionError(
            f"inner dimensions {a.ncols} and {b.nrows} differ")
    if params is None:
        params = default_params()
    c = BitMatrix(a.nrows, b.ncols, a.device, _overwritten=a.ncols > 0)
    if a.nrows and b.ncols and a.ncols:
        _strassen(c, a, b, params, False)
    return c


def addmul(c: Mat, a: Mat, b: Mat, params: MulParams | None = None) -> None:
    """C += A.B at Strassen scale (cfg4/cfg5 addmul). The reference spells
    this add_into(C, C, mul_strassen(A, B)); here the final
    Winograd combination XORs straight into C (a window is fine)."""
    if a.ncols != b.nrows:
        raise DimensionError(
            f"inner dimensions {a.ncols} and {b.nrows} differ")
    if c.nrows != a.nrows or c.ncols != b.ncols:
        raise DimensionError(
            f"target {c.nrows}x{c.ncols} != product {a.nrows}x{b.ncols}")
    if params is None:
        params = default_params()
    _strassen(c, a, b, params, True)


def mul_direct(a: Mat, b: Mat) -> BitMatrix:
    """One product launch with the current engine (set_engine), without the
    Strassen recursion: the tensor-core contraction of north_star (c) when a
    tcgen05 engine is selected, the M4RM kernel otherwise."""
    if a.ncols != b.nrows:
        raise DimensionError(
            f"inner dimensions {a.ncols} and {b.nrows} differ")
    c = BitMatrix(a.nrows, b.ncols, a.device, _overwritten=True)
    _check_cuda_dev(c, a, b)
    _lib.check(_lib.lib_cuda().gf2_mul(c._view(), a._view(), b._view(), 0,
                                       _stream()))
    return c


def addmul_direct(c: Mat, a: Mat, b: Mat) -> None:
    """C += A.B in one product launch with the current engine."""
    _check_cuda_dev(c, a, b)
    _lib.check(_lib.lib_cuda().gf2_mul(c._view(), a._view(), b._view(), 1,
                                       _stream()))


class StrassenPlan:
    """A captured multiply (CUDA graph, gf2_plan_strassen): C (+)= A.B on
    these matrices, replayed by `run()` with one graph launch instead of the
    per-call host work of mul_strassen / addmul (~45 us: validation,
    planning, tensor-map encoding, 4-6 launches). Each run reads the
    operands' current contents, so a serving loop refills A and B in place
    and re-runs. The plan keeps its matrices alive."""

    def __init__(self, c: Mat, a: Mat, b: Mat, params: MulParams | None = None,
                 accumulate: bool = False):
        import ctypes
        if a.ncols != b.nrows:
            raise DimensionError(
                f"inner dimensions {a.ncols} and {b.nrows} differ")
        if c.nrows != a.nrows or c.ncols != b.ncols:
            raise DimensionError(
                f"target {c.nrows}x{c.ncols} != product {a.nrows}x{b.ncols}")
        _check_cuda_dev(c, a, b)
        params = params or default_params()
        self._mats = (c, a, b)
        self._lib = _lib.lib_cuda()
        h = ctypes.c_void_p()
        _lib.check(self._lib.gf2_plan_strassen(
            ctypes.byref(h), c._view(), a._view(), b._view(),
            int(params.cutoff), int(params.k), int(accumulate)))
        self._h = h

    @property
    def c(self):
        return self._mats[0]

    def run(self) -> None:
        """Launch the captured multiply on the current stream."""
        _lib.check(self._lib.gf2_plan_launch(self._h, _stream()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.gf2_plan_destroy(h)
            self._h = None
