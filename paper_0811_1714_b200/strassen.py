"""Strassen-Winograd with peeling on B200 -- the reference's entry points
(strassen.py:27-84, 257-282) with the same signatures and validation.

The recursion itself runs natively (csrc/gf2_strassen.cu): the same peel
rule and the same depth as the reference for the given cutoff, but each
recursion level is one batched device launch (all 7^s sub-products at
once) instead of a depth-first walk with two scratch quadrants.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import NamedTuple

from . import _lib
from .core import BitMatrix, Mat, _check_cuda_dev, _stream
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


def default_params() -> MulParams:
    """Device defaults (the reference derives its from CPU cache sizes,
    tuning.py:47-65): recursion above GPU_CUTOFF, the selected base-case
    engine below (tcgen05 kind::mxf4 by default; small leaves run M4RM)."""
    return MulParams(cutoff=GPU_CUTOFF, k=8, t=8)


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
