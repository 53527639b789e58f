"""Method of the Four Russians on B200 -- the reference's M4RM entry points
(m4rm.py:124-155) with the same signatures, validation and errors, backed by
the sm_100a kernel in csrc/gf2_m4rm.cu.

k, t and b_s are the reference's CPU knobs (table width, tables per fused
update, cache row block). They are validated exactly as the reference does
(StripeSpec, m4rm.py:28-42); the device kernel fixes its own geometry
(8-bit Gray tables, 4 per 32-row half stage, register-resident C tiles),
which changes nothing in the result: the product is exact.

Dispatch (gf2_mul_base): products past the measured crossover -- at least
1e10 bit-ops with every side >= 640 -- run on the selected tensor engine
(tcgen05 kind::mxf4 by default), which computes the same product faster
(the reference's cfg4 call mul_m4rm_into(C, A, B, 8, 512, 8): 0.54 ms on the
M4RM kernel, ~0.28 ms on tc-f4); smaller products, e.g. cfg1's 1024^3, run
the M4RM kernel. set_engine("m4rm") forces the M4RM kernel everywhere.

M4rmPlan captures one such product on fixed matrices as a CUDA graph
(gf2_plan_m4rm): for small products the host path (validation, geometry,
tensor maps, up to three launches) costs more than the kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib
from .core import BitMatrix, Mat, _check_cuda_dev, _stream
from .errors import DimensionError, ParameterError

MAX_K = 16


@dataclass(frozen=True)
class StripeSpec:
    """m4rm.py:28-42 -- validated stripe parameters."""

    k: int
    t: int = 1
    b_s: int = 1

    def __post_init__(self):
        if not 1 <= self.k <= MAX_K:
            raise ParameterError(f"k={self.k} outside 1..{MAX_K}")
        if not 1 <= self.t <= 8:
            raise ParameterError(f"t={self.t} outside 1..8")
        if self.b_s < 1:
            raise ParameterError(f"block size {self.b_s} < 1")


def _validate(a: Mat, b: Mat, k: int, t: int, b_s: int) -> StripeSpec:
    """m4rm.py:69-74"""
    if a.ncols != b.nrows:
        raise DimensionError(
            f"inner dimensions {a.ncols} and {b.nrows} differ")
    return StripeSpec(k, t, b_s)


def _mul_into(c: Mat, a: Mat, b: Mat, k: int, accumulate: bool) -> None:
    _check_cuda_dev(c, a, b)
    _lib.check(_lib.lib_cuda().gf2_mul_base(c._view(), a._view(), b._view(),
                                            int(k), int(accumulate), _stream()))


def mul_m4rm(a: Mat, b: Mat, k: int) -> BitMatrix:
    """m4rm.py:124-129 -- basic Four-Russians product."""
    _validate(a, b, k, 1, 1)
    c = BitMatrix(a.nrows, b.ncols, a.device, _overwritten=True)
    _mul_into(c, a, b, k, False)
    return c


def mul_m4rm_blocked(a: Mat, b: Mat, k: int, b_s: int) -> BitMatrix:
    """m4rm.py:132-137"""
    _validate(a, b, k, 1, b_s)
    c = BitMatrix(a.nrows, b.ncols, a.device, _overwritten=True)
    _mul_into(c, a, b, k, False)
    return c


def mul_m4rm_multitable(a: Mat, b: Mat, k: int, t: int,
                        b_s: int) -> BitMatrix:
    """m4rm.py:140-147"""
    _validate(a, b, k, t, b_s)
    c = BitMatrix(a.nrows, b.ncols, a.device, _overwritten=True)
    _mul_into(c, a, b, k, False)
    return c


def mul_m4rm_into(c: BitMatrix, a: Mat, b: Mat, k: int,
                  b_s: int | None = None, t: int = 1) -> None:
    """m4rm.py:150-155 -- c += a @ b into an owned c."""
    b_s = max(a.nrows, 1) if b_s is None else b_s
    _validate(a, b, k, t, b_s)
    assert isinstance(c, BitMatrix), "M4RM writes into owned C only"
    if c.nrows != a.nrows or c.ncols != b.ncols:
        raise DimensionError(
            f"target {c.nrows}x{c.ncols} != product {a.nrows}x{b.ncols}")
    _mul_into(c, a, b, k, True)


class M4rmPlan:
    """A captured mul_m4rm / mul_m4rm_into (CUDA graph, gf2_plan_m4rm):
    C = A.B (or C ^= A.B with accumulate=True) on these matrices, replayed
    by `run()` with one graph launch. Each run reads the operands' current
    contents; the plan keeps its matrices alive."""

    def __init__(self, c: Mat, a: Mat, b: Mat, k: int = 8, accumulate: bool = False):
        import ctypes
        _validate(a, b, k, 1, 1)
        if c.nrows != a.nrows or c.ncols != b.ncols:
            raise DimensionError(
                f"target {c.nrows}x{c.ncols} != product {a.nrows}x{b.ncols}")
        _check_cuda_dev(c, a, b)
        self._mats = (c, a, b)
        self._lib = _lib.lib_cuda()
        h = ctypes.c_void_p()
        _lib.check(self._lib.gf2_plan_m4rm(ctypes.byref(h), c._view(), a._view(), b._view(),
                                           int(k), int(accumulate)))
        self._h = h

    @property
    def c(self):
        return self._mats[0]

    def run(self) -> None:
        """Launch the captured product on the current stream."""
        _lib.check(self._lib.gf2_plan_launch(self._h, _stream()))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.gf2_plan_destroy(h)
            self._h = None
