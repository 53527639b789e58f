"""B200-native dense GF(2) matrix multiplication -- a drop-in for the hot
path of the reference package gf2mat v0.1.0 (arXiv 0811.1714, M4RI).

Same names, signatures and exception classes as gf2mat for the multiply
path (packed matrices, windows, M4RM, Strassen-Winograd, C += A.B), with
every matrix resident in B200 HBM and every operation executed by
hand-written sm_100a kernels in libgf2b200.so. No CPU fallback exists: if
the library or the GPU is missing, operations raise NativeUnavailable.
"""

from ._lib import (DeviceError, NativeUnavailable, get_engine, launch_count,
                   release_workspace, set_engine)
from .core import (BitMatrix, HostMatrix, MatrixWindow, add, add_into,
                   bernoulli, copy_into, copy_out, create, equal,
                   first_difference, from_dense, from_host, from_numpy,
                   identity, random, random_into, tail_mask, to_dense,
                   to_numpy, trailing_bits_clean, window, words_per_row,
                   zero_into)
from .errors import (AlignmentError, DimensionError, FormatError, GF2MatError,
                     ParameterError)
from .m4rm import (M4rmPlan, StripeSpec, mul_m4rm, mul_m4rm_blocked, mul_m4rm_into,
                   mul_m4rm_multitable)
from .gf2m import load, save
from .graycode import CombinationTable, GrayCode, build_gray, make_table
from .strassen import (GPU_CUTOFF, MulParams, PeelSplit, StrassenPlan,
                       addmul, addmul_direct, choose_k, default_params,
                       mul_direct, mul_strassen, peel_fixup, peel_split,
                       schedule_winograd)
from .structure import augment, mul_cubic, stack, transpose

__version__ = "0.1.0"

__all__ = [
    "AlignmentError", "BitMatrix", "DeviceError", "DimensionError",
    "FormatError", "GF2MatError", "GPU_CUTOFF", "HostMatrix", "MatrixWindow",
    "MulParams", "NativeUnavailable", "ParameterError", "PeelSplit",
    "StrassenPlan", "StripeSpec", "add", "add_into", "addmul", "addmul_direct", "bernoulli", "copy_into",
    "copy_out", "create", "default_params", "equal", "first_difference",
    "from_dense", "from_host", "from_numpy", "get_engine", "identity",
    "launch_count",
    "mul_direct", "mul_m4rm", "mul_m4rm_blocked", "mul_m4rm_into", "mul_m4rm_multitable",
    "mul_strassen", "peel_split", "random", "release_workspace", "set_engine",
    "tail_mask",
    "to_dense",
    "to_numpy", "trailing_bits_clean", "window", "words_per_row", "zero_into",
    "augment", "load", "mul_cubic", "save", "stack", "transpose",
    "CombinationTable", "GrayCode", "build_gray", "make_table", "choose_k",
    "peel_fixup", "schedule_winograd", "random_into", "M4rmPlan",
]
