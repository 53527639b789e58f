"""ctypes binding of libgf2b200.so (include/gf2b200.h).

There is no CPU fallback: if the library or a CUDA device is missing,
every device operation raises `NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (AlignmentError, DimensionError, GF2MatError,
                     ParameterError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgf2b200.so")

GF2_OK = 0
GF2_ERR_DIMENSION = 1
GF2_ERR_ALIGNMENT = 2
GF2_ERR_PARAMETER = 3
GF2_ERR_CUDA = 4
GF2_ERR_OOM = 5
GF2_ERR_INTERNAL = 6
GF2_ERR_NCCL = 7


class NativeUnavailable(RuntimeError):
    """libgf2b200.so could not be loaded or no CUDA device is present."""


class DeviceError(GF2MatError):
    """A CUDA runtime failure inside the native library."""


class Gf2View(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("pitch", ctypes.c_int64),
                ("nrows", ctypes.c_int64), ("ncols", ctypes.c_int64)]


# name -> (restype, argtypes); every exported symbol of include/gf2b200.h
_V = ctypes.POINTER(Gf2View)
_P = ctypes.c_void_p
SIGNATURES = {
    "gf2_version": (ctypes.c_char_p, []),
    "gf2_last_error": (ctypes.c_char_p, []),
    "gf2_pitch_words": (ctypes.c_int64, [ctypes.c_int64]),
    "gf2_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, _V, _P]),
    "gf2_free": (ctypes.c_int, [_V, _P]),
    "gf2_upload": (ctypes.c_int, [_V, _P, ctypes.c_int64, _P]),
    "gf2_download": (ctypes.c_int, [_V, _P, ctypes.c_int64, _P]),
    "gf2_zero": (ctypes.c_int, [_V, _P]),
    "gf2_random": (ctypes.c_int, [_V, ctypes.c_uint64, ctypes.c_int64, _P]),
    "gf2_bernoulli": (ctypes.c_int, [_V, ctypes.c_uint64, ctypes.c_uint64,
                                     ctypes.c_int64, _P]),
    "gf2_add": (ctypes.c_int, [_V, _V, _V, _P]),
    "gf2_copy": (ctypes.c_int, [_V, _V, _P]),
    "gf2_m4rm": (ctypes.c_int, [_V, _V, _V, ctypes.c_int, ctypes.c_int, _P]),
    "gf2_mul": (ctypes.c_int, [_V, _V, _V, ctypes.c_int, _P]),
    "gf2_mul_base": (ctypes.c_int, [_V, _V, _V, ctypes.c_int, ctypes.c_int, _P]),
    "gf2_make_table": (ctypes.c_int, [_V, _V, ctypes.c_int, _P]),
    "gf2_peel_fixup": (ctypes.c_int, [_V, _V, _V, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, _P]),
    "gf2_transpose": (ctypes.c_int, [_V, _V, _P]),
    "gf2_cubic": (ctypes.c_int, [_V, _V, _V, ctypes.c_int, _P]),
    "gf2_copy_cols": (ctypes.c_int, [_V, ctypes.c_int64, _V, _P]),
    "gf2_strassen": (ctypes.c_int, [_V, _V, _V, ctypes.c_int64, ctypes.c_int,
                                    ctypes.c_int, _P]),
    "gf2_plan_strassen": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), _V, _V, _V,
                                         ctypes.c_int64, ctypes.c_int, ctypes.c_int]),
    "gf2_plan_m4rm": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), _V, _V, _V,
                                     ctypes.c_int, ctypes.c_int]),
    "gf2_plan_launch": (ctypes.c_int, [_P, _P]),
    "gf2_plan_destroy": (ctypes.c_int, [_P]),
    "gf2_peel_split": (ctypes.c_int, [ctypes.c_int64] * 4
                       + [ctypes.POINTER(ctypes.c_int64)]),
    "gf2_launch_count": (ctypes.c_int64, []),
    "gf2_m4rm_launch_count": (ctypes.c_int64, []),
    "gf2_workspace_peak": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    "gf2_timer_enable": (ctypes.c_int, [ctypes.c_int]),
    "gf2_mul_sharded": (ctypes.c_int, [_V, _V, _V, _P, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int64, ctypes.c_int, _P]),
    "gf2_release_workspace": (ctypes.c_int, []),
    "gf2_stream_sync": (ctypes.c_int, [ctypes.c_void_p]),
    "gf2_set_engine": (ctypes.c_int, [ctypes.c_int]),
    "gf2_get_engine": (ctypes.c_int, []),
    "gf2_timer_read": (ctypes.c_int, [ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_int64)]),
}

_lib = None


def load():
    """Load the native library (no GPU needed to load it)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is not built; run __graft_entry__.build() "
                "(make -C paper_0811_1714_b200/csrc)")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_cuda_checked = False


def lib_cuda():
    """The library, after checking that a CUDA device is usable."""
    global _cuda_checked
    lib = load()
    if not _cuda_checked:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable(
                "no CUDA device: the B200 path has no CPU fallback")
        _cuda_checked = True
    return lib


def check(rc: int) -> None:
    if rc == GF2_OK:
        return
    msg = load().gf2_last_error().decode(errors="replace")
    if rc == GF2_ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == GF2_ERR_ALIGNMENT:
        raise AlignmentError(msg)
    if rc == GF2_ERR_PARAMETER:
        raise ParameterError(msg)
    if rc == GF2_ERR_OOM:
        raise MemoryError(msg)
    raise DeviceError(f"native error {rc}: {msg}")


def _raw_stream_fn():
    import torch
    c = torch._C
    if hasattr(c, "_cuda_getCurrentRawStream") and hasattr(c, "_cuda_getDevice"):
        return lambda: c._cuda_getCurrentRawStream(c._cuda_getDevice())
    return lambda: torch.cuda.current_stream().cuda_stream  # public API fallback


_raw_stream = None


def current_stream() -> int:
    """Raw cudaStream_t of torch's current stream on the current device
    (the same value as torch.cuda.current_stream().cuda_stream, without
    building a Stream object: ~0.3 us instead of ~3.5 us per call)."""
    global _raw_stream
    if _raw_stream is None:
        _raw_stream = _raw_stream_fn()
    return _raw_stream()


def launch_count() -> int:
    return int(load().gf2_launch_count())


def m4rm_launch_count() -> int:
    """Launches of the M4RM kernel alone (which engine ran a product)."""
    return int(load().gf2_m4rm_launch_count())


def workspace_peak(reset: bool = False) -> int:
    """Bytes: high-water mark of the library's pooled device workspace
    since the last reset (reset=True restarts it at the current use)."""
    v = ctypes.c_int64()
    check(load().gf2_workspace_peak(ctypes.byref(v), int(reset)))
    return int(v.value)


def timer_enable(on: bool = True) -> None:
    check(load().gf2_timer_enable(int(on)))


def timer_read():
    """(kernel_ms, bitops, launches) of the M4RM launches timed since
    timer_enable(True); synchronizes the recorded events."""
    ms, ops, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    check(load().gf2_timer_read(ctypes.byref(ms), ctypes.byref(ops),
                                ctypes.byref(n)))
    return ms.value, ops.value, n.value


ENGINES = {"m4rm": 0, "tc-i8": 1, "tc-f8": 2, "tc-f4": 3}


def set_engine(name: str) -> None:
    """Select the product engine: "m4rm" (shared-memory Gray tables),
    "tc-i8", "tc-f8" or "tc-f4" (tcgen05 tensor cores; tc-f4 is the
    block-scaled kind::mxf4 MMA on e2m1 nibbles). Results are identical."""
    if name not in ENGINES:
        raise ValueError(f"engine {name!r} not in {sorted(ENGINES)}")
    check(load().gf2_set_engine(ENGINES[name]))


def release_workspace() -> None:
    """Return the device workspace cached by the stream-ordered pool
    (Strassen level buffers, tensor-core operands) to the system;
    synchronizes the current device."""
    check(lib_cuda().gf2_release_workspace())


def get_engine() -> str:
    e = int(load().gf2_get_engine())
    return {v: k for k, v in ENGINES.items()}[e]
