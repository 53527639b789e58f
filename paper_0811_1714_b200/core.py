"""Device-resident bit-packed GF(2) matrices and windows (B200).

Mirrors the reference's storage layer (core.py:57-341, gf2mat v0.1.0) over
HBM: 64 columns per word, column c at bit 63 - c % 64 of word c // 64, rows
padded to a device pitch (16-byte multiple; 128-byte multiple once a row
spans 16 words) so row starts are aligned for vector / TMA access. Storage
is a torch int64 tensor (torch's caching allocator and streams are the
plumbing); every operation is a call into libgf2b200.so on the current
torch stream. Windows (core.py:110-170) are non-owning views at word-aligned
column offsets; writes through them keep the bits beyond their right edge.
"""

from __future__ import annotations

import sys

import numpy as np

from . import _lib
from .errors import AlignmentError, DimensionError

WORD_BITS = 64
_FULL = 0xFFFFFFFFFFFFFFFF


def words_per_row(ncols: int) -> int:
    """core.py:45-46"""
    return (ncols + WORD_BITS - 1) // WORD_BITS


def tail_mask(ncols: int) -> int:
    """core.py:49-54 (as a Python int)."""
    rem = ncols % WORD_BITS
    return _FULL if rem == 0 else (_FULL << (WORD_BITS - rem)) & _FULL


def _signed(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


def _torch():
    import torch
    return torch


class BitMatrix:
    """Owned device matrix (core.py:57-107).

    Attributes: nrows, ncols, width (words per row), pitch (device row
    stride in words), storage (torch int64 tensor [nrows, pitch] on cuda).
    Padding words beyond `width` stay zero; trailing bits stay zero.
    """

    __slots__ = ("nrows", "ncols", "width", "pitch", "storage", "__weakref__")

    def __init__(self, nrows: int, ncols: int, device=None,
                 _overwritten: bool = False):
        if nrows < 0 or ncols < 0:
            raise DimensionError(f"negative dimensions {nrows}x{ncols}")
        lib = _lib.lib_cuda()
        torch = _torch()
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.width = words_per_row(ncols)
        self.pitch = int(lib.gf2_pitch_words(ncols))
        if device is None:
            device = torch.cuda.current_device()  # index on the current device
        self.storage = torch.empty((self.nrows, self.pitch),
                                   dtype=torch.int64, device=device)
        # zero-filled (core.py:176-178) by the library (a 2-D memset, no
        # kernel): the whole pitch, or for a product target -- whose words
        # the kernels overwrite, merging into a ragged last word -- only
        # that last word and the padding words after it
        first = 0
        if _overwritten:
            first = self.width - 1 if ncols % 64 else self.width
        if first < self.pitch and self.nrows:
            z = _lib.Gf2View(self.storage.data_ptr() + 8 * first, self.pitch,
                             self.nrows, (self.pitch - first) * WORD_BITS)
            if self.storage.get_device() == _current_device():
                _lib.check(lib.gf2_zero(z, _stream()))
            else:
                with torch.cuda.device(self.storage.device):
                    _lib.check(lib.gf2_zero(z, _lib.current_stream()))

    # reference-compatible accessors
    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    @property
    def device(self):
        return self.storage.device

    @property
    def words(self):
        """(nrows, width) int64 torch view of the packed words."""
        return self.storage[:, :self.width]

    def _view(self) -> _lib.Gf2View:
        return _lib.Gf2View(self.storage.data_ptr() or None, self.pitch,
                            self.nrows, self.ncols)

    def to_numpy(self, out: np.ndarray | None = None) -> np.ndarray:
        return _download(self, out)

    def to_host(self):
        return _to_host(self)

    def __eq__(self, other) -> bool:
        if not isinstance(other, (BitMatrix, MatrixWindow)):
            return NotImplemented
        return equal(self, other)

    def __hash__(self):
        return id(self)

    def __repr__(self) -> str:
        return f"BitMatrix({self.nrows}x{self.ncols}, {self.device})"


class MatrixWindow:
    """Non-owning view of a rectangle of a BitMatrix (core.py:110-170)."""

    __slots__ = ("parent", "row_offset", "col_offset", "nrows", "ncols",
                 "width")

    def __init__(self, parent: BitMatrix, row_offset: int, col_offset: int,
                 nrows: int, ncols: int):
        if col_offset % WORD_BITS != 0:
            raise AlignmentError(
                f"window column offset {col_offset} is not a multiple of 64")
        if nrows < 0 or ncols < 0:
            raise DimensionError(f"negative window {nrows}x{ncols}")
        if row_offset < 0 or col_offset < 0 \
                or row_offset + nrows > parent.nrows \
                or col_offset + ncols > parent.ncols:
            raise DimensionError(
                f"window {nrows}x{ncols}@({row_offset},{col_offset}) exceeds "
                f"parent {parent.nrows}x{parent.ncols}")
        self.parent = parent
        self.row_offset = row_offset
        self.col_offset = col_offset
        self.nrows = nrows
        self.ncols = ncols
        self.width = words_per_row(ncols)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.nrows, self.ncols)

    @property
    def device(self):
        return self.parent.storage.device

    @property
    def pitch(self) -> int:
        return self.parent.pitch

    @property
    def words(self):
        w0 = self.col_offset // WORD_BITS
        return self.parent.storage[self.row_offset:self.row_offset + self.nrows,
                                   w0:w0 + self.width]

    def _view(self) -> _lib.Gf2View:
        p = self.parent
        base = p.storage.data_ptr()
        off = self.row_offset * p.pitch + self.col_offset // WORD_BITS
        ptr = base + 8 * off if base else None
        return _lib.Gf2View(ptr, p.pitch, self.nrows, self.ncols)

    def to_numpy(self, out: np.ndarray | None = None) -> np.ndarray:
        return _download(self, out)

    def to_host(self):
        return _to_host(self)

    def __eq__(self, other) -> bool:
        if not isinstance(other, (BitMatrix, MatrixWindow)):
            return NotImplemented
        return equal(self, other)

    def __hash__(self):
        return id(self)

    def __repr__(self) -> str:
        return (f"MatrixWindow({self.nrows}x{self.ncols}@"
                f"({self.row_offset},{self.col_offset}))")


Mat = BitMatrix | MatrixWindow


class HostMatrix:
    """Host copy with the reference BitMatrix's read-only attribute surface
    (nrows, ncols, width, data, words, row_index, buf), so reference-side
    tooling such as gf2mat._reference.unpack_entries accepts it."""

    __slots__ = ("nrows", "ncols", "width", "words")

    def __init__(self, nrows: int, ncols: int, words: np.ndarray):
        self.nrows, self.ncols = nrows, ncols
        self.width = words_per_row(ncols)
        self.words = words

    @property
    def data(self) -> np.ndarray:
        return self.words.reshape(-1)

    buf = data

    @property
    def row_index(self) -> np.ndarray:
        return np.arange(self.nrows, dtype=np.int64) * self.width

    @property
    def shape(self):
        return (self.nrows, self.ncols)


def _to_host(m):
    """Owned host copy: a real `gf2mat.BitMatrix` (core.py:57-82, built with
    gf2mat.create and filled through its `words` view) when the caller has
    imported the reference package, else a HostMatrix with the same
    attribute surface. This package never imports gf2mat itself."""
    words = m.to_numpy()
    if words.size:
        # a window's last word may carry its parent's bits beyond the right
        # edge; an owned copy keeps the clean-tail invariant (core.py:335-341)
        words[:, -1] &= np.uint64(tail_mask(m.ncols))
    ref = sys.modules.get("gf2mat")
    if ref is not None and hasattr(ref, "create"):
        out = ref.create(m.nrows, m.ncols)
        if m.nrows and words.shape[1]:
            out.words[:, :] = words
        return out
    return HostMatrix(m.nrows, m.ncols, words)


def _stream():
    return _lib.current_stream()


_cur_dev = None


def _current_device() -> int:
    global _cur_dev
    if _cur_dev is None:
        c = _torch()._C
        _cur_dev = getattr(c, "_cuda_getDevice", None) or \
            _torch().cuda.current_device
    return _cur_dev()


def _check_cuda_dev(*mats):
    """Every operand on one device, and that device the current one: each
    operation runs on the current device's current stream, so device-1
    pointers launched from device 0 would fault (compared as indices,
    without building torch.device objects)."""
    d0 = _storage(mats[0]).get_device()
    for m in mats[1:]:
        if _storage(m).get_device() != d0:
            devs = {str(x.device) for x in mats}
            raise DimensionError(f"operands live on different devices: {devs}")
    cur = _current_device()
    if d0 != cur:
        raise DimensionError(
            f"operands live on cuda:{d0} but the current device is cuda:{cur}; "
            f"run under torch.cuda.device({d0})")


def _storage(m):
    if isinstance(m, BitMatrix):
        return m.storage
    if isinstance(m, MatrixWindow):
        return m.parent.storage
    raise TypeError(f"expected a device BitMatrix or MatrixWindow, got {type(m).__name__} "
                    "(upload host matrices with from_host)")


# ------------------------------------------------------------ constructors
def create(nrows: int, ncols: int, device=None) -> BitMatrix:
    """All-zero matrix (core.py:176-178)."""
    return BitMatrix(nrows, ncols, device)


def random(nrows: int, ncols: int, seed: int, device=None,
           row_base: int = 0) -> BitMatrix:
    """core.py:202-208 on device (splitmix64 over the flat word index).
    `row_base` produces rows [row_base, row_base + nrows) of a taller
    matrix with the same seed -- how row shards are generated in place."""
    m = BitMatrix(nrows, ncols, device)
    if m.nrows and m.width:
        _check_cuda_dev(m)
        _lib.check(_lib.lib_cuda().gf2_random(
            m._view(), seed & _FULL, row_base, _stream()))
    return m


def random_into(out: BitMatrix, seed: int, row_base: int = 0) -> None:
    """Refill an owned matrix with `random(out.nrows, out.ncols, seed,
    row_base=row_base)` in place (no allocation)."""
    if not isinstance(out, BitMatrix):
        raise TypeError("random_into fills an owned BitMatrix")
    if out.nrows and out.width:
        _check_cuda_dev(out)
        _lib.check(_lib.lib_cuda().gf2_random(
            out._view(), seed & _FULL, row_base, _stream()))


def bernoulli(nrows: int, ncols: int, seed: int, p: float | None = None,
              threshold: int | None = None, device=None,
              row_base: int = 0) -> BitMatrix:
    """Bernoulli(p) matrix of SURVEY.md §8(d) (cfg4): entry e = r*ncols + c
    is 1 iff splitmix64(seed, e) < floor(p * 2^64)."""
    if threshold is None:
        if p is None:
            raise ValueError("give p or threshold")
        from fractions import Fraction
        threshold = _FULL if p >= 1 else int(Fraction(str(p)) * (1 << 64))
    m = BitMatrix(nrows, ncols, device)
    if m.nrows and m.width:
        _check_cuda_dev(m)
        _lib.check(_lib.lib_cuda().gf2_bernoulli(
            m._view(), seed & _FULL, threshold & _FULL, row_base, _stream()))
    return m


def identity(n: int, device=None) -> BitMatrix:
    dense = np.eye(n, dtype=np.uint8)
    return from_dense(dense, device)


def window(a: Mat, row_offset: int, col_offset: int, nrows: int,
           ncols: int) -> MatrixWindow:
    """core.py:326-332 -- a window of a window flattens onto the root."""
    if isinstance(a, MatrixWindow):
        return MatrixWindow(a.parent, a.row_offset + row_offset,
                            a.col_offset + col_offset, nrows, ncols)
    return MatrixWindow(a, row_offset, col_offset, nrows, ncols)


# ------------------------------------------------------------ host interop
def from_numpy(words: np.ndarray, ncols: int, device=None,
               out: BitMatrix | None = None,
               nonblocking: bool = False) -> BitMatrix:
    """Upload (nrows, width) uint64 words (reference dense layout). The
    words are taken as-is (trailing bits must already be clean). With
    `nonblocking`, the copy is left in flight on the current stream: the
    caller keeps `words` alive (pinned memory makes it truly async)."""
    words = np.asarray(words)
    if words.dtype != np.uint64 or words.ndim != 2:
        raise DimensionError("from_numpy expects a 2-D uint64 array")
    nrows = words.shape[0]
    if words.shape[1] != words_per_row(ncols):
        raise DimensionError(
            f"{words.shape[1]} words per row for {ncols} columns")
    m = BitMatrix(nrows, ncols, device) if out is None else out
    if m.shape != (nrows, ncols):
        raise DimensionError(f"upload target {m.shape} != ({nrows}, {ncols})")
    if nrows and m.width:
        if words.strides[1] != 8 or words.strides[0] % 8:
            words = np.ascontiguousarray(words)
            nonblocking = False
        _check_cuda_dev(m)
        _lib.check(_lib.lib_cuda().gf2_upload(
            m._view(), words.ctypes.data, words.strides[0] // 8, _stream()))
        if not nonblocking:
            _torch().cuda.current_stream().synchronize()
    return m


def from_host(m, device=None) -> BitMatrix:
    """Upload anything with the reference's attribute surface
    (`nrows`, `ncols`, `words`): gf2mat.BitMatrix / MatrixWindow, HostMatrix.
    Window sources are copied with their right edge masked."""
    words = np.ascontiguousarray(np.asarray(m.words, dtype=np.uint64))
    if words.size:
        words = words.copy()
        words[:, -1] &= np.uint64(tail_mask(m.ncols))
    return from_numpy(words.reshape(m.nrows, words_per_row(m.ncols)), m.ncols,
                      device)


def _download(a: Mat, out: np.ndarray | None,
              nonblocking: bool = False) -> np.ndarray:
    w = words_per_row(a.ncols)
    if out is None:
        out = np.empty((a.nrows, w), dtype=np.uint64)
    if out.shape != (a.nrows, w) or out.dtype != np.uint64 \
            or out.strides[1] != 8:
        raise DimensionError(f"download buffer {out.shape} != ({a.nrows}, {w})")
    if a.nrows and w:
        _check_cuda_dev(a)
        _lib.check(_lib.lib_cuda().gf2_download(
            a._view(), out.ctypes.data, out.strides[0] // 8, _stream()))
        if not nonblocking:
            _torch().cuda.current_stream().synchronize()
    return out


def to_numpy(a: Mat) -> np.ndarray:
    """(nrows, width) uint64 words, raw (a window's last word may carry the
    parent's bits beyond its edge, exactly as `window.words` in core.py)."""
    return _download(a, None)


def to_dense(a: Mat) -> np.ndarray:
    """core.py:409-414"""
    if a.nrows == 0 or a.ncols == 0:
        return np.zeros((a.nrows, a.ncols), dtype=np.uint8)
    by = to_numpy(a).astype(">u8").view(np.uint8).reshape(a.nrows, -1)
    return np.unpackbits(by, axis=1, bitorder="big")[:, :a.ncols]


def from_dense(dense: np.ndarray, device=None) -> BitMatrix:
    """core.py:417-432"""
    dense = np.asarray(dense, dtype=np.uint8) & 1
    if dense.ndim != 2:
        raise DimensionError("from_dense expects a 2-D array")
    nrows, ncols = dense.shape
    w = words_per_row(ncols)
    if nrows == 0 or ncols == 0:
        return BitMatrix(nrows, ncols, device)
    packed = np.packbits(dense, axis=1, bitorder="big")
    if packed.shape[1] < w * 8:
        packed = np.pad(packed, ((0, 0), (0, w * 8 - packed.shape[1])))
    words = np.ascontiguousarray(packed).view(">u8").astype(np.uint64)
    return from_numpy(words.reshape(nrows, w), ncols, device)


# ------------------------------------------------------------ word ops
def add_into(out: Mat, a: Mat, b: Mat) -> None:
    """out = a XOR b; out may alias a or b (core.py:278-300)."""
    _check_cuda_dev(out, a, b)
    _lib.check(_lib.lib_cuda().gf2_add(out._view(), a._view(), b._view(),
                                       _stream()))


def add(a: Mat, b: Mat) -> BitMatrix:
    """core.py:303-309"""
    if a.shape != b.shape:
        raise DimensionError(f"add shapes {a.shape} and {b.shape} differ")
    out = BitMatrix(a.nrows, a.ncols, a.device)
    add_into(out, a, b)
    return out


def copy_into(out: Mat, a: Mat) -> None:
    """core.py:312-323 -- preserves bits beyond out's right edge."""
    if out.shape != a.shape:
        raise DimensionError(f"copy shapes {a.shape} -> {out.shape} differ")
    _check_cuda_dev(out, a)
    _lib.check(_lib.lib_cuda().gf2_copy(out._view(), a._view(), _stream()))


def copy_out(w: Mat) -> BitMatrix:
    """core.py:335-341 -- fresh owned copy with a clean tail."""
    out = BitMatrix(w.nrows, w.ncols, w.device)
    copy_into(out, w)
    return out


def zero_into(out: Mat) -> None:
    _check_cuda_dev(out)
    _lib.check(_lib.lib_cuda().gf2_zero(out._view(), _stream()))


def equal(a: Mat, b: Mat) -> bool:
    """core.py:379-388 -- entry equality (tails masked), on device."""
    if a.shape != b.shape:
        return False
    if a.nrows == 0 or a.width == 0:
        return True
    torch = _torch()
    wa, wb = a.words, b.words
    if wb.device != wa.device:
        wb = wb.to(wa.device)
    if not torch.equal(wa[:, :-1], wb[:, :-1]):
        return False
    tm = _signed(tail_mask(a.ncols))
    return bool(torch.equal(wa[:, -1] & tm, wb[:, -1] & tm))


def trailing_bits_clean(a: Mat) -> bool:
    """core.py:435-440"""
    if a.nrows == 0 or a.width == 0:
        return True
    spare = _signed(~tail_mask(a.ncols) & _FULL)
    return not bool((a.words[:, -1] & spare).any())


def first_difference(a: Mat, b: Mat):
    """core.py:391-406 (via host copies)."""
    if a.shape != b.shape:
        raise DimensionError(f"shapes {a.shape} and {b.shape} differ")
    if a.nrows == 0 or a.width == 0:
        return None
    diff = to_numpy(a) ^ to_numpy(b)
    diff[:, -1] &= np.uint64(tail_mask(a.ncols))
    rows = np.nonzero(diff.any(axis=1))[0]
    if rows.size == 0:
        return None
    r = int(rows[0])
    w = int(np.nonzero(diff[r])[0][0])
    word = int(diff[r, w])
    return (r, w * WORD_BITS + (WORD_BITS - word.bit_length()))
