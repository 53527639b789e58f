"""GF2M matrix files straight to / from device matrices (core.py:443-484):
magic "GF2M", version byte 0x01, nrows and ncols as little-endian u64, then
nrows * ceil(ncols/64) little-endian words, trailing bits zero. Same checks,
messages and byte offsets as the reference's `save` / `load`."""

from __future__ import annotations

import os

import numpy as np

from .core import BitMatrix, Mat, from_numpy, tail_mask, to_numpy, words_per_row
from .errors import FormatError

_MAGIC = b"GF2M"
_VERSION = 1
_HEADER = 4 + 1 + 8 + 8


def save(a: Mat, path) -> None:
    """core.py:443-452 -- writes the window contents with a masked tail."""
    header = (_MAGIC + bytes([_VERSION]) + int(a.nrows).to_bytes(8, "little")
              + int(a.ncols).to_bytes(8, "little"))
    body = to_numpy(a) if a.nrows and a.ncols else \
        np.zeros((a.nrows, words_per_row(a.ncols)), dtype=np.uint64)
    if body.size:
        body[:, -1] &= np.uint64(tail_mask(a.ncols))
    with open(path, "wb") as fh:
        fh.write(header)
        fh.write(body.astype("<u8").tobytes())


def load(path, device=None) -> BitMatrix:
    """core.py:455-484 -- rejects bad magic, version, size or dirty bits,
    naming the byte offset; the words are uploaded to HBM."""
    with open(os.fspath(path), "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEADER:
        raise FormatError(f"truncated header at offset {len(raw)}")
    if raw[:4] != _MAGIC:
        raise FormatError("bad magic at offset 0")
    if raw[4] != _VERSION:
        raise FormatError(f"unsupported version {raw[4]} at offset 4")
    nrows = int.from_bytes(raw[5:13], "little")
    ncols = int.from_bytes(raw[13:21], "little")
    width = words_per_row(ncols)
    expect = _HEADER + nrows * width * 8
    if len(raw) != expect:
        raise FormatError(
            f"file length {len(raw)} != expected {expect} at offset "
            f"{min(len(raw), expect)}")
    words = np.frombuffer(raw, dtype="<u8", offset=_HEADER) \
        .astype(np.uint64).reshape(nrows, width)
    if words.size:
        spare = ~np.uint64(tail_mask(ncols))
        dirty = np.nonzero(words[:, -1] & spare)[0]
        if dirty.size:
            r = int(dirty[0])
            off = _HEADER + (r * width + width - 1) * 8
            raise FormatError(f"dirty trailing bits in row {r} at offset {off}")
    return from_numpy(np.ascontiguousarray(words), ncols, device)
