"""Host-buffer multiply pipeline: C_i = A_i . B_i for a stream of host
matrices, with PCIe copies overlapped with compute.

Serving-style use of the drop-in API (each product is what
`mul_strassen(from_numpy(A_i), from_numpy(B_i)).to_numpy()` returns),
scheduled over three CUDA streams and two device buffer sets:

    h2d stream     : upload A_i, B_i into set i%2        (copy engine H2D)
    compute stream : C_i = A_i . B_i (Strassen-Winograd)  (SMs)
    d2h stream     : download C_i into the caller's host buffer (copy engine D2H)

Step i's uploads overlap step i-1's compute; step i's download overlaps step
i+1's compute. Events order reuse of each buffer set. Host buffers should be
pinned (torch `pin_memory=True` tensors viewed as numpy) for the copies to
be asynchronous.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import BitMatrix, words_per_row
from .errors import DimensionError
from .strassen import MulParams, default_params


class HostPipeline:
    """Double-buffered host->device->host multiply pipeline for fixed shapes
    (m x l) . (l x n)."""

    def __init__(self, m: int, l: int, n: int,
                 params: MulParams | None = None, device=None):
        import torch
        self.m, self.l, self.n = m, l, n
        self.params = params or default_params()
        self.device = device if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        self.h2d = torch.cuda.Stream(self.device)
        self.comp = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.sets = [(BitMatrix(m, l, self.device), BitMatrix(l, n, self.device),
                      BitMatrix(m, n, self.device)) for _ in range(2)]
        ev = lambda: torch.cuda.Event()  # noqa: E731
        self.uploaded = [ev(), ev()]
        self.computed = [ev(), ev()]
        self.downloaded = [ev(), ev()]
        self.used = [False, False]
        self.i = 0

    def _check(self, arr: np.ndarray, rows: int, cols: int, what: str):
        if arr.dtype != np.uint64 or arr.shape != (rows, words_per_row(cols)):
            raise DimensionError(
                f"{what}: expected uint64 ({rows}, {words_per_row(cols)}), "
                f"got {arr.dtype} {arr.shape}")

    def submit(self, a_words: np.ndarray, b_words: np.ndarray,
               c_out: np.ndarray, c_in: np.ndarray | None = None) -> None:
        """Queue C = A.B -- or, with `c_in`, C = C_in + A.B (the addmul of
        cfg4 / cfg5: C_in is uploaded with A and B and the product is XORed
        into it); c_out is filled once `sync()` (or a later `submit` that
        reuses this buffer set) has completed."""
        import torch
        self._check(a_words, self.m, self.l, "A")
        self._check(b_words, self.l, self.n, "B")
        self._check(c_out, self.m, self.n, "C")
        if c_in is not None:
            self._check(c_in, self.m, self.n, "C_in")
        k = self.i % 2
        a, b, c = self.sets[k]
        lib = _lib.lib_cuda()
        with torch.cuda.stream(self.h2d):
            if self.used[k]:
                self.h2d.wait_event(self.computed[k])      # set k's A, B consumed
            s = self.h2d.cuda_stream
            _lib.check(lib.gf2_upload(a._view(), a_words.ctypes.data,
                                      a_words.strides[0] // 8, s))
            _lib.check(lib.gf2_upload(b._view(), b_words.ctypes.data,
                                      b_words.strides[0] // 8, s))
            if c_in is not None:
                if self.used[k]:
                    self.h2d.wait_event(self.downloaded[k])  # set k's C read out
                _lib.check(lib.gf2_upload(c._view(), c_in.ctypes.data,
                                          c_in.strides[0] // 8, s))
            self.uploaded[k].record(self.h2d)
        with torch.cuda.stream(self.comp):
            self.comp.wait_event(self.uploaded[k])
            if self.used[k]:
                self.comp.wait_event(self.downloaded[k])   # set k's C read out
            _lib.check(lib.gf2_strassen(
                c._view(), a._view(), b._view(), int(self.params.cutoff),
                int(self.params.k), int(c_in is not None), self.comp.cuda_stream))
            self.computed[k].record(self.comp)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.computed[k])
            _lib.check(lib.gf2_download(c._view(), c_out.ctypes.data,
                                        c_out.strides[0] // 8,
                                        self.d2h.cuda_stream))
            self.downloaded[k].record(self.d2h)
        self.used[k] = True
        self.i += 1

    def sync(self) -> None:
        """Wait until every submitted product has landed in its host buffer."""
        self.d2h.synchronize()

    @property
    def streams(self):
        return self.h2d, self.comp, self.d2h


class ShardedHostPipeline:
    """HostPipeline for one rank of a row-sharded multi-GPU multiply
    (sharded.py): per product this rank uploads its rows of A and its block
    of B's rows (`owned_rows(l, world, rank, None)`) over its own PCIe link,
    `mul_sharded(src=None)` broadcasts every rank's block over NCCL while the
    K-panels multiply, and the rank downloads its rows of C. Same three
    streams, two buffer sets and event ordering as HostPipeline; every rank
    of the group calls `submit` for every product, in the same order."""

    def __init__(self, m_shard: int, l: int, n: int,
                 params: MulParams | None = None, device=None, group=None,
                 npanels: int = 2):
        import torch
        import torch.distributed as dist
        from .sharded import owned_rows
        self.m, self.l, self.n = m_shard, l, n
        self.params = params or default_params()
        self.group, self.npanels = group, npanels
        self.device = device if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self.owned = owned_rows(l, world, rank, None)
        self.h2d = torch.cuda.Stream(self.device)
        self.comp = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)
        self.sets = [(BitMatrix(m_shard, l, self.device), BitMatrix(l, n, self.device),
                      BitMatrix(m_shard, n, self.device)) for _ in range(2)]
        ev = lambda: torch.cuda.Event()  # noqa: E731
        self.uploaded = [ev(), ev()]
        self.computed = [ev(), ev()]
        self.downloaded = [ev(), ev()]
        self.used = [False, False]
        self.i = 0

    def submit(self, a_words: np.ndarray, b_words: np.ndarray,
               c_out: np.ndarray, c_in: np.ndarray | None = None) -> None:
        """Queue C_p = A_p . B (or, with `c_in`, C_p = C_in,p + A_p . B).
        `a_words`: this rank's rows of A; `b_words`: (l, width) with at
        least this rank's block of rows filled (the rest is not read);
        `c_in` / `c_out`: this rank's rows of C."""
        import torch
        from .core import window
        from .sharded import mul_sharded
        HostPipeline._check(self, a_words, self.m, self.l, "A")
        HostPipeline._check(self, b_words, self.l, self.n, "B")
        HostPipeline._check(self, c_out, self.m, self.n, "C")
        if c_in is not None:
            HostPipeline._check(self, c_in, self.m, self.n, "C_in")
        k = self.i % 2
        a, b, c = self.sets[k]
        lib = _lib.lib_cuda()
        with torch.cuda.stream(self.h2d):
            if self.used[k]:
                self.h2d.wait_event(self.computed[k])      # set k consumed
            s = self.h2d.cuda_stream
            _lib.check(lib.gf2_upload(a._view(), a_words.ctypes.data,
                                      a_words.strides[0] // 8, s))
            for k0, k1 in self.owned:
                _lib.check(lib.gf2_upload(
                    window(b, k0, 0, k1 - k0, self.n)._view(),
                    b_words[k0:k1].ctypes.data, b_words.strides[0] // 8, s))
            if c_in is not None:
                if self.used[k]:
                    self.h2d.wait_event(self.downloaded[k])  # set k's C read out
                _lib.check(lib.gf2_upload(c._view(), c_in.ctypes.data,
                                          c_in.strides[0] // 8, s))
            self.uploaded[k].record(self.h2d)
        with torch.cuda.stream(self.comp):
            self.comp.wait_event(self.uploaded[k])
            if self.used[k]:
                self.comp.wait_event(self.downloaded[k])   # set k's C read out
            mul_sharded(a, b, self.params, src=None, group=self.group,
                        npanels=self.npanels, c=c, accumulate=c_in is not None)
            self.computed[k].record(self.comp)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(self.computed[k])
            _lib.check(lib.gf2_download(c._view(), c_out.ctypes.data,
                                        c_out.strides[0] // 8,
                                        self.d2h.cuda_stream))
            self.downloaded[k].record(self.d2h)
        self.used[k] = True
        self.i += 1

    def sync(self) -> None:
        self.d2h.synchronize()

    @property
    def streams(self):
        return self.h2d, self.comp, self.d2h
