"""Device-resident containers and host<->device plumbing.

Matrices live in HBM as torch tensors in the library's layouts:
CSR = (int64 indptr, int32 indices, float64 values); dense = row-major
float64.  Host copies are made only when a caller asks for them.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _lib
from .validation import as_csr


def torch():
    return _lib._torch()


def device():
    t = torch()
    return t.device("cuda", t.cuda.current_device())


_H2D_CHUNK = 16 << 20


def h2d(arr: np.ndarray, dtype=None):
    """Host numpy -> device tensor (through pinned memory, async on the current stream).  Large
    arrays are staged into a page-locked block from torch's caching host allocator by a parallel
    (intra-op threads) copy; the allocator keeps the block until the stream has consumed it."""
    t = torch()
    a = np.ascontiguousarray(arr if dtype is None else arr.astype(dtype, copy=False))
    host = t.from_numpy(a)
    if a.nbytes >= 2 * _H2D_CHUNK:
        # chunked: the staging copy of chunk k runs while the DMA of chunk k - 1 is in flight, so the
        # upload costs the staging pass plus one chunk's transfer instead of staging + the whole transfer
        dev = t.empty(host.shape, dtype=host.dtype, device=device())
        fh, fd = host.reshape(-1), dev.view(-1)
        step = max(1, _H2D_CHUNK // a.itemsize)
        for off in range(0, fh.numel(), step):
            n = min(step, fh.numel() - off)
            staged = t.empty(n, dtype=host.dtype, pin_memory=True)
            staged.copy_(fh[off:off + n])
            fd[off:off + n].copy_(staged, non_blocking=True)
        return dev
    if a.nbytes >= (1 << 20):
        staged = t.empty(host.shape, dtype=host.dtype, pin_memory=True)
        staged.copy_(host)
        host = staged
    return host.to(device(), non_blocking=True)


def d2h(t_) -> np.ndarray:
    """Device tensor -> numpy through page-locked memory (torch's caching host allocator)."""
    t = torch()
    if t_.numel() * t_.element_size() < (1 << 20):
        return t_.detach().to("cpu").numpy()
    host = t.empty(t_.shape, dtype=t_.dtype, pin_memory=True)
    host.copy_(t_.detach())
    return host.numpy()


def empty(shape, dtype="f64"):
    t = torch()
    dt = {"f64": t.float64, "i64": t.int64, "i32": t.int32, "u8": t.uint8}[dtype]
    return t.empty(shape, dtype=dt, device=device())


def zeros(shape, dtype="f64"):
    t = torch()
    dt = {"f64": t.float64, "i64": t.int64, "i32": t.int32}[dtype]
    return t.zeros(shape, dtype=dt, device=device())


class DeviceCSR:
    """Canonical CSR in HBM: sorted indices, no duplicates, no explicit zeros."""

    __slots__ = ("shape", "indptr", "indices", "values")

    def __init__(self, shape, indptr, indices, values):
        self.shape = (int(shape[0]), int(shape[1]))
        self.indptr = indptr
        self.indices = indices
        self.values = values

    @property
    def nnz(self) -> int:
        return int(self.indices.numel())

    @classmethod
    def empty(cls, p, q, nnz):
        return cls((p, q), empty(p + 1, "i64"), empty(max(nnz, 0), "i32"), empty(max(nnz, 0), "f64"))

    @classmethod
    def from_host(cls, A, canonicalize: bool = True) -> "DeviceCSR":
        """Upload a scipy/array matrix; check_csr's canonicalisation runs on the GPU."""
        A = as_csr(A)
        m, n = A.shape
        raw = cls((m, n), h2d(A.indptr, np.int64), h2d(A.indices, np.int32), h2d(A.data, np.float64))
        if not canonicalize:
            return raw
        return raw.canonical()

    def canonical(self) -> "DeviceCSR":
        m, n = self.shape
        out = DeviceCSR.empty(m, n, self.nnz)
        kept = C.c_int64(0)
        _lib.call("fpi_csr_canonicalize", m, n, self.nnz, _lib.ptr(self.indptr), _lib.ptr(self.indices),
                  _lib.ptr(self.values), _lib.ptr(out.indptr), _lib.ptr(out.indices), _lib.ptr(out.values),
                  C.byref(kept))
        k = int(kept.value)
        if k != self.nnz:
            out.indices = out.indices[:k]
            out.values = out.values[:k]
        return out

    def transpose(self) -> "DeviceCSR":
        p, q = self.shape
        out = DeviceCSR.empty(q, p, self.nnz)
        _lib.call("fpi_csr_transpose", p, q, self.nnz, _lib.ptr(self.indptr), _lib.ptr(self.indices),
                  _lib.ptr(self.values), _lib.ptr(out.indptr), _lib.ptr(out.indices), _lib.ptr(out.values))
        return out

    def row_slice(self, r0: int, r1: int) -> "DeviceCSR":
        """Rows [r0, r1) as a CSR view with rebased row pointers."""
        ptr = self.indptr[r0:r1 + 1]
        b = int(ptr[0].item()) if r1 > r0 else 0
        e = int(ptr[-1].item()) if r1 > r0 else 0
        return DeviceCSR((r1 - r0, self.shape[1]), ptr - b, self.indices[b:e], self.values[b:e])

    def to_host(self) -> sp.csr_matrix:
        return sp.csr_matrix((d2h(self.values), d2h(self.indices), d2h(self.indptr)), shape=self.shape)
