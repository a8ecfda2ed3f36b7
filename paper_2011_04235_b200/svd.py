"""SVD engines -- the reference's svd.py API (``/root/reference/pkg/src/fastpi/svd.py``)
on the B200 core.  Factors stay in HBM; ``SvdFactors.U`` / ``.Vt`` are
materialised on the host on first access.
"""

from __future__ import annotations

import ctypes as C
import math
import struct
from pathlib import Path

import numpy as np
import scipy.sparse as sp

from . import _lib
from ._device import DeviceCSR, d2h, empty, h2d, torch
from .validation import BLOCK_CAPACITY, DENSE_CAPACITY, CapacityError, as_csr


class _Dense:
    """Device-resident dense factors: U (p x r), sigma (r), Vt (r x q), row-major float64."""

    kind = "dense"

    def __init__(self, U, sigma, Vt):
        self.U, self.sigma, self.Vt = U, sigma, Vt


class _Block:
    """Device-resident block-sparse factors (block_diagonal_svd): U, Vt as DeviceCSR."""

    kind = "block"

    def __init__(self, U: DeviceCSR, sigma, Vt: DeviceCSR):
        self.U, self.sigma, self.Vt = U, sigma, Vt


class SvdFactors:
    """Factor triplet ``U @ diag(sigma) @ Vt`` of a p x q matrix (svd.py:21-77)."""

    def __init__(self, U=None, sigma=None, Vt=None, is_sorted=True, *, _dev=None, _shape=None):
        self._dev = _dev
        self.is_sorted = bool(is_sorted)
        self._U = U
        self._Vt = Vt
        self._sigma = None
        if _dev is not None:
            # factors produced on the device: sigma is copied to the host on first access only, so a
            # stage hands its factors to the next one without draining the stream (the kernels emit
            # non-negative, and when flagged sorted, non-increasing sigma)
            if _shape is None:
                _shape = (int(_dev.U.shape[0]), int(_dev.Vt.shape[1]))
            self._shape = _shape
            return
        self._sigma = np.asarray(sigma, dtype=np.float64).ravel()
        if U.shape[1] != len(self._sigma) or Vt.shape[0] != len(self._sigma):
            raise ValueError(f"inconsistent factor shapes: U {U.shape}, sigma ({len(self._sigma)},), "
                             f"Vt {Vt.shape}")
        self._shape = (U.shape[0], Vt.shape[1])
        if len(self._sigma) and self._sigma.min() < 0:
            raise ValueError("singular values must be non-negative")
        if self.is_sorted and len(self._sigma) > 1 and np.any(np.diff(self._sigma) > 0):
            raise ValueError("factors flagged sorted but sigma is not non-increasing")

    @property
    def sigma(self) -> np.ndarray:
        if self._sigma is None:
            self._sigma = d2h(self._dev.sigma).astype(np.float64).ravel()
        return self._sigma

    @sigma.setter
    def sigma(self, value):
        self._sigma = np.asarray(value, dtype=np.float64).ravel()

    # -- host views (lazy) --------------------------------------------------
    @property
    def U(self):
        if self._U is None:
            self._U = self._dev.U.to_host() if self._dev.kind == "block" else d2h(self._dev.U)
        return self._U

    @property
    def Vt(self):
        if self._Vt is None:
            self._Vt = self._dev.Vt.to_host() if self._dev.kind == "block" else d2h(self._dev.Vt)
        return self._Vt

    @property
    def rank(self) -> int:
        if self._sigma is None:
            return int(self._dev.sigma.numel())
        return len(self._sigma)

    @property
    def shape(self) -> tuple:
        return self._shape

    # -- device view ----------------------------------------------------------
    def device(self):
        """Device representation (uploads host factors on first use)."""
        if self._dev is None:
            sig = h2d(self.sigma, np.float64)
            if sp.issparse(self._U) or sp.issparse(self._Vt):
                self._dev = _Block(DeviceCSR.from_host(sp.csr_matrix(self._U), canonicalize=False),
                                   sig, DeviceCSR.from_host(sp.csr_matrix(self._Vt), canonicalize=False))
            else:
                self._dev = _Dense(h2d(np.asarray(self._U, np.float64)), sig, h2d(np.asarray(self._Vt, np.float64)))
        return self._dev

    def orthonormality_defect(self) -> float:
        if self.rank == 0:
            return 0.0
        U = _to_dense(self.U)
        Vt = _to_dense(self.Vt)
        eye = np.eye(self.rank)
        return float(max(np.abs(U.T @ U - eye).max(), np.abs(Vt @ Vt.T - eye).max()))

    def validate(self, tol: float = 1e-10):
        defect = self.orthonormality_defect()
        if defect > tol:
            raise ValueError(f"factor orthonormality defect {defect:.3e} exceeds {tol:.1e}")
        return self

    def dense_reconstruction(self) -> np.ndarray:
        p, q = self.shape
        if p * q > DENSE_CAPACITY:
            raise CapacityError(f"reconstruction would materialize {p}x{q} entries")
        return (_to_dense(self.U) * self.sigma) @ _to_dense(self.Vt)

    def __repr__(self):
        return f"SvdFactors(shape={self.shape}, rank={self.rank}, sorted={self.is_sorted})"


def _to_dense(M) -> np.ndarray:
    if sp.issparse(M):
        return np.asarray(M.todense(), dtype=np.float64)
    return np.asarray(M, dtype=np.float64)


def gaussian_sketch_device(seed: int, rows: int, cols: int):
    """svd.py:131-132 -- numpy ``default_rng(seed).standard_normal((rows, cols))``, bitwise, in HBM."""
    X = empty((rows, cols), "f64")
    _lib.call("fpi_sketch_normal", int(seed), int(rows), int(cols), _lib.ptr(X), int(cols))
    return X


def _dense_device(A):
    t = torch()
    if _is_tensor(A):
        return A.to(t.float64).contiguous()
    if sp.issparse(A):
        if A.shape[0] * A.shape[1] > DENSE_CAPACITY:
            raise CapacityError(f"dense SVD of a {A.shape[0]}x{A.shape[1]} matrix exceeds the "
                                f"{DENSE_CAPACITY}-entry guard")
        A = A.toarray()
    A = np.asarray(A, dtype=np.float64)
    if A.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got ndim={A.ndim}")
    return h2d(A)


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def dense_svd_device(M, rank=None) -> SvdFactors:
    p, q = int(M.shape[0]), int(M.shape[1])
    if p * q > DENSE_CAPACITY:
        raise CapacityError(f"dense SVD of a {p}x{q} matrix exceeds the {DENSE_CAPACITY}-entry guard")
    if p * q and not bool(torch().isfinite(M).all()):
        raise ValueError("matrix contains non-finite entries")
    r = min(p, q) if rank is None else int(rank)
    U, sig, Vt = empty((p, r)), empty(r), empty((r, q))
    if r:
        _lib.call("fpi_dense_svd", p, q, _lib.ptr(M), q, r, _lib.ptr(U), _lib.ptr(sig), _lib.ptr(Vt))
    return SvdFactors(_dev=_Dense(U, sig, Vt), is_sorted=True, _shape=(p, q))


def dense_svd(A) -> SvdFactors:
    """svd.py:86-106: full-accuracy SVD of a dense (or densifiable) matrix."""
    return dense_svd_device(_dense_device(A))


def truncate(factors: SvdFactors, rank: int) -> SvdFactors:
    """svd.py:109-117: keep the leading ``rank`` triplets of sorted factors."""
    if not factors.is_sorted:
        raise ValueError("truncate requires sorted factors")
    if not 1 <= rank <= factors.rank:
        raise ValueError(f"target rank {rank} out of range [1, {factors.rank}]")
    d = factors.device()
    if d.kind != "dense":
        return SvdFactors(_to_dense(factors.U)[:, :rank], factors.sigma[:rank].copy(),
                          _to_dense(factors.Vt)[:rank, :], True)
    return SvdFactors(_dev=_Dense(d.U[:, :rank].contiguous(), d.sigma[:rank].clone(), d.Vt[:rank].contiguous()),
                      is_sorted=True, _shape=factors.shape)


def randomized_svd_device(Adev: DeviceCSR, rank: int, seed: int, At: DeviceCSR = None) -> SvdFactors:
    p, q = Adev.shape
    if not 1 <= rank <= min(p, q):
        raise ValueError(f"target rank {rank} out of range [1, {min(p, q)}]")
    At = At if At is not None else Adev.transpose()
    U, sig, Vt = empty((p, rank)), empty(rank), empty((rank, q))
    _lib.call("fpi_randomized_svd", p, q, _lib.ptr(Adev.indptr), _lib.ptr(Adev.indices), _lib.ptr(Adev.values),
              _lib.ptr(At.indptr), _lib.ptr(At.indices), _lib.ptr(At.values), int(rank), int(seed),
              _lib.ptr(U), _lib.ptr(sig), _lib.ptr(Vt))
    return SvdFactors(_dev=_Dense(U, sig, Vt), is_sorted=True, _shape=(p, q))


def randomized_svd(A, rank: int, seed: int) -> SvdFactors:
    """svd.py:120-138: Gaussian 2r sketch (numpy-exact), orthonormal basis, small SVD, lift."""
    dev = A if isinstance(A, DeviceCSR) else DeviceCSR.from_host(A)
    return randomized_svd_device(dev, rank, seed)


def block_diagonal_svd_device(a11: DeviceCSR, spans_dev, alpha: float) -> SvdFactors:
    """svd.py:141-193 on the spoke CSR + device span table (the hot path).  (A sharded solve
    factors only its own block range: fpi_block_svd_range, sharded.py.)"""
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"target rank ratio alpha must be in (0, 1], got {alpha}")
    m1, n1 = a11.shape
    nsp = int(spans_dev.numel() // 4)
    plan = _lib.BlockPlan()
    _lib.call("fpi_block_svd_plan", nsp, _lib.ptr(spans_dev), float(alpha), C.byref(plan))
    r = plan.rank11
    U = DeviceCSR.empty(m1, r, plan.nnz_u11)
    Vt = DeviceCSR.empty(r, n1, plan.nnz_vt11)
    sig = empty(r)
    _lib.call("fpi_block_svd", m1, n1, _lib.ptr(a11.indptr), _lib.ptr(a11.indices), _lib.ptr(a11.values), nsp,
              _lib.ptr(spans_dev), float(alpha), _lib.ptr(sig), _lib.ptr(U.indptr), _lib.ptr(U.indices),
              _lib.ptr(U.values), _lib.ptr(Vt.indptr), _lib.ptr(Vt.indices), _lib.ptr(Vt.values), C.byref(plan))
    return SvdFactors(_dev=_Block(U, sig, Vt), is_sorted=False, _shape=(m1, n1))


def block_diagonal_svd(blocks, alpha: float) -> SvdFactors:
    """svd.py:141-193: blocks is the list of diagonal blocks (dense or sparse)."""
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"target rank ratio alpha must be in (0, 1], got {alpha}")
    mats, spans = [], []
    ro = co = 0
    for b in blocks:
        h, w = b.shape
        if h and w and h * w > BLOCK_CAPACITY:
            raise CapacityError(f"diagonal block of {h}x{w} entries exceeds the {BLOCK_CAPACITY}-entry "
                                "guard; reordering produced a pathological block")
        mats.append(sp.csr_matrix(b) if not sp.issparse(b) else b.tocsr())
        spans.append((ro, h, co, w))
        ro += h
        co += w
    spoke = sp.block_diag(mats, format="csr") if mats else sp.csr_matrix((0, 0))
    spoke = sp.csr_matrix(spoke, shape=(ro, co))
    dev = DeviceCSR.from_host(spoke)
    spans_dev = h2d(np.asarray(spans, np.int64).reshape(-1), np.int64)
    return block_diagonal_svd_device(dev, spans_dev, alpha)


def reconstruction_error(A, factors: SvdFactors, chunk: int = 1 << 20) -> float:
    """svd.py:196-223: ||A - U diag(sigma) Vt||_F via ||A||^2 - 2<A,B> + ||B||^2.

    A parity-check utility, not part of the solve: the products run
    on the library's SpMM / GEMM, the final r x r reductions on torch."""
    del chunk
    dev = A if isinstance(A, DeviceCSR) else DeviceCSR.from_host(A)
    t = torch()
    na = float(t.dot(dev.values, dev.values).item()) if dev.nnz else 0.0
    if factors.rank == 0:
        return math.sqrt(na)
    d = factors.device()
    if d.kind != "dense":
        U = h2d(_to_dense(factors.U))
        Vt = h2d(_to_dense(factors.Vt))
        sig = d.sigma
    else:
        U, sig, Vt = d.U, d.sigma, d.Vt
    p, q = dev.shape
    r = factors.rank
    # cross = sum_k sigma_k u_k^T A v_k ;  P = A Vt^T (p x r)
    Vtt = Vt.t().contiguous()   # check path only (a16): a transposed copy
    P = empty((p, r))
    _lib.call("fpi_spmm", p, q, r, _lib.ptr(dev.indptr), _lib.ptr(dev.indices), _lib.ptr(dev.values), 1.0,
              _lib.ptr(Vtt), r, 0.0, _lib.ptr(P), r)
    cross = float(((U * P).sum(dim=0) * sig).sum().item())
    GU = empty((r, r))
    GV = empty((r, r))
    _lib.call("fpi_gemm", 1, 0, r, r, p, 1.0, _lib.ptr(U), r, _lib.ptr(U), r, 0.0, _lib.ptr(GU), r)
    _lib.call("fpi_gemm", 0, 1, r, r, q, 1.0, _lib.ptr(Vt), q, _lib.ptr(Vt), q, 0.0, _lib.ptr(GV), r)
    nb = float((sig[:, None] * sig[None, :] * GU * GV).sum().item())
    return math.sqrt(max(na - 2.0 * cross + nb, 0.0))


_HEADER = struct.Struct("<QQQB")


def save_factors(factors: SvdFactors, path):
    """svd.py:226-238 binary layout."""
    p, q = factors.shape
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(p, q, factors.rank, 1 if factors.is_sorted else 0))
        fh.write(np.ascontiguousarray(_to_dense(factors.U), dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(factors.sigma, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(_to_dense(factors.Vt), dtype="<f8").tobytes())


def load_factors(path) -> SvdFactors:
    """svd.py:241-250."""
    raw = Path(path).read_bytes()
    p, q, r, flag = _HEADER.unpack_from(raw, 0)
    off = _HEADER.size
    U = np.frombuffer(raw, dtype="<f8", count=p * r, offset=off).reshape(p, r)
    off += 8 * p * r
    sigma = np.frombuffer(raw, dtype="<f8", count=r, offset=off)
    off += 8 * r
    Vt = np.frombuffer(raw, dtype="<f8", count=r * q, offset=off).reshape(r, q)
    return SvdFactors(U.copy(), sigma.copy(), Vt.copy(), bool(flag))
