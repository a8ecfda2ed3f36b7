"""FastPI driver, incremental updates and pseudoinverse assembly -- the
reference's pinv.py API (``/root/reference/pkg/src/fastpi/pinv.py``) on the
B200 core.  Every stage runs in HBM; the returned objects expose the
reference's numpy / scipy attributes lazily.
"""

from __future__ import annotations

import ctypes as C
import math
import struct
import time
import warnings
from dataclasses import dataclass
from pathlib import Path
from typing import NamedTuple

import numpy as np
import scipy.sparse as sp

from . import _lib
from ._device import DeviceCSR, d2h, empty, h2d, torch
from .reorder import Permutation, ReorderResult, partition_original, reorder_device
from .svd import SvdFactors, _Dense, _to_dense, block_diagonal_svd_device, dense_svd, truncate
from .validation import DENSE_CAPACITY, CapacityError, as_csr

EPS = float(np.finfo(np.float64).eps)

STAGES = ("reorder", "block_svd", "row_update", "column_update", "pinv_assembly")


@dataclass(frozen=True)
class FastpiConfig:
    """pinv.py:32-46."""

    alpha: float = 1.0
    k: float = 0.01
    seed: int = 0
    low_rank_threshold: float = 0.3
    pinv_cutoff_factor: float = EPS

    def __post_init__(self):
        if not 0.0 < self.alpha <= 1.0:
            raise ValueError(f"alpha must be in (0, 1], got {self.alpha}")
        if not 0.0 < self.k < 1.0:
            raise ValueError(f"k must be in (0, 1), got {self.k}")


class _DevPinv:
    """Pseudoinverse factors in reordered coordinates: U (m x r), sdag (r), Vt (r x n) + permutations."""

    def __init__(self, U, sdag, Vt, row_fwd, col_fwd):
        self.U, self.sdag, self.Vt, self.row_fwd, self.col_fwd = U, sdag, Vt, row_fwd, col_fwd
        self.m, self.r = int(U.shape[0]), int(U.shape[1])
        self.n = int(Vt.shape[1])


class Pseudoinverse:
    """Factored pseudoinverse ``V @ diag(sigma_dagger) @ Ut`` of an m x n matrix (pinv.py:49-92)."""

    def __init__(self, V=None, sigma_dagger=None, Ut=None, tolerance_used=0.0, all_filtered=False, *, _dev=None):
        self._dev = _dev
        self._V = None if V is None else np.asarray(V, dtype=np.float64)
        self._Ut = None if Ut is None else np.asarray(Ut, dtype=np.float64)
        if sigma_dagger is None and _dev is not None:
            sigma_dagger = d2h(_dev.sdag)
        self.sigma_dagger = np.asarray(sigma_dagger, dtype=np.float64).ravel()
        self.tolerance_used = float(tolerance_used)
        self.all_filtered = bool(all_filtered)

    def _device(self) -> _DevPinv:
        if self._dev is None:
            t = torch()
            n, r = self._V.shape
            m = self._Ut.shape[1]
            dev = t.device("cuda", t.cuda.current_device())
            U = h2d(np.ascontiguousarray(self._Ut.T))
            Vt = h2d(np.ascontiguousarray(self._V.T))
            self._dev = _DevPinv(U, h2d(self.sigma_dagger), Vt, t.arange(m, device=dev, dtype=t.int64),
                                 t.arange(n, device=dev, dtype=t.int64))
        return self._dev

    def _unfold(self, want_v: bool):
        d = self._dev
        out = empty((d.n, d.r)) if want_v else empty((d.r, d.m))
        _lib.call("fpi_unfold", d.m, d.n, d.r, _lib.ptr(d.U), _lib.ptr(d.Vt), _lib.ptr(d.row_fwd),
                  _lib.ptr(d.col_fwd), _lib.ptr(out) if want_v else None, None if want_v else _lib.ptr(out))
        return d2h(out)

    @property
    def V(self) -> np.ndarray:
        if self._V is None:
            self._V = self._unfold(True)
        return self._V

    @property
    def Ut(self) -> np.ndarray:
        if self._Ut is None:
            self._Ut = self._unfold(False)
        return self._Ut

    @property
    def shape(self) -> tuple:
        if self._dev is not None:
            return (self._dev.n, self._dev.m)
        return (self._V.shape[0], self._Ut.shape[1])

    @property
    def retained_rank(self) -> int:
        return int(np.count_nonzero(self.sigma_dagger))

    def apply_device(self, B):
        """pinv @ B for a device operand (DeviceCSR or dense tensor); returns a device tensor."""
        d = self._device()
        if isinstance(B, DeviceCSR):
            if B.shape[0] != d.m:
                raise ValueError(f"dimension mismatch: pseudoinverse expects {d.m} rows, got {B.shape[0]}")
            L = B.shape[1]
            Z = empty((d.n, L))
            _lib.call("fpi_pinv_apply_csr", d.m, d.n, d.r, _lib.ptr(d.U), _lib.ptr(d.sdag), _lib.ptr(d.Vt),
                      _lib.ptr(d.row_fwd), _lib.ptr(d.col_fwd), L, B.nnz, _lib.ptr(B.indptr), _lib.ptr(B.indices),
                      _lib.ptr(B.values), _lib.ptr(Z))
            return Z
        t = torch()
        Bd = B.to(t.float64).contiguous()
        vec = Bd.dim() == 1
        if vec:
            Bd = Bd.reshape(-1, 1)
        if Bd.shape[0] != d.m:
            raise ValueError(f"dimension mismatch: pseudoinverse expects {d.m} rows, got {Bd.shape[0]}")
        L = int(Bd.shape[1])
        Z = empty((d.n, L))
        _lib.call("fpi_pinv_apply_dense", d.m, d.n, d.r, _lib.ptr(d.U), _lib.ptr(d.sdag), _lib.ptr(d.Vt),
                  _lib.ptr(d.row_fwd), _lib.ptr(d.col_fwd), L, _lib.ptr(Bd), L, _lib.ptr(Z))
        return Z.reshape(-1) if vec else Z

    def apply(self, B) -> np.ndarray:
        """pinv.py:72-81: ``pinv @ B`` right-to-left without materialising pinv."""
        if sp.issparse(B):
            return self._apply_csr_to_host(DeviceCSR.from_host(B))
        elif isinstance(B, DeviceCSR) or type(B).__module__.startswith("torch"):
            Z = self.apply_device(B)
        else:
            Z = self.apply_device(h2d(np.asarray(B, dtype=np.float64)))
        return d2h(Z)

    def _apply_csr_to_host(self, Bd: DeviceCSR) -> np.ndarray:
        """Sparse ``pinv @ B`` returned in host memory: the lift's row chunks are copied out while the
        next chunk computes (fpi_pinv_apply_csr_host), into page-locked memory."""
        d = self._device()
        if Bd.shape[0] != d.m:
            raise ValueError(f"dimension mismatch: pseudoinverse expects {d.m} rows, got {Bd.shape[0]}")
        t = torch()
        L = Bd.shape[1]
        try:
            Zh = t.empty((d.n, L), dtype=t.float64, pin_memory=True)
        except RuntimeError:  # page-locked memory exhausted: pageable copies are still correct
            Zh = t.empty((d.n, L), dtype=t.float64)
        _lib.call("fpi_pinv_apply_csr_host", d.m, d.n, d.r, _lib.ptr(d.U), _lib.ptr(d.sdag), _lib.ptr(d.Vt),
                  _lib.ptr(d.row_fwd), _lib.ptr(d.col_fwd), L, Bd.nnz, _lib.ptr(Bd.indptr), _lib.ptr(Bd.indices),
                  _lib.ptr(Bd.values), Zh.data_ptr())
        return Zh.numpy()

    def validate(self, tol: float = 1e-8):
        r = len(self.sigma_dagger)
        if r:
            V, Ut = self.V, self.Ut
            defect = max(np.abs(V.T @ V - np.eye(r)).max(), np.abs(Ut @ Ut.T - np.eye(r)).max())
            if defect > tol:
                raise ValueError(f"pseudoinverse factor defect {defect:.3e} exceeds {tol:.1e}")
        return self


class StageTime(NamedTuple):
    stage: str
    seconds: float
    rank: int


class FastpiResult(NamedTuple):
    """pinv.py:101-108."""

    pseudoinverse: Pseudoinverse
    factors: SvdFactors
    reordering: ReorderResult
    timings: list


def _empty_factors(p: int, q: int) -> SvdFactors:
    return SvdFactors(np.zeros((p, 0)), np.zeros(0), np.zeros((0, q)), is_sorted=True)


def _csr_of(f_mat) -> DeviceCSR:
    """Device CSR of a factor matrix (block CSR, scipy, numpy or dense tensor)."""
    if isinstance(f_mat, DeviceCSR):
        return f_mat
    if type(f_mat).__module__.startswith("torch"):
        f_mat = d2h(f_mat)
    return DeviceCSR.from_host(sp.csr_matrix(f_mat), canonicalize=False)


def row_update_device(f11: SvdFactors, a21: DeviceCSR, s: int, *, low_rank_threshold=0.3, seed=0):
    """pinv.py:131-171 with device operands; returns (SvdFactors, engine)."""
    m2, n1 = a21.shape
    m1 = f11.shape[0]
    if f11.shape[1] != n1:
        raise ValueError(f"dimension mismatch: factors cover {f11.shape[1]} columns, appended rows have {n1}")
    r_avail = f11.rank
    max_rank = min(r_avail + m2, n1)
    if s == 0:
        return _empty_factors(m1 + m2, n1), 0
    if not 1 <= s <= max_rank:
        raise ValueError(f"target rank {s} out of range [1, {max_rank}]")
    d = f11.device()
    if d.kind == "block":
        Ucsr, Vcsr = d.U, d.Vt
    else:
        Ucsr, Vcsr = _csr_of(d.U), _csr_of(d.Vt)
    m = m1 + m2
    U, sig, Vt = empty((m, s)), empty(s), empty((s, n1))
    eng = C.c_int32(0)
    _lib.call("fpi_row_update", m1, n1, r_avail, _lib.ptr(d.sigma), _lib.ptr(Ucsr.indptr), _lib.ptr(Ucsr.indices),
              _lib.ptr(Ucsr.values), _lib.ptr(Vcsr.indptr), _lib.ptr(Vcsr.indices), _lib.ptr(Vcsr.values), m2,
              _lib.ptr(a21.indptr), _lib.ptr(a21.indices), _lib.ptr(a21.values), int(s), float(low_rank_threshold),
              int(seed), _lib.ptr(U), _lib.ptr(sig), _lib.ptr(Vt), C.byref(eng))
    return SvdFactors(_dev=_Dense(U, sig, Vt), is_sorted=True, _shape=(m, n1)), int(eng.value)


def row_update(f11: SvdFactors, A_below, s: int, *, low_rank_threshold: float = 0.3, seed: int = 0) -> SvdFactors:
    """pinv.py:131-171: factors of [A11; A_below] from factors of A11."""
    a21 = A_below if isinstance(A_below, DeviceCSR) else DeviceCSR.from_host(A_below)
    return row_update_device(f11, a21, s, low_rank_threshold=low_rank_threshold, seed=seed)[0]


def column_update_device(f: SvdFactors, T: DeviceCSR, Tt: DeviceCSR, r: int, *, low_rank_threshold=0.3, seed=0):
    """pinv.py:174-208 with device operands; returns (SvdFactors, engine)."""
    m, n2 = T.shape
    if f.shape[0] != m:
        raise ValueError(f"dimension mismatch: factors cover {f.shape[0]} rows, appended columns have {m}")
    s_prev = f.rank
    n1 = f.shape[1]
    max_rank = min(s_prev + n2, m)
    if r == 0:
        return _empty_factors(m, n1 + n2), 0
    if not 1 <= r <= max_rank:
        raise ValueError(f"target rank {r} out of range [1, {max_rank}]")
    d = f.device()
    if d.kind != "dense":
        d = _Dense(h2d(_to_dense(f.U)), d.sigma, h2d(_to_dense(f.Vt)))
    U, sig, Vt = empty((m, r)), empty(r), empty((r, n1 + n2))
    eng = C.c_int32(0)
    _lib.call("fpi_column_update", m, s_prev, n1, _lib.ptr(d.U), _lib.ptr(d.sigma), _lib.ptr(d.Vt), n2,
              _lib.ptr(T.indptr), _lib.ptr(T.indices), _lib.ptr(T.values), _lib.ptr(Tt.indptr),
              _lib.ptr(Tt.indices), _lib.ptr(Tt.values), int(r), float(low_rank_threshold), int(seed),
              _lib.ptr(U), _lib.ptr(sig), _lib.ptr(Vt), C.byref(eng))
    return SvdFactors(_dev=_Dense(U, sig, Vt), is_sorted=True, _shape=(m, n1 + n2)), int(eng.value)


def column_update(f: SvdFactors, T, r: int, *, low_rank_threshold: float = 0.3, seed: int = 0) -> SvdFactors:
    """pinv.py:174-208: factors of [A_left | T] from factors of A_left."""
    Td = T if isinstance(T, DeviceCSR) else DeviceCSR.from_host(T)
    return column_update_device(f, Td, Td.transpose(), r, low_rank_threshold=low_rank_threshold, seed=seed)[0]


def _assemble(f: SvdFactors, row_fwd, col_fwd, cutoff_factor: float) -> Pseudoinverse:
    d = f.device()
    r = f.rank
    p, q = f.shape
    sdag = empty(r)
    tol = C.c_double(0.0)
    af = C.c_int32(0)
    _lib.call("fpi_pinv_assemble", r, _lib.ptr(d.sigma), p, q, float(cutoff_factor), _lib.ptr(sdag),
              C.byref(tol), C.byref(af))
    if af.value:
        warnings.warn("all singular values filtered; returning the zero pseudoinverse")
    return Pseudoinverse(tolerance_used=tol.value, all_filtered=bool(af.value),
                         _dev=_DevPinv(d.U, sdag, d.Vt, row_fwd, col_fwd))


def pinv_from_svd(factors: SvdFactors, cutoff_factor: float = EPS) -> Pseudoinverse:
    """pinv.py:211-231."""
    if not factors.is_sorted:
        raise ValueError("pseudoinverse assembly requires sorted factors")
    d = factors.device()
    if d.kind != "dense":
        factors = SvdFactors(_to_dense(factors.U), factors.sigma, _to_dense(factors.Vt), True)
    t = torch()
    p, q = factors.shape
    dev = t.device("cuda", t.cuda.current_device())
    return _assemble(factors, t.arange(p, device=dev, dtype=t.int64), t.arange(q, device=dev, dtype=t.int64),
                     cutoff_factor)


def materialize(pinv: Pseudoinverse) -> np.ndarray:
    """pinv.py:234-239."""
    n, m = pinv.shape
    if n * m > DENSE_CAPACITY:
        raise CapacityError(f"materializing a {n}x{m} pseudoinverse exceeds the capacity guard")
    return (pinv.V * pinv.sigma_dagger) @ pinv.Ut


_PINV_HEADER = struct.Struct("<QQQB")


def save_pseudoinverse(pinv: Pseudoinverse, path):
    """pinv.py:242-254."""
    n, m = pinv.shape
    r = len(pinv.sigma_dagger)
    with open(path, "wb") as fh:
        fh.write(_PINV_HEADER.pack(n, m, r, 1 if pinv.all_filtered else 0))
        fh.write(np.ascontiguousarray(pinv.V, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(pinv.sigma_dagger, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(pinv.Ut, dtype="<f8").tobytes())
        fh.write(struct.pack("<d", pinv.tolerance_used))


def load_pseudoinverse(path) -> Pseudoinverse:
    """pinv.py:257-268."""
    raw = Path(path).read_bytes()
    n, m, r, flag = _PINV_HEADER.unpack_from(raw, 0)
    off = _PINV_HEADER.size
    V = np.frombuffer(raw, dtype="<f8", count=n * r, offset=off).reshape(n, r)
    off += 8 * n * r
    sd = np.frombuffer(raw, dtype="<f8", count=r, offset=off)
    off += 8 * r
    Ut = np.frombuffer(raw, dtype="<f8", count=r * m, offset=off).reshape(r, m)
    off += 8 * r * m
    (tol,) = struct.unpack_from("<d", raw, off)
    return Pseudoinverse(V.copy(), sd.copy(), Ut.copy(), tol, bool(flag))


def _unfold(factors: SvdFactors, result: ReorderResult) -> SvdFactors:
    """pinv.py:271-275: reordered-coordinate factors in original coordinates."""
    U = _to_dense(factors.U)[result.row_perm.forward, :]
    Vt = _to_dense(factors.Vt)[:, result.col_perm.forward]
    return SvdFactors(U, factors.sigma.copy(), Vt, is_sorted=factors.is_sorted)


class _Timer:
    def __init__(self):
        self.t = torch()

    def __enter__(self):
        self.t.cuda.synchronize()
        self.t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        self.t.cuda.synchronize()
        self.seconds = time.perf_counter() - self.t0


class _StageClock:
    """Stage boundaries as CUDA events on the current stream: no host synchronisation inside the
    solve (a wall-clock timer would drain the GPU at every stage edge and leave it idle while Python
    sets up the next stage).  ``resolve`` waits for the last boundary once and returns the
    reference's StageTime list (pinv.py:95-98) with device-measured seconds."""

    def __init__(self):
        self.t = torch()
        self.t0 = time.perf_counter()
        self.ev = [self._event()]
        self.stages = []

    def _event(self):
        e = self.t.cuda.Event(enable_timing=True)
        e.record()
        return e

    def mark(self, stage: str, rank: int):
        self.ev.append(self._event())
        self.stages.append((stage, int(rank)))

    def resolve(self) -> list:
        self.ev[-1].synchronize()
        return [StageTime(name, self.ev[i].elapsed_time(self.ev[i + 1]) * 1e-3, rank)
                for i, (name, rank) in enumerate(self.stages)]


_TRACE = bool(__import__("os").environ.get("FPI_TRACE_REORDER"))


def _trace_mark(label, tm):
    import sys
    torch().cuda.synchronize()
    print(f"[fastpi] {label} done at {(time.perf_counter() - tm.t0) * 1e3:.2f} ms", file=sys.stderr)


class _Owned:
    """A device buffer handed over by fpi_fastpi_take, viewed by torch through the CUDA array
    interface (the tensor keeps this object alive); freed stream-ordered (fpi_device_free) with the
    last tensor that views it."""

    def __init__(self, ptr, shape, typestr, device):
        self.ptr, self.device = ptr, device
        self.__cuda_array_interface__ = {"shape": tuple(int(x) for x in shape), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 2}

    def __del__(self):
        if self.ptr:
            try:
                with torch().cuda.device(self.device):
                    _lib.call("fpi_device_free", C.c_void_p(self.ptr))
            except Exception:  # interpreter shutdown: the process exit releases the pool
                pass


def _adopt(ptr, shape, dtype, device):
    t = torch()
    if ptr is None or math.prod(shape) == 0:
        if ptr:
            _Owned(ptr, (0,), "<f8", device)  # freed at once
        return t.empty(shape, dtype=dtype, device=t.device("cuda", device))
    typestr = "<f8" if dtype == t.float64 else "<i8"
    return t.as_tensor(_Owned(ptr, shape, typestr, device), device=t.device("cuda", device))


def _fastpi_one_call(dev: DeviceCSR, cfg: FastpiConfig, flags: int = _lib.FASTPI_CANONICAL) -> FastpiResult:
    """Algorithm 1 behind one C call (fpi_fastpi_ex, csrc/fastpi_capi.cu): the same stage entry points
    as the stage-by-stage mirror below, in the same order with the same ranks and seeds (identical
    bits, tests/test_pipeline_gpu.py), without a Python round trip and its allocations between the
    stages; the factors are adopted as torch tensors (fpi_fastpi_take)."""
    m, n = dev.shape
    t = torch()
    device = t.cuda.current_device()
    info = _lib.FastpiInfo()
    _lib.call("fpi_fastpi_ex", m, n, dev.nnz, _lib.ptr(dev.indptr), _lib.ptr(dev.indices), _lib.ptr(dev.values),
              float(cfg.alpha), float(cfg.k), int(cfg.seed), float(cfg.low_rank_threshold),
              float(cfg.pinv_cutoff_factor), flags, C.byref(info))
    if info.rank_clamped:
        warnings.warn(f"row-update target rank clamped from {math.ceil(cfg.alpha * info.n1)} to {info.s} "
                      "(block stage produced less derivable rank)")
    bufs = _lib.FastpiBuffers()
    gcc = (C.c_int64 * max(info.n_gcc, 1))()
    ms = (C.c_float * len(STAGES))()
    _lib.call("fpi_fastpi_take", C.byref(bufs), gcc, max(info.n_gcc, 1), ms)
    r = int(info.rank)
    f64, i64 = t.float64, t.int64
    U = _adopt(bufs.U, (m, r), f64, device)
    sigma = _adopt(bufs.sigma, (r,), f64, device)
    Vt = _adopt(bufs.Vt, (r, n), f64, device)
    sdag = _adopt(bufs.sigma_dagger, (r,), f64, device)
    row_fwd = _adopt(bufs.row_fwd, (m,), i64, device)
    col_fwd = _adopt(bufs.col_fwd, (n,), i64, device)
    spans = _adopt(bufs.spans, (4 * int(info.n_spans),), i64, device)
    ordering = ReorderResult(Permutation(row_fwd), Permutation(col_fwd), info.m1, info.n1, info.m2, info.n2, None,
                             info.n_iterations, [gcc[i] for i in range(info.n_gcc)], spans_device=spans)
    ordering.edges_visited, ordering.nodes_visited = int(info.edges_visited), int(info.nodes_visited)
    if info.all_filtered:
        warnings.warn("all singular values filtered; returning the zero pseudoinverse")
    pv = Pseudoinverse(tolerance_used=info.tolerance_used, all_filtered=bool(info.all_filtered),
                       _dev=_DevPinv(U, sdag, Vt, row_fwd, col_fwd))
    factors = SvdFactors(_dev=_Dense(U, sigma, Vt), is_sorted=True, _shape=(m, n))
    ranks = (0, int(info.rank11), int(info.s), r, pv.retained_rank)
    timings = [StageTime(name, ms[i] * 1e-3, ranks[i]) for i, name in enumerate(STAGES)]
    return FastpiResult(pv, factors, ordering, timings)


_STAGEWISE = bool(__import__("os").environ.get("FPI_STAGEWISE"))
_NO_DEFER = bool(__import__("os").environ.get("FPI_NO_DEFERRED_UPLOAD"))


def fastpi_device(dev: DeviceCSR, cfg: FastpiConfig, *, stats: dict | None = None,
                  stagewise: bool = False) -> FastpiResult:
    """Algorithm 1 on a canonical device CSR (m >= n); everything stays in HBM.

    By default the whole solve is one C call (``_fastpi_one_call``); ``stats`` (per-stage
    intermediates for tests and the bench's structure record), ``stagewise=True`` or FPI_STAGEWISE=1
    run the stage-by-stage mirror of pinv.py:278-347 below instead -- same kernels, same bits."""
    if stats is None and not stagewise and not _STAGEWISE and not _TRACE:
        return _fastpi_one_call(dev, cfg)
    m, n = dev.shape
    clock = _StageClock()
    ordering = reorder_device(dev, cfg.k)
    if _TRACE:
        _trace_mark("reorder_device", clock)
    part = partition_original(dev, ordering, transposes=True)
    clock.mark("reorder", 0)

    f11 = block_diagonal_svd_device(part.a11, ordering.spans_device(), cfg.alpha)
    clock.mark("block_svd", f11.rank)

    n1, m2, n2 = ordering.n_spoke_cols, ordering.n_hub_rows, ordering.n_hub_cols
    want_s = math.ceil(cfg.alpha * n1)
    s = min(want_s, f11.rank + m2, n1)
    if s < want_s:
        warnings.warn(f"row-update target rank clamped from {want_s} to {s} "
                      "(block stage produced less derivable rank)")
    f_rows, eng_r = row_update_device(f11, part.a21, s, low_rank_threshold=cfg.low_rank_threshold, seed=cfg.seed + 1)
    diag_r = _lib.svd_diag() if stats is not None else None
    clock.mark("row_update", f_rows.rank)

    r = min(math.ceil(cfg.alpha * n), f_rows.rank + n2, m)
    f_full, eng_c = column_update_device(f_rows, part.T, part.Tt, r, low_rank_threshold=cfg.low_rank_threshold,
                                         seed=cfg.seed + 2)
    diag_c = _lib.svd_diag() if stats is not None else None
    core_c = _lib.sparse_core_info() if stats is not None else None
    clock.mark("column_update", f_full.rank)

    pv = _assemble(f_full, ordering.row_perm.device_forward(), ordering.col_perm.device_forward(),
                   cfg.pinv_cutoff_factor)
    clock.mark("pinv_assembly", pv.retained_rank)
    timings = clock.resolve()
    if stats is not None:
        stats.update(engines=(eng_r, eng_c), s=s, r=r, rank11=f11.rank, m1=ordering.n_spoke_rows, n1=n1, m2=m2,
                     n2=n2, T=ordering.n_iterations, nnz_a12=part.info.nnz_a12, nnz_a22=part.info.nnz_a22,
                     nnz_a21=part.info.nnz_a21, nnz_a11=part.info.nnz_a11, f11=f11, f_rows=f_rows, part=part,
                     svd_diag_row=diag_r, svd_diag_col=diag_c, sparse_core=core_c)
    return FastpiResult(pv, f_full, ordering, timings)


def _swap(res: FastpiResult) -> FastpiResult:
    """pinv.py:291-303: results of fastpi(A^T) expressed for A."""
    pv = res.pseudoinverse
    d = pv._dev
    # pinv(A) = pinv(A^T)^T : U_A = V_{A^T}, Vt_A = U_{A^T}^T  (reordered coordinates swap roles)
    Ua = d.Vt.t().contiguous()
    Vta = d.U.t().contiguous()
    swapped = Pseudoinverse(sigma_dagger=pv.sigma_dagger.copy(), tolerance_used=pv.tolerance_used,
                            all_filtered=pv.all_filtered, _dev=_DevPinv(Ua, d.sdag, Vta, d.col_fwd, d.row_fwd))
    fd = res.factors.device()
    factors = SvdFactors(_dev=_Dense(fd.Vt.t().contiguous(), fd.sigma, fd.U.t().contiguous()), is_sorted=True,
                         _shape=(res.factors.shape[1], res.factors.shape[0]))
    return FastpiResult(swapped, factors, res.reordering, res.timings)


_DEFER_MIN_NNZ = 1 << 20
_DEFER_TRACE = bool(__import__("os").environ.get("FPI_DEFER_TRACE"))
_UPLOADER = None


def _uploader():
    """One long-lived worker thread for the deferred uploads (its CUDA context binding and torch's
    per-thread state are set up once, not per solve)."""
    global _UPLOADER
    if _UPLOADER is None:
        from concurrent.futures import ThreadPoolExecutor
        _UPLOADER = ThreadPoolExecutor(max_workers=1, thread_name_prefix="fastpi-values-upload")
    return _UPLOADER


def _fastpi_host_overlapped(A, cfg: FastpiConfig):
    """fastpi(A) for a host CSR with the upload of A's values hidden behind the reorder.

    Algorithm 2 (reorder.py:158-287) reads only the sparsity pattern, and the values are 2/3 of a
    CSR's bytes: the pattern is uploaded first, a worker thread stages the values into page-locked
    memory and copies them on a side stream while the solve's C call (FPI_FASTPI_DEFERRED_VALUES)
    runs the reorder; the call waits for the copy's event before the partition.  check_csr's
    canonical-form test (validation.py:38-55) runs in its two halves (pattern before the reorder,
    values before the partition); an input that is not canonical already makes the call return
    FPI_ERETRY, and None is returned for the plain path (canonicalize, then solve).  Same bits."""
    import threading
    t = torch()
    trace = [] if _DEFER_TRACE else None
    t_0 = time.perf_counter()
    m, n = A.shape
    nnz = int(A.nnz)
    device = t.cuda.current_device()
    main = t.cuda.current_stream()
    indptr = h2d(A.indptr, np.int64)
    indices = h2d(A.indices, np.int32)
    values = t.empty(nnz, dtype=t.float64, device=t.device("cuda", device))
    ready = t.cuda.Event()
    ready.record(main)          # the side stream must not write the block before main could have freed it
    copied = t.cuda.Event()
    side = t.cuda.Stream(device=device)
    enqueued = threading.Event()
    failure: list = []
    data = np.ascontiguousarray(A.data, dtype=np.float64)

    def upload():
        try:
            if trace is not None:
                trace.append(("worker starts", time.perf_counter() - t_0))
            t.cuda.set_device(device)
            with t.cuda.stream(side):
                side.wait_event(ready)
                src = t.from_numpy(data)
                step = max(1, (16 << 20) // 8)  # 16 MB chunks: staging of chunk k overlaps the DMA of k - 1
                for off in range(0, nnz, step):
                    cnt = min(step, nnz - off)
                    staged = t.empty(cnt, dtype=t.float64, pin_memory=True)
                    staged.copy_(src[off:off + cnt])
                    values[off:off + cnt].copy_(staged, non_blocking=True)
                if trace is not None:
                    trace.append(("staged", time.perf_counter() - t_0))
                copied.record(side)
            if trace is not None:
                trace.append(("enqueued", time.perf_counter() - t_0))
        except BaseException as e:  # surfaced through the hook's return code
            failure.append(e)
        finally:
            enqueued.set()

    @_lib.VALUES_HOOK
    def hook(_ctx, event_out):
        if trace is not None:
            trace.append(("hook called", time.perf_counter() - t_0))
        enqueued.wait()
        if failure:
            return 1
        event_out[0] = copied.cuda_event
        return 0

    worker = _uploader().submit(upload)
    if trace is not None:
        trace.append(("pattern uploaded, worker submitted", time.perf_counter() - t_0))
    dev = DeviceCSR((m, n), indptr, indices, values)
    try:
        _lib.call("fpi_fastpi_values_hook", hook, None)
        res = _fastpi_one_call(dev, cfg, _lib.FASTPI_CANONICAL | _lib.FASTPI_DEFERRED_VALUES)
    except _lib.RetryError:
        res = None
    finally:
        worker.result()
        if not failure:
            main.wait_event(copied)  # later work on the main stream (and the block's reuse) follows the copy
    if trace is not None:
        trace.append(("call returned", time.perf_counter() - t_0))
        print("[deferred upload] " + "  ".join(f"{k} {1e3 * v:.2f}" for k, v in sorted(trace, key=lambda x: x[1])),
              file=__import__("sys").stderr, flush=True)
    if failure:
        raise failure[0]
    if res is None:
        return None, dev
    return res, dev


def fastpi(A, config: FastpiConfig | None = None) -> FastpiResult:
    """pinv.py:278-347: reorder, block SVD, two incremental updates, assembly."""
    cfg = config or FastpiConfig()
    if (not isinstance(A, DeviceCSR) and not _STAGEWISE and not _TRACE and not _NO_DEFER):
        A = as_csr(A)
        if A.shape[0] >= A.shape[1] > 0 and A.nnz >= _DEFER_MIN_NNZ:
            res, raw = _fastpi_host_overlapped(A, cfg)
            if res is not None:
                return res
            A = raw.canonical()  # not canonical: check_csr's copy, then the plain path below
    dev = A if isinstance(A, DeviceCSR) else DeviceCSR.from_host(A)
    m, n = dev.shape
    if m == 0 or n == 0:
        raise ValueError("cannot factorize a zero-dimension matrix")
    if m < n:
        return _swap(fastpi_device(dev.transpose(), cfg))
    return fastpi_device(dev, cfg)
