"""Multi-GPU FastPI: one process per GPU, torch.distributed (NCCL over NVLink /
NVSwitch) for the exchanges.

What shards and what is replicated:

* reorder, partition, row update: replicated.  Every rank holds A and computes
  them itself (deterministic kernels, so the ranks agree bit for bit).
* block SVD (svd.py:141-193): the diagonal blocks are independent units -- each
  rank factors its share (round-robin for the many small blocks, LPT by
  h w min(h, w) for the large ones, fpi_block_svd_shard) and one all-reduce of
  sigma / U11 / Vt11 values (disjoint supports, so the sum is the union)
  gives every rank the full block factors for the replicated row update.
* column update (pinv.py:174-208, the FP64 GEMM-bound stage): the m rows of
  [U Sigma | T] are split into contiguous shards.  Every rank regenerates the
  full sketch X (svd.py:131-132), forms its B_i = M_i X, and the two
  reductions of the randomized SVD are all-reduces:
      G = sum_i B_i^T B_i          (2r x 2r,  svd.py:134's QR Gram)
      Z = sum_i M_i^T B_i          ((s+n2) x 2r, svd.py:135's Q^T M)
  The small SVD of Y^T = Z L^-T is replicated; U_i = B_i L^-T U~ stays local.
  The dense engine (small problems) runs replicated and keeps its row shard.
* apply (pinv.py:72-81): W = sum_i Y_i^T U_i is all-reduced (L x r); the lift
  Z = V Sigma+ W^T is replicated.

The algorithm is written against two small interfaces -- ``ops`` (the
library's kernels on device tensors, ``GpuOps``) and ``comm`` (the
all-reduce) -- so the same code runs with world size 1, with N GPUs over
NCCL, and in the CPU tests with a numpy stand-in for ``ops`` over gloo.
"""

from __future__ import annotations

import ctypes as C
import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import DeviceCSR, d2h, empty, torch
from .pinv import (FastpiConfig, StageTime, _assemble, _Timer, column_update_device, row_update_device)
from .reorder import partition_original, reorder_device
from .svd import block_diagonal_svd_device


# ---------------------------------------------------------------- communication
class Comm:
    """Rank / world of the current torch.distributed group (world 1 when not initialised)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self._dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.world = self._dist.get_world_size(group) if self._dist else 1
        self.rank = self._dist.get_rank(group) if self._dist else 0

    def all_reduce_(self, t):
        """In-place sum over ranks (NCCL for device tensors, gloo for host tensors)."""
        if self.world > 1:
            self._dist.all_reduce(t, group=self.group)
        return t

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch as T
        dev = "cuda" if self._dist.get_backend(self.group) == "nccl" else "cpu"
        t = T.tensor([x], dtype=T.float64, device=dev)
        self._dist.all_reduce(t, op=self._dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


def shard_bounds(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced row ranges (the first m % world shards get one extra row)."""
    base, extra = divmod(m, world)
    out, r0 = [], 0
    for i in range(world):
        ln = base + (1 if i < extra else 0)
        out.append((r0, r0 + ln))
        r0 += ln
    return out


# ---------------------------------------------------------------- kernels on the device
class GpuOps:
    """The library's sm_100a kernels on torch device tensors (row-major float64)."""

    def empty(self, shape):
        return empty(shape)

    def zeros(self, shape):
        t = empty(shape)
        t.zero_()
        return t

    def sketch(self, seed, rows, cols):
        X = empty((rows, cols))
        if rows and cols:
            _lib.call("fpi_sketch_normal", int(seed), rows, cols, _lib.ptr(X), cols)
        return X

    def gemm(self, A, B, ta=False, tb=False, out=None, beta=0.0):
        M = A.shape[1] if ta else A.shape[0]
        K = A.shape[0] if ta else A.shape[1]
        N = B.shape[0] if tb else B.shape[1]
        C_ = out if out is not None else empty((M, N))
        _lib.call("fpi_gemm", int(ta), int(tb), M, N, K, 1.0, _lib.ptr(A), A.shape[1], _lib.ptr(B), B.shape[1],
                  float(beta), _lib.ptr(C_), N)
        return C_

    def gram(self, B):
        """B^T B for a p x k row shard (symmetric product)."""
        p, k = B.shape
        G = empty((k, k))
        _lib.call("fpi_gram", 1, k, p, _lib.ptr(B), k, _lib.ptr(G), k)
        return G

    def spmm(self, A: DeviceCSR, X, out, beta=0.0):
        p, q = A.shape
        k = X.shape[1]
        if p and k:
            if A.nnz == 0 or q == 0:
                if beta == 0.0:
                    out.zero_()
            else:
                _lib.call("fpi_spmm", p, q, k, _lib.ptr(A.indptr), _lib.ptr(A.indices), _lib.ptr(A.values), 1.0,
                          _lib.ptr(X), k, float(beta), _lib.ptr(out), k)
        return out

    def scale_rows(self, A, s):
        _lib.call("fpi_scale_rows", A.shape[0], A.shape[1], _lib.ptr(A), A.shape[1], _lib.ptr(s))
        return A

    def orth_factor(self, G):
        k = G.shape[0]
        Linv = empty((k, k))
        cond = C.c_double(0.0)
        _lib.call("fpi_orth_factor", k, _lib.ptr(G), _lib.ptr(Linv), C.byref(cond))
        return Linv

    def dense_svd(self, M, rank):
        p, q = M.shape
        U, s, Vt = empty((p, rank)), empty(rank), empty((rank, q))
        _lib.call("fpi_dense_svd", p, q, _lib.ptr(M), q, int(rank), _lib.ptr(U), _lib.ptr(s), _lib.ptr(Vt))
        return U, s, Vt

    def transpose(self, A):
        At = empty((A.shape[1], A.shape[0]))
        _lib.call("fpi_transpose", A.shape[0], A.shape[1], _lib.ptr(A), A.shape[1], _lib.ptr(At), A.shape[0])
        return At

    def canonical_signs(self, U, Vt):
        r, q = Vt.shape
        _lib.call("fpi_canonical_signs", r, U.shape[0], q, _lib.ptr(U), U.shape[1], _lib.ptr(Vt), q)

    def slice_rows(self, A, r0, r1):
        return A[r0:r1]

    def csr_rows(self, A: DeviceCSR, r0, r1):
        return A.row_slice(r0, r1)

    def csr_transpose(self, A: DeviceCSR):
        return A.transpose()

    def copy(self, A):
        return A.clone()

    def hstack_lift(self, Vt, Vt_prev, s, n1, n2):
        """[Vt[:, :s] Vt_prev | Vt[:, s:]] (pinv.py:205-207)."""
        r = Vt.shape[0]
        out = empty((r, n1 + n2))
        if n1:
            if s:
                _lib.call("fpi_gemm", 0, 0, r, n1, s, 1.0, _lib.ptr(Vt), Vt.shape[1], _lib.ptr(Vt_prev), n1, 0.0,
                          _lib.ptr(out), n1 + n2)
            else:
                out[:, :n1].zero_()
        if n2:
            out[:, n1:].copy_(Vt[:, s:])
        return out


# ---------------------------------------------------------------- column update (row-sharded)
def column_update_shard(ops, comm, U_i, sigma, Vt_prev, T_i, Tt_i, m: int, r: int, seed: int):
    """Randomized engine of pinv.py:174-208 on the row shard M_i = [U_i diag(sigma) | T_i].

    Returns (U_out_i, sigma_out, Vt_out) with Vt_out the lifted r x (n1 + n2) factor, identical
    on every rank.  Mirrors svd_engine.cu's randomized_svd step by step (svd.py:120-138)."""
    s = int(sigma.shape[0])
    n1 = int(Vt_prev.shape[1])
    n2 = int(T_i.shape[1])
    q = s + n2
    k = 2 * r
    m_i = int(T_i.shape[0])
    X = ops.sketch(seed, q, k)                              # svd.py:131-132 (same on every rank)
    B = ops.zeros((m_i, k))
    if s:
        X1 = ops.copy(X[:s])
        ops.scale_rows(X1, sigma)                           # diag(sigma) X1
        ops.gemm(U_i, X1, out=B)
    if n2:
        ops.spmm(T_i, X[s:], out=B, beta=1.0 if s else 0.0)  # + T_i X2      (svd.py:133)
    G = comm.all_reduce_(ops.gram(B))                       # B^T B        (svd.py:134)
    Linv = ops.orth_factor(G)
    Z = ops.zeros((q, k))                                   # M^T B
    if s:
        ops.gemm(U_i, B, ta=True, out=Z[:s])
        ops.scale_rows(Z[:s], sigma)
    if n2:
        ops.spmm(Tt_i, B, out=Z[s:])
    comm.all_reduce_(Z)
    Yt = ops.gemm(Z, Linv, tb=True)                         # Y^T = Z L^-T (svd.py:135)
    Vy, sig, Uyt = ops.dense_svd(Yt, r)                     # svd.py:136
    Vt = ops.transpose(Vy)
    Mx = ops.gemm(Linv, Uyt, ta=True, tb=True)              # L^-T U~
    U_out = ops.gemm(B, Mx)                                 # svd.py:137, local rows
    ops.canonical_signs(U_out, Vt)                          # sign from Vt: same on every rank
    return U_out, sig, ops.hstack_lift(Vt, Vt_prev, s, n1, n2)


# ---------------------------------------------------------------- results
class ShardedPseudoinverse:
    """pinv(A) with U row-sharded in reordered coordinates: rank i holds rows [r0, r1)."""

    def __init__(self, comm, U_i, r0, m, sdag, Vt, row_fwd, col_fwd, tolerance_used, all_filtered):
        self.comm, self.U_i, self.r0, self.m = comm, U_i, r0, m
        self.sdag, self.Vt, self.row_fwd, self.col_fwd = sdag, Vt, row_fwd, col_fwd
        self.tolerance_used, self.all_filtered = tolerance_used, all_filtered
        self.r = int(sdag.shape[0])
        self.n = int(Vt.shape[1])

    @property
    def sigma_dagger(self) -> np.ndarray:
        return d2h(self.sdag)

    def apply_device(self, Y: DeviceCSR):
        """pinv @ Y (Y CSR m x L, original rows): the full n x L result on every rank."""
        if Y.shape[0] != self.m:
            raise ValueError(f"dimension mismatch: pseudoinverse expects {self.m} rows, got {Y.shape[0]}")
        L = Y.shape[1]
        W = empty((L, self.r))
        _lib.call("fpi_pinv_project_csr", self.r0, int(self.U_i.shape[0]), self.r, _lib.ptr(self.U_i),
                  _lib.ptr(self.row_fwd), self.m, L, Y.nnz, _lib.ptr(Y.indptr), _lib.ptr(Y.indices),
                  _lib.ptr(Y.values), _lib.ptr(W))
        self.comm.all_reduce_(W)
        Z = empty((self.n, L))
        _lib.call("fpi_pinv_lift", self.n, self.r, _lib.ptr(self.sdag), _lib.ptr(self.Vt), _lib.ptr(self.col_fwd), L,
                  _lib.ptr(W), _lib.ptr(Z))
        return Z


@dataclass
class ShardedResult:
    pseudoinverse: ShardedPseudoinverse
    sigma: object
    reordering: object
    timings: list
    engine: int


def fastpi_sharded(dev: DeviceCSR, cfg: FastpiConfig, comm: Comm | None = None, *, stats: dict | None = None,
                   ops=None) -> ShardedResult:
    """Algorithm 1 (pinv.py:278-347) on every rank of ``comm``; m >= n.  The column update and
    the apply are row-sharded; the earlier stages are replicated."""
    comm = comm or Comm()
    ops = ops or GpuOps()
    m, n = dev.shape
    if m < n:
        raise ValueError("fastpi_sharded expects m >= n (transpose the problem first)")
    timings = []
    with _Timer() as tm:
        ordering = reorder_device(dev, cfg.k)
        part = partition_original(dev, ordering, transposes=False)
    timings.append(StageTime("reorder", tm.seconds, comm.rank))
    with _Timer() as tm:
        f11 = block_diagonal_svd_device(part.a11, ordering.spans_device(), cfg.alpha, comm)
    timings.append(StageTime("block_svd", tm.seconds, comm.rank))
    n1, m2, n2 = ordering.n_spoke_cols, ordering.n_hub_rows, ordering.n_hub_cols
    with _Timer() as tm:
        want_s = math.ceil(cfg.alpha * n1)
        s = min(want_s, f11.rank + m2, n1)
        if s < want_s:
            warnings.warn(f"row-update target rank clamped from {want_s} to {s} "
                          "(block stage produced less derivable rank)")
        f_rows, _ = row_update_device(f11, part.a21, s, low_rank_threshold=cfg.low_rank_threshold, seed=cfg.seed + 1)
    timings.append(StageTime("row_update", tm.seconds, comm.rank))

    r = min(math.ceil(cfg.alpha * n), f_rows.rank + n2, m)
    q = f_rows.rank + n2
    r0, r1 = shard_bounds(m, comm.world)[comm.rank]
    with _Timer() as tm:
        randomized = r >= 1 and r < cfg.low_rank_threshold * q and m > 2 * r
        if randomized:
            d = f_rows.device()
            T_i = ops.csr_rows(part.T, r0, r1)
            U_i, sig, Vt = column_update_shard(ops, comm, ops.slice_rows(d.U, r0, r1), d.sigma, d.Vt, T_i,
                                               ops.csr_transpose(T_i), m, r, cfg.seed + 2)
            engine = 1
        else:
            # dense engine (or r == 0): replicated, each rank keeps its rows of U
            f_full, engine = column_update_device(f_rows, part.T, part.T.transpose(), r,
                                                  low_rank_threshold=cfg.low_rank_threshold, seed=cfg.seed + 2)
            fd = f_full.device()
            U_i, sig, Vt = fd.U[r0:r1].contiguous(), fd.sigma, fd.Vt
    timings.append(StageTime("column_update", tm.seconds, comm.rank))

    with _Timer() as tm:
        # pinv.py:211-231 on the replicated sigma: the same sigma+ on every rank
        from .svd import SvdFactors, _Dense
        probe = _assemble(SvdFactors(_dev=_Dense(empty((0, r)), sig, Vt), is_sorted=True, _shape=(m, n)),
                          ordering.row_perm.device_forward(), ordering.col_perm.device_forward(),
                          cfg.pinv_cutoff_factor)
        pdev = probe._dev
        pv = ShardedPseudoinverse(comm, U_i, r0, m, pdev.sdag, Vt, pdev.row_fwd, pdev.col_fwd, probe.tolerance_used,
                                  probe.all_filtered)
    timings.append(StageTime("pinv_assembly", tm.seconds, comm.rank))
    if stats is not None:
        stats.update(engine=engine, r=r, q=q, shard=(r0, r1), world=comm.world)
    return ShardedResult(pv, sig, ordering, timings, engine)


def fastpi_distributed(A, config: FastpiConfig | None = None, comm: Comm | None = None) -> ShardedResult:
    """Public multi-GPU entry (host or device A, m >= n): every rank of the current
    torch.distributed group calls it with the same A and config."""
    cfg = config or FastpiConfig()
    dev = A if isinstance(A, DeviceCSR) else DeviceCSR.from_host(A)
    if dev.shape[0] == 0 or dev.shape[1] == 0:
        raise ValueError("cannot factorize a zero-dimension matrix")
    return fastpi_sharded(dev, cfg, comm)


def apply_distributed(pv: ShardedPseudoinverse, Y) -> np.ndarray:
    """pinv @ Y for host (scipy) or device Y; the n x L result as numpy on every rank."""
    Yd = Y if isinstance(Y, DeviceCSR) else DeviceCSR.from_host(Y)
    return d2h(pv.apply_device(Yd))
