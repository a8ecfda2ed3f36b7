"""Multi-GPU FastPI: one process per GPU; the exchanges run inside the library
(csrc/sharded.cu) on the handle's communicator (csrc/comm.cu: NCCL over
NVLink / NVSwitch, loaded from the libnccl.so.2 torch ships).
section 8(e).

Ownership (``fpi_shard_plan``): rank i owns a contiguous range of the A11
diagonal blocks (balanced by the rows' work, the blocks' columns and their
h w min(h, w) SVD cost) -- hence spoke rows [r_lo, r_hi) and spoke columns
[c_lo, c_hi) -- plus a chunk [h_lo, h_hi) of the m2 hub rows and a chunk
[hc_lo, hc_hi) of the n2 hub columns.  Its rows of U, T, A21, Y are its spoke
rows then its hub rows; its columns of Vt and its rows of Z are its spoke
columns then its hub columns.

=============================  ==================================================================
stage (reference)              what each rank does / what is exchanged
=============================  ==================================================================
reorder, partition             replicated (deterministic kernels: identical on every rank)
block SVD (svd.py:141-193)     its own blocks only (``fpi_block_svd_range``); nothing exchanged
row update (pinv.py:131-171)   rows of inner = its kept Sigma Vt11 rows + its A21 rows;
                               G = sum B_i^T B_i (all-reduce 2s x 2s); Z = inner^T B reduced onto
                               the owner of each spoke-column range (one ncclReduce per rank, the
                               reduce-scatter of Y); Gram of Y^T all-reduced; eigensolve
                               replicated; U rows and Vt columns local
column update (pinv.py:174-   rows of [U Sigma | T]; Z = sum M_i^T B_i (all-reduce (s+n2) x 2r);
208)                           G = X^T Z split over the ranks (all-reduce); small SVD replicated;
                               U rows local; Vt columns = [Vt~[:, :s] Vt_prev_loc | own hub cols]
apply (pinv.py:72-81)          W = sum Y_i^T U_i (all-reduce L x r); each rank the rows of Z of its
                               own columns (its V-row slice); gathered at the host boundary
=============================  ==================================================================

Small problems whose updates take the dense engine run the single-GPU
pipeline on every rank and keep their slices (the sharded engines are the
randomized ones; the dense path is for inner matrices below the 1e8-entry
guard).

``FPI_COMM=callback`` (or a non-NCCL torch.distributed backend) routes the
exchanges through a host callback over torch.distributed -- the functional
test of the pattern with several ranks on one GPU.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import traceback
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import DeviceCSR, d2h, empty, torch
from .pinv import FastpiConfig, StageTime, _StageClock, fastpi_device
from .reorder import partition_original, reorder_device

PLAN_FIELDS = ("b_lo", "b_hi", "r_lo", "r_hi", "c_lo", "c_hi", "h_lo", "h_hi", "hc_lo", "hc_hi")


# ---------------------------------------------------------------- communication
class _DeviceView:
    """A raw device buffer as a torch tensor (CUDA array interface), for the callback exchanges."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr or 0), False),
                                         "version": 3}


def _view(ptr, n):
    return torch().as_tensor(_DeviceView(ptr, n), device="cuda")


class Comm:
    """Rank / world of the current torch.distributed group, and the binding of the library
    handle's communicator: native NCCL when the group's backend is NCCL, a torch.distributed
    callback otherwise (world 1: the identity)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self._dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.world = self._dist.get_world_size(group) if self._dist else 1
        self.rank = self._dist.get_rank(group) if self._dist else 0
        self.backend = self._dist.get_backend(group) if self._dist else "none"
        self._cb = None
        self._bound = set()
        self.kind = None

    def bind(self):
        """Attach a communicator to this thread's library handle on the current device (once)."""
        h = _lib.handle()
        if h.value in self._bound:
            return
        lib = _lib.load()
        if self.world == 1:
            rc = lib.fpi_comm_init_self(h)
            self.kind = "self"
        elif self.backend == "nccl" and os.environ.get("FPI_COMM", "nccl") != "callback":
            uid = C.create_string_buffer(128)
            if self.rank == 0:
                err = C.create_string_buffer(256)
                if lib.fpi_comm_nccl_id(uid, err, len(err)) != _lib.FPI_OK:
                    raise RuntimeError(f"NCCL unavailable: {err.value.decode()}")
            obj = [bytes(uid.raw)]
            self._dist.broadcast_object_list(obj, src=0, group=self.group)
            rc = lib.fpi_comm_init_nccl(h, obj[0], self.rank, self.world)
            self.kind = "nccl"
        else:
            self._cb = _lib.COMM_FN(self._callback)
            rc = lib.fpi_comm_init_callback(h, self.rank, self.world, self._cb, None)
            self.kind = "callback"
        if rc != _lib.FPI_OK:
            raise RuntimeError(f"communicator setup failed: {lib.fpi_last_error(h).decode()}")
        self._bound.add(h.value)

    def _callback(self, user, op, send, recv, count, root):
        """Exchanges staged through host memory (gloo); device pointers in, device memory out."""
        try:
            t = torch()
            d = self._dist
            if op in (0, 1):
                buf = _view(recv, count)
                hb = buf.cpu()
                d.all_reduce(hb, op=d.ReduceOp.SUM if op == 0 else d.ReduceOp.MAX, group=self.group)
                buf.copy_(hb)
            elif op == 2:
                hs = _view(send, count).cpu()
                parts = [t.empty_like(hs) for _ in range(self.world)]
                d.all_gather(parts, hs, group=self.group)
                _view(recv, count * self.world).copy_(t.cat(parts))
            elif op == 3:
                hs = _view(send, count).cpu().clone()
                d.reduce(hs, dst=root, group=self.group)
                if self.rank == root:
                    _view(recv, count).copy_(hs)
            else:
                return 1
            t.cuda.synchronize()
            return 0
        except Exception:  # pragma: no cover - reported through the status code
            traceback.print_exc()
            return 1

    def all_gather_object(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self._dist.all_gather_object(out, obj, group=self.group)
        return out

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = torch()
        dev = "cuda" if self.backend == "nccl" else "cpu"
        v = t.tensor([x], dtype=t.float64, device=dev)
        self._dist.all_reduce(v, op=self._dist.ReduceOp.MAX, group=self.group)
        return float(v.item())


def shard_bounds(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced ranges (the first m % world get one extra)."""
    base, extra = divmod(m, world)
    out, r0 = [], 0
    for i in range(world):
        ln = base + (1 if i < extra else 0)
        out.append((r0, r0 + ln))
        r0 += ln
    return out


def shard_plan(ordering, T: DeviceCSR, world: int) -> np.ndarray:
    """(world, 10) int64 ownership table, columns PLAN_FIELDS (fpi_shard_plan)."""
    m, n2 = T.shape
    out = np.zeros((world, len(PLAN_FIELDS)), np.int64)
    spans = ordering.spans_device()
    _lib.call("fpi_shard_plan", m, ordering.n_spoke_rows, ordering.n_spoke_cols, n2, int(spans.numel() // 4),
              _lib.ptr(spans), _lib.ptr(T.indptr), int(world), out.ctypes.data_as(C.c_void_p))
    return out


def _rows_of(A: DeviceCSR, ranges) -> DeviceCSR:
    """The rows of several [a, b) ranges of a CSR, stacked in order."""
    t = torch()
    parts = [A.row_slice(a, b) for a, b in ranges if b > a]
    rows = sum(b - a for a, b in ranges)
    if not parts:
        return DeviceCSR((0, A.shape[1]), t.zeros(1, dtype=t.int64, device="cuda"), A.indices[:0], A.values[:0])
    ptrs, off = [parts[0].indptr], int(parts[0].indptr[-1].item())
    for p in parts[1:]:
        ptrs.append(p.indptr[1:] + off)
        off += p.nnz
    return DeviceCSR((rows, A.shape[1]), t.cat(ptrs), t.cat([p.indices for p in parts]),
                     t.cat([p.values for p in parts]))


# ---------------------------------------------------------------- results
class ShardedPseudoinverse:
    """pinv(A) with this rank's slices: U_loc (its rows, reordered coordinates), Vt_loc (its
    columns), sigma+ replicated."""

    def __init__(self, comm, plan_row, m, n, m1, n1, U_loc, sdag, Vt_loc, row_fwd, col_perm, tolerance_used,
                 all_filtered):
        self.comm, self.m, self.n, self.m1, self.n1 = comm, m, n, m1, n1
        self.p = dict(zip(PLAN_FIELDS, (int(x) for x in plan_row)))
        self.U_loc, self.sdag, self.Vt_loc, self.row_fwd = U_loc, sdag, Vt_loc, row_fwd
        self.tolerance_used, self.all_filtered = tolerance_used, all_filtered
        self.r = int(sdag.shape[0])
        p = self.p
        reord = np.concatenate([np.arange(p["c_lo"], p["c_hi"]), n1 + np.arange(p["hc_lo"], p["hc_hi"])])
        self.cols = col_perm.backward[reord] if len(reord) else np.zeros(0, np.int64)  # original column ids

    @property
    def sigma_dagger(self) -> np.ndarray:
        return d2h(self.sdag)

    def apply_local(self, Y: DeviceCSR):
        """(original column ids, Z rows of this rank's columns on the device) of Z = pinv @ Y."""
        if Y.shape[0] != self.m:
            raise ValueError(f"dimension mismatch: pseudoinverse expects {self.m} rows, got {Y.shape[0]}")
        self.comm.bind()
        L = Y.shape[1]
        p = self.p
        Z = empty((len(self.cols), L))
        _lib.call("fpi_pinv_apply_shard", self.m, self.m1, p["r_lo"], p["r_hi"], p["h_lo"], p["h_hi"], self.r,
                  _lib.ptr(self.U_loc), _lib.ptr(self.sdag), _lib.ptr(self.Vt_loc), len(self.cols),
                  _lib.ptr(self.row_fwd), L, Y.nnz, _lib.ptr(Y.indptr), _lib.ptr(Y.indices), _lib.ptr(Y.values),
                  _lib.ptr(Z))
        return self.cols, Z

    def apply(self, Y) -> np.ndarray:
        """The full n x L Z on every rank (each rank's rows gathered on the host)."""
        Yd = Y if isinstance(Y, DeviceCSR) else DeviceCSR.from_host(Y)
        cols, Z = self.apply_local(Yd)
        parts = self.comm.all_gather_object((cols, d2h(Z)))
        out = np.zeros((self.n, Yd.shape[1]))
        for c, z in parts:
            out[c] = z
        return out


@dataclass
class ShardedResult:
    pseudoinverse: ShardedPseudoinverse
    sigma: object
    reordering: object
    timings: list
    engines: tuple
    sharded: bool


def fastpi_sharded(dev: DeviceCSR, cfg: FastpiConfig, comm: Comm | None = None, *,
                   stats: dict | None = None) -> ShardedResult:
    """Algorithm 1 (pinv.py:278-347) over the ranks of ``comm``; m >= n."""
    comm = comm or Comm()
    comm.bind()
    m, n = dev.shape
    if m < n:
        raise ValueError("fastpi_sharded expects m >= n (transpose the problem first)")
    clock = _StageClock()
    ordering = reorder_device(dev, cfg.k)
    part = partition_original(dev, ordering, transposes=False)
    clock.mark("reorder", 0)
    m1, n1 = ordering.n_spoke_rows, ordering.n_spoke_cols
    m2, n2 = ordering.n_hub_rows, ordering.n_hub_cols
    plan = shard_plan(ordering, part.T, comm.world)
    P = dict(zip(PLAN_FIELDS, (int(x) for x in plan[comm.rank])))
    spans = ordering.spans_device()
    nsp = int(spans.numel() // 4)
    thr = cfg.low_rank_threshold

    bplan = _lib.BlockPlan()
    _lib.call("fpi_block_svd_plan", nsp, _lib.ptr(spans), float(cfg.alpha), C.byref(bplan))
    rank11 = int(bplan.rank11)
    U11 = DeviceCSR.empty(m1, rank11, bplan.nnz_u11)
    Vt11 = DeviceCSR.empty(rank11, n1, bplan.nnz_vt11)
    sig11 = empty(rank11)
    krange = (C.c_int64 * 2)()
    _lib.call("fpi_block_svd_range", m1, n1, _lib.ptr(part.a11.indptr), _lib.ptr(part.a11.indices),
              _lib.ptr(part.a11.values), nsp, _lib.ptr(spans), float(cfg.alpha), P["b_lo"], P["b_hi"],
              _lib.ptr(sig11), _lib.ptr(U11.indptr), _lib.ptr(U11.indices), _lib.ptr(U11.values),
              _lib.ptr(Vt11.indptr), _lib.ptr(Vt11.indices), _lib.ptr(Vt11.values), C.byref(bplan), krange)
    k_lo, k_hi = int(krange[0]), int(krange[1])
    clock.mark("block_svd", rank11)

    want_s = math.ceil(cfg.alpha * n1)
    s = min(want_s, rank11 + m2, n1)
    if s < want_s:
        warnings.warn(f"row-update target rank clamped from {want_s} to {s} (block stage produced less derivable rank)")
    r = min(math.ceil(cfg.alpha * n), s + n2, m)
    row_sharded = 1 <= s < thr * n1 and rank11 + m2 > 2 * s
    col_sharded = 1 <= r < thr * (s + n2) and m > 2 * r
    if not (row_sharded and col_sharded):
        return _replicated(dev, cfg, comm, plan, P, ordering, stats)

    r_rows, m2_loc = P["r_hi"] - P["r_lo"], P["h_hi"] - P["h_lo"]
    nc_loc = P["c_hi"] - P["c_lo"]
    zoff = np.ascontiguousarray(np.append(plan[:, 4], n1).astype(np.int64))  # spoke-column ranges
    U_rows = empty((r_rows + m2_loc, s))
    sig_rows = empty(s)
    Vt_rows = empty((s, nc_loc))
    _lib.call("fpi_row_update_shard", n1, _lib.ptr(sig11), _lib.ptr(Vt11.indptr), _lib.ptr(Vt11.indices),
              _lib.ptr(Vt11.values), k_lo, k_hi - k_lo, _lib.ptr(U11.indptr), _lib.ptr(U11.indices),
              _lib.ptr(U11.values), P["r_lo"], r_rows, _lib.ptr(part.a21.indptr), _lib.ptr(part.a21.indices),
              _lib.ptr(part.a21.values), P["h_lo"], m2_loc, rank11 + m2, s, float(thr), cfg.seed + 1,
              zoff.ctypes.data_as(C.c_void_p), _lib.ptr(U_rows), _lib.ptr(sig_rows), _lib.ptr(Vt_rows))
    diag_r = _lib.svd_diag() if stats is not None else None
    clock.mark("row_update", s)

    T_loc = _rows_of(part.T, [(P["r_lo"], P["r_hi"]), (m1 + P["h_lo"], m1 + P["h_hi"])])
    Tt_loc = T_loc.transpose()
    m_loc = T_loc.shape[0]
    nh_loc = P["hc_hi"] - P["hc_lo"]
    U_loc = empty((m_loc, r))
    sig = empty(r)
    Vt_loc = empty((r, nc_loc + nh_loc))
    _lib.call("fpi_column_update_shard", m_loc, s, _lib.ptr(U_rows), _lib.ptr(sig_rows), _lib.ptr(Vt_rows),
              nc_loc, n2, _lib.ptr(T_loc.indptr), _lib.ptr(T_loc.indices), _lib.ptr(T_loc.values),
              _lib.ptr(Tt_loc.indptr), _lib.ptr(Tt_loc.indices), _lib.ptr(Tt_loc.values), m, P["hc_lo"],
              P["hc_hi"], r, float(thr), cfg.seed + 2, _lib.ptr(U_loc), _lib.ptr(sig), _lib.ptr(Vt_loc))
    diag_c = _lib.svd_diag() if stats is not None else None
    clock.mark("column_update", r)

    sdag = empty(r)
    tol = C.c_double(0.0)
    af = C.c_int32(0)
    _lib.call("fpi_pinv_assemble", r, _lib.ptr(sig), m, n, float(cfg.pinv_cutoff_factor), _lib.ptr(sdag),
              C.byref(tol), C.byref(af))
    if af.value:
        warnings.warn("every singular value fell below the cutoff; the pseudoinverse is zero")
    pv = ShardedPseudoinverse(comm, plan[comm.rank], m, n, m1, n1, U_loc, sdag, Vt_loc,
                              ordering.row_perm.device_forward(), ordering.col_perm, float(tol.value),
                              bool(af.value))
    clock.mark("pinv_assembly", r)
    timings = clock.resolve()
    if stats is not None:
        stats.update(engines=(1, 1), s=s, r=r, rank11=rank11, m1=m1, n1=n1, m2=m2, n2=n2,
                     T=ordering.n_iterations, plan=plan, world=comm.world, sharded=True, svd_diag_row=diag_r,
                     svd_diag_col=diag_c)
    return ShardedResult(pv, sig, ordering, timings, (1, 1), True)


def _replicated(dev, cfg, comm, plan, P, ordering, stats):
    """Small problems (a dense-engine update): the single-GPU pipeline on every rank, each rank
    keeping its rows of U and its columns of Vt."""
    res = fastpi_device(dev, cfg, stats=stats)
    fd = res.factors.device()
    m1, n1 = ordering.n_spoke_rows, ordering.n_spoke_cols
    t = torch()
    U_loc = t.cat([fd.U[P["r_lo"]:P["r_hi"]], fd.U[m1 + P["h_lo"]:m1 + P["h_hi"]]]).contiguous()
    Vt_loc = t.cat([fd.Vt[:, P["c_lo"]:P["c_hi"]], fd.Vt[:, n1 + P["hc_lo"]:n1 + P["hc_hi"]]], dim=1).contiguous()
    pvd = res.pseudoinverse._dev
    m, n = dev.shape
    pv = ShardedPseudoinverse(comm, plan[comm.rank], m, n, m1, n1, U_loc, pvd.sdag, Vt_loc, pvd.row_fwd,
                              res.reordering.col_perm, res.pseudoinverse.tolerance_used,
                              res.pseudoinverse.all_filtered)
    if stats is not None:
        stats.update(plan=plan, world=comm.world, sharded=False)
    return ShardedResult(pv, fd.sigma, res.reordering, res.timings, tuple(stats.get("engines", (0, 0)))
                         if stats else (0, 0), False)


def fastpi_distributed(A, config: FastpiConfig | None = None, comm: Comm | None = None) -> ShardedResult:
    """Public multi-GPU entry (host or device A, m >= n): every rank of the current
    torch.distributed group calls it with the same A and config."""
    cfg = config or FastpiConfig()
    dev = A if isinstance(A, DeviceCSR) else DeviceCSR.from_host(A)
    if dev.shape[0] == 0 or dev.shape[1] == 0:
        raise ValueError("cannot factorize a zero-dimension matrix")
    return fastpi_sharded(dev, cfg, comm)


def apply_local(pv: ShardedPseudoinverse, Y):
    """This rank's rows of Z = pinv @ Y as (original column ids, host array): the per-GPU
    device->host copies run in parallel; the caller assembles them."""
    Yd = Y if isinstance(Y, DeviceCSR) else DeviceCSR.from_host(Y)
    cols, Z = pv.apply_local(Yd)
    return cols, d2h(Z)


def apply_distributed(pv: ShardedPseudoinverse, Y) -> np.ndarray:
    """pinv @ Y for host (scipy) or device Y; the full n x L result as numpy on every rank."""
    return pv.apply(Y)
