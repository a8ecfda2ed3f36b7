"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy/scipy restatement of the reference FastPI path
(``/root/reference/pkg/src/fastpi``), used as the checker for the B200
implementation.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package (``paper_2011_04235_b200``) never imports, calls or
links anything under ``oracle/``.

Pinning: the reference ships no golden vectors.  This
restatement is pinned against the reference itself, imported in the build
container: ``oracle/pin_against_reference.py`` checks every stage bit-for-bit
(permutations, spans, per-stage sigma / U / Vt, Z) and writes the golden
fixtures under ``tests/golden/`` that travel to the GPU box.  The dense
algebra calls the same numpy / scipy routines in the same order as the
reference (numpy 2.3.5 LAPACK ``dgesdd`` / ``dgeqrf+dorgqr``, scipy 1.18.1
sparsetools), so on this image it reproduces the reference bit-exactly.

Third-party arithmetic the reference delegates (not under /root/reference):
numpy 2.3.5 (``Generator(PCG64).standard_normal``, ``linalg.svd/qr`` on
OpenBLAS 0.3.30) and scipy 1.18.1 (sparsetools SpMM,
``csgraph.connected_components``).  Those versions are the pins.
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

EPS = float(np.finfo(np.float64).eps)
DENSE_CAPACITY = 100_000_000   # validation.py:15
BLOCK_CAPACITY = 4_000_000     # validation.py:19


class OracleCapacityError(RuntimeError):
    pass


class OracleStructuralError(RuntimeError):
    pass


# --------------------------------------------------------------------------
# validation.py:38-55  -- canonical float64 CSR
# --------------------------------------------------------------------------
def canonical_csr(A) -> sp.csr_matrix:
    if sp.issparse(A):
        out = A.tocsr().astype(np.float64)
    else:
        arr = np.asarray(A, dtype=np.float64)
        if arr.ndim != 2:
            raise ValueError("matrix must be 2-D")
        out = sp.csr_matrix(arr)
    out.sum_duplicates()
    out.eliminate_zeros()
    out.sort_indices()
    return out


# --------------------------------------------------------------------------
# reorder.py:149-287 -- hub removal + connected components (Algorithm 2)
# --------------------------------------------------------------------------
@dataclass
class Ordering:
    row_fwd: np.ndarray      # forward[old] = new
    col_fwd: np.ndarray
    m1: int
    n1: int
    m2: int
    n2: int
    spans: np.ndarray        # (B, 4) int64: row_start, row_len, col_start, col_len
    n_iterations: int
    gcc_sizes: tuple
    edges_visited: int = 0   # sum_t E_t (edges with both endpoints active at entry), SURVEY 8(d)
    nodes_visited: int = 0   # sum_t V_t (active nodes at entry)


def _hub_order(deg, active, quota):
    """reorder.py:149-155: active positive-degree nodes by (degree desc, id asc)."""
    cand = np.flatnonzero(active & (deg > 0))
    if quota <= 0 or cand.size == 0:
        return cand[:0]
    order = np.lexsort((cand, -deg[cand]))
    return cand[order[:min(quota, cand.size)]]


def reorder(m: int, n: int, indptr, indices, k: float) -> Ordering:
    """reorder.py:158-287 restated with vectorised component emission."""
    if not 0.0 < k < 1.0:
        raise ValueError(f"hub selection ratio k must be in (0, 1), got {k}")
    if m == 0 or n == 0:
        raise ValueError("graph has an empty node side")
    er = np.repeat(np.arange(m, dtype=np.int64), np.diff(np.asarray(indptr, dtype=np.int64)))
    ec = np.asarray(indices, dtype=np.int64)
    row_new = np.full(m, -1, dtype=np.int64)
    col_new = np.full(n, -1, dtype=np.int64)
    lo_t = lo_f = 0
    hi_t, hi_f = m - 1, n - 1
    act_t = np.ones(m, dtype=bool)
    act_f = np.ones(n, dtype=bool)
    spans = []
    gcc_sizes = []
    it = 0
    e_sum = v_sum = 0
    while True:
        it += 1
        q_t = math.ceil(k * int(act_t.sum()))          # reorder.py:196-199
        q_f = math.ceil(k * int(act_f.sum()))
        live = act_t[er] & act_f[ec]                    # edges inside the current graph
        er, ec = er[live], ec[live]
        e_sum += int(er.size)
        v_sum += int(act_t.sum()) + int(act_f.sum())
        deg_t = np.bincount(er, minlength=m)            # reorder.py:201-202
        deg_f = np.bincount(ec, minlength=n)
        hubs_t = _hub_order(deg_t, act_t, q_t)
        hubs_f = _hub_order(deg_f, act_f, q_f)
        row_new[hubs_t] = hi_t - np.arange(hubs_t.size)  # reorder.py:207-212
        col_new[hubs_f] = hi_f - np.arange(hubs_f.size)
        hi_t -= hubs_t.size
        hi_f -= hubs_f.size
        act_t[hubs_t] = False
        act_f[hubs_f] = False

        nodes = np.concatenate([np.flatnonzero(act_t), np.flatnonzero(act_f) + m])
        if nodes.size == 0:                              # reorder.py:224-226
            gcc_sizes.append(0)
            break
        keep = act_t[er] & act_f[ec]                     # reorder.py:215-220
        g = sp.csr_matrix((np.ones(int(keep.sum())), (er[keep], ec[keep] + m)), shape=(m + n, m + n))
        _, labels = connected_components(g, directed=False)
        lab = labels[nodes]
        # Component representative = smallest member id (nodes are ascending).
        uniq, first, size = np.unique(lab, return_index=True, return_counts=True)
        rep = nodes[first]
        corder = np.lexsort((rep, -size))               # (size desc, min id asc): reorder.py:234,247
        rank_of_label = np.empty(labels.max() + 1, dtype=np.int64)
        rank_of_label[uniq[corder]] = np.arange(uniq.size)
        crank = rank_of_label[lab]                       # 0 == giant component
        csize = size[corder]
        is_row = nodes < m
        rows_per = np.bincount(crank, weights=is_row, minlength=uniq.size).astype(np.int64)
        cols_per = csize - rows_per

        # Spoke components (rank >= 1) get the lowest free ids, in rank order,
        # members ascending within each side (reorder.py:246-257).
        sp_rows = rows_per[1:]
        sp_cols = cols_per[1:]
        row_off = lo_t + np.concatenate([[0], np.cumsum(sp_rows)[:-1]]) if sp_rows.size else sp_rows
        col_off = lo_f + np.concatenate([[0], np.cumsum(sp_cols)[:-1]]) if sp_cols.size else sp_cols
        sel = crank > 0
        snodes, srank = nodes[sel], crank[sel]
        o = np.lexsort((snodes, srank))
        snodes, srank = snodes[o], srank[o]
        start = np.concatenate([[0], np.cumsum(csize[1:])[:-1]]) if csize.size > 1 else np.zeros(0, np.int64)
        pos = np.arange(snodes.size) - start[srank - 1] if snodes.size else snodes
        r_mask = snodes < m
        row_new[snodes[r_mask]] = row_off[srank[r_mask] - 1] + pos[r_mask]
        col_new[snodes[~r_mask] - m] = (col_off[srank[~r_mask] - 1] + pos[~r_mask]
                                        - sp_rows[srank[~r_mask] - 1])
        if sp_rows.size:
            spans.append(np.stack([row_off, sp_rows, col_off, sp_cols], axis=1))
        lo_t += int(sp_rows.sum())
        lo_f += int(sp_cols.sum())

        giant = nodes[crank == 0]
        act_t = np.zeros(m, dtype=bool)
        act_f = np.zeros(n, dtype=bool)
        act_t[giant[giant < m]] = True
        act_f[giant[giant >= m] - m] = True
        g_t = int(rows_per[0])
        g_f = int(cols_per[0])
        gcc_sizes.append(g_t + g_f)
        if g_t < q_t or g_f < q_f:                       # reorder.py:268-269
            break

    rem_t = np.flatnonzero(act_t)                        # reorder.py:272-275
    rem_f = np.flatnonzero(act_f)
    row_new[rem_t] = lo_t + np.arange(rem_t.size)
    col_new[rem_f] = lo_f + np.arange(rem_f.size)
    spans_arr = np.concatenate(spans) if spans else np.zeros((0, 4), dtype=np.int64)
    return Ordering(row_new, col_new, lo_t, lo_f, m - lo_t, n - lo_f,
                    spans_arr.astype(np.int64), it, tuple(gcc_sizes), e_sum, v_sum)


# --------------------------------------------------------------------------
# reorder.py:290-337 -- permute + 2x2 partition
# --------------------------------------------------------------------------
def permute(A, row_fwd, col_fwd) -> sp.csr_matrix:
    """reorder.py:290-307: (i, j, v) -> (row_fwd[i], col_fwd[j], v), sorted CSR."""
    A = canonical_csr(A)
    coo = A.tocoo()
    out = sp.csr_matrix((coo.data, (row_fwd[coo.row], col_fwd[coo.col])), shape=A.shape)
    out.sort_indices()
    return out


def partition(Ap: sp.csr_matrix, o: Ordering):
    """reorder.py:310-337.  A11 is returned as the spoke CSR (blocks are sliced lazily)."""
    m1, n1 = o.m1, o.n1
    spoke = Ap[:m1, :n1].tocsr()
    # StructuralViolationError check (reorder.py:329-333), vectorised.
    if spoke.nnz:
        blk_of_row = np.full(m1, -1, dtype=np.int64)
        for b, (rs, rl, cs, cl) in enumerate(o.spans):
            blk_of_row[rs:rs + rl] = b
        rr = np.repeat(np.arange(m1), np.diff(spoke.indptr))
        b = blk_of_row[rr]
        cs = o.spans[np.maximum(b, 0), 2]
        cl = o.spans[np.maximum(b, 0), 3]
        inside = (b >= 0) & (spoke.indices >= cs) & (spoke.indices < cs + cl)
        if not inside.all():
            raise OracleStructuralError(f"{int((~inside).sum())} spoke-region nonzeros outside every block span")
    return spoke, Ap[:m1, n1:].tocsr(), Ap[m1:, :n1].tocsr(), Ap[m1:, n1:].tocsr()


# --------------------------------------------------------------------------
# svd.py -- factor container and SVD engines
# --------------------------------------------------------------------------
@dataclass
class Factors:
    U: object
    sigma: np.ndarray
    Vt: object
    is_sorted: bool

    @property
    def rank(self):
        return len(self.sigma)


def dense(M):
    return np.asarray(M.todense() if sp.issparse(M) else M, dtype=np.float64)


def block_svd(spoke: sp.csr_matrix, spans, alpha: float) -> Factors:
    """svd.py:141-193: per-block LAPACK SVD, keep ceil(alpha*min(h,w)), block-sparse CSR U/Vt."""
    if not 0.0 < alpha <= 1.0:
        raise ValueError("alpha must be in (0, 1]")
    ur, uc, uv, vr, vc, vv, sig = [], [], [], [], [], [], []
    row_off = col_off = rank_off = 0
    for rs, h, cs, w in np.asarray(spans, dtype=np.int64):
        h, w = int(h), int(w)
        if h == 0 or w == 0:
            row_off += h
            col_off += w
            continue
        if h * w > BLOCK_CAPACITY:
            raise OracleCapacityError("block exceeds capacity")
        blk = spoke[rs:rs + h, cs:cs + w].toarray()
        U, s, Vt = np.linalg.svd(blk, full_matrices=False)
        keep = int(np.ceil(alpha * min(h, w)))
        ur.append(np.repeat(np.arange(h), keep) + row_off)
        uc.append(np.tile(np.arange(keep), h) + rank_off)
        uv.append(U[:, :keep].ravel())
        vr.append(np.repeat(np.arange(keep), w) + rank_off)
        vc.append(np.tile(np.arange(w), keep) + col_off)
        vv.append(Vt[:keep].ravel())
        sig.append(s[:keep])
        row_off += h
        col_off += w
        rank_off += keep
    sigma = np.concatenate(sig) if sig else np.zeros(0)

    def build(r, c, v, shape):
        if not r:
            return sp.csr_matrix(shape)
        return sp.csr_matrix((np.concatenate(v), (np.concatenate(r), np.concatenate(c))), shape=shape)

    return Factors(build(ur, uc, uv, (row_off, rank_off)), sigma,
                   build(vr, vc, vv, (rank_off, col_off)), False)


def gaussian_sketch(seed: int, rows: int, cols: int) -> np.ndarray:
    """svd.py:131-132."""
    return np.random.default_rng(seed).standard_normal((rows, cols))


def randomized_svd(A, rank: int, seed: int) -> Factors:
    """svd.py:120-138 (no power iterations, 2r oversampling)."""
    A = canonical_csr(A)
    m, n = A.shape
    if not 1 <= rank <= min(m, n):
        raise ValueError(f"target rank {rank} out of range [1, {min(m, n)}]")
    X = gaussian_sketch(seed, n, 2 * rank)
    B = np.asarray(A @ X)
    Q, _ = np.linalg.qr(B)
    Y = np.asarray(A.T @ Q).T
    Us, s, Vt = np.linalg.svd(Y, full_matrices=False)
    return Factors(Q @ Us[:, :rank], s[:rank].copy(), Vt[:rank, :], True)


def dense_truncated_svd(M, rank: int) -> Factors:
    """svd.py:86-117 (dense_svd + truncate)."""
    M = dense(M)
    if M.shape[0] * M.shape[1] > DENSE_CAPACITY:
        raise OracleCapacityError("dense SVD exceeds capacity")
    if M.size and not np.all(np.isfinite(M)):
        raise ValueError("matrix contains non-finite entries")
    U, s, Vt = np.linalg.svd(M, full_matrices=False)
    if not 1 <= rank <= len(s):
        raise ValueError("target rank out of range")
    return Factors(U[:, :rank], s[:rank].copy(), Vt[:rank, :], True)


def inner_svd(dense_parts, sparse_parts, rank, n_cols, thr, seed, stack):
    """pinv.py:115-128: engine by rank < thr * n_cols."""
    if rank < thr * n_cols:
        pieces = [sp.csr_matrix(p) for p in dense_parts] + list(sparse_parts)
        inner = sp.vstack(pieces).tocsr() if stack == "v" else sp.hstack(pieces).tocsr()
        return randomized_svd(inner, rank, seed), "randomized"
    pieces = [np.asarray(p) for p in dense_parts] + [s.toarray() for s in sparse_parts]
    inner = np.vstack(pieces) if stack == "v" else np.hstack(pieces)
    return dense_truncated_svd(inner, rank), "dense"


def _empty(p, q):
    return Factors(np.zeros((p, 0)), np.zeros(0), np.zeros((0, q)), True)


def row_update(f11: Factors, A21, s: int, thr=0.3, seed=0):
    """pinv.py:131-171."""
    A21 = canonical_csr(A21)
    m2, n1 = A21.shape
    m1 = f11.U.shape[0]
    if f11.Vt.shape[1] != n1:
        raise ValueError("dimension mismatch")
    r_avail = f11.rank
    if s == 0:
        return _empty(m1 + m2, n1), None
    if not 1 <= s <= min(r_avail + m2, n1):
        raise ValueError("target rank out of range")
    if sp.issparse(f11.Vt):
        scaled = (sp.diags(f11.sigma) @ f11.Vt).tocsr()
        inner, eng = inner_svd([], [scaled, A21], s, n1, thr, seed, "v")
    else:
        scaled = f11.sigma[:, None] * f11.Vt
        inner, eng = inner_svd([scaled], [A21], s, n1, thr, seed, "v")
    iu = dense(inner.U)
    top = f11.U @ iu[:r_avail, :]
    U = np.vstack([np.asarray(top), iu[r_avail:, :]])
    return Factors(U, inner.sigma, dense(inner.Vt), True), eng


def column_update(f: Factors, T, r: int, thr=0.3, seed=0):
    """pinv.py:174-208."""
    T = canonical_csr(T)
    m, n2 = T.shape
    if f.U.shape[0] != m:
        raise ValueError("dimension mismatch")
    s_prev = f.rank
    n1 = f.Vt.shape[1]
    if r == 0:
        return _empty(m, n1 + n2), None
    if not 1 <= r <= min(s_prev + n2, m):
        raise ValueError("target rank out of range")
    scaled = dense(f.U) * f.sigma
    inner, eng = inner_svd([scaled], [T], r, s_prev + n2, thr, seed, "h")
    ivt = dense(inner.Vt)
    Vt = np.hstack([ivt[:, :s_prev] @ dense(f.Vt), ivt[:, s_prev:]])
    return Factors(dense(inner.U), inner.sigma, Vt, True), eng


@dataclass
class Pinv:
    V: np.ndarray
    sigma_dagger: np.ndarray
    Ut: np.ndarray
    tolerance_used: float
    all_filtered: bool


def pinv_from_svd(f: Factors, cutoff=EPS) -> Pinv:
    """pinv.py:211-231."""
    if not f.is_sorted:
        raise ValueError("pseudoinverse assembly requires sorted factors")
    p, q = f.U.shape[0], f.Vt.shape[1]
    smax = float(f.sigma[0]) if len(f.sigma) else 0.0
    tol = cutoff * smax * max(p, q, 1)
    keep = f.sigma > tol
    sd = np.zeros_like(f.sigma)
    np.divide(1.0, f.sigma, out=sd, where=keep)
    all_filtered = bool(len(f.sigma)) and not bool(keep.any())
    return Pinv(dense(f.Vt).T.copy(), sd, dense(f.U).T.copy(), tol, all_filtered)


def unfold(f: Factors, o: Ordering) -> Factors:
    """pinv.py:271-275."""
    return Factors(dense(f.U)[o.row_fwd, :], f.sigma.copy(), dense(f.Vt)[:, o.col_fwd], f.is_sorted)


def apply_pinv(pv: Pinv, B):
    """pinv.py:72-81 (Pseudoinverse.apply)."""
    if sp.issparse(B):
        inner = np.asarray((B.T @ pv.Ut.T).T)
    else:
        inner = pv.Ut @ np.asarray(B, dtype=np.float64)
    if inner.ndim == 1:
        return pv.V @ (pv.sigma_dagger * inner)
    return pv.V @ (pv.sigma_dagger[:, None] * inner)


def reconstruction_error(A, f: Factors, chunk=1 << 20) -> float:
    """svd.py:196-223 (Gram trick, cross term at A's stored coordinates)."""
    A = canonical_csr(A)
    U, Vt, s = dense(f.U), dense(f.Vt), f.sigma
    na = float(A.data @ A.data)
    if f.rank == 0:
        return math.sqrt(na)
    nb = float(((s[:, None] * s[None, :]) * (U.T @ U) * (Vt @ Vt.T)).sum())
    coo = A.tocoo()
    Us = U * s
    cross = 0.0
    step = max(1, chunk // max(1, f.rank))
    for lo in range(0, A.nnz, step):
        hi = min(A.nnz, lo + step)
        cross += float(np.einsum("ij,ji->i", Us[coo.row[lo:hi]], Vt[:, coo.col[lo:hi]]) @ coo.data[lo:hi])
    return math.sqrt(max(na - 2.0 * cross + nb, 0.0))


# --------------------------------------------------------------------------
# pinv.py:278-347 -- Algorithm 1 driver
# --------------------------------------------------------------------------
def fastpi(A, alpha=1.0, k=0.01, seed=0, thr=0.3, cutoff=EPS, keep_stages=True):
    """Returns a dict with every stage output (factors in reordered coordinates)."""
    if not 0.0 < alpha <= 1.0 or not 0.0 < k < 1.0:
        raise ValueError("alpha in (0,1], k in (0,1)")
    A = canonical_csr(A)
    m, n = A.shape
    if m == 0 or n == 0:
        raise ValueError("cannot factorize a zero-dimension matrix")
    if m < n:
        out = fastpi(A.T.tocsr(), alpha, k, seed, thr, cutoff, keep_stages)
        pv = out["pinv"]
        out["pinv"] = Pinv(pv.Ut.T.copy(), pv.sigma_dagger.copy(), pv.V.T.copy(),
                           pv.tolerance_used, pv.all_filtered)
        ft = out["factors"]
        out["factors"] = Factors(dense(ft.Vt).T, ft.sigma.copy(), dense(ft.U).T, True)
        out["transposed"] = True
        return out
    t = {}
    t0 = time.perf_counter()
    o = reorder(m, n, A.indptr, A.indices, k)
    Ap = permute(A, o.row_fwd, o.col_fwd)
    spoke, A12, A21, A22 = partition(Ap, o)
    t["reorder"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    f11 = block_svd(spoke, o.spans, alpha)
    t["block_svd"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    want_s = math.ceil(alpha * o.n1)
    s = min(want_s, f11.rank + o.m2, o.n1)
    clamped = s < want_s
    if clamped:
        warnings.warn(f"row-update target rank clamped from {want_s} to {s}")
    f_rows, eng_r = row_update(f11, A21, s, thr, seed + 1)
    t["row_update"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    T = sp.vstack([A12, A22]).tocsr() if o.n2 else sp.csr_matrix((m, 0))
    r = min(math.ceil(alpha * n), f_rows.rank + o.n2, m)
    f_full, eng_c = column_update(f_rows, T, r, thr, seed + 2)
    t["column_update"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pv = pinv_from_svd(unfold(f_full, o), cutoff)
    if pv.all_filtered:
        warnings.warn("all singular values filtered; returning the zero pseudoinverse")
    t["pinv_assembly"] = time.perf_counter() - t0
    out = {"ordering": o, "factors": f_full, "pinv": pv, "timings": t, "s": s, "r": r,
           "engines": (eng_r, eng_c), "clamped": clamped, "transposed": False}
    if keep_stages:
        out.update({"A_perm": Ap, "spoke": spoke, "A12": A12, "A21": A21, "A22": A22, "T": T,
                    "f11": f11, "f_rows": f_rows})
    return out
