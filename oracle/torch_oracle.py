"""CPU/GPU ORACLE -- TEST INFRASTRUCTURE ONLY.

The reference's update stages (pinv.py:131-208 over svd.py:86-138) restated on torch tensors, so
the checker itself can run at the largest BASELINE config (c5: the column update's B and Q panels
are 2M x 2000 f64, 32 GB each -- too large for the box's host RAM next to the rest of the test,
comfortable in HBM).  Same algorithm, same order of operations as `fastpi_oracle` (and therefore
the reference): the Gaussian sketch is numpy's PCG64 stream (`fastpi_oracle.gaussian_sketch`,
bit-exact), B = inner @ X, Householder QR of B (`torch.linalg.qr`: geqrf + orgqr, as numpy's
`np.linalg.qr`), Y = (inner^T Q)^T, SVD of Y, U = Q Us[:, :r].  Only the BLAS / LAPACK engine
differs (cuBLAS / cuSPARSE / cuSOLVER through torch, or torch's CPU kernels), so results agree
with `fastpi_oracle` to rounding, up to the sign of each singular pair (LAPACK-internal, SURVEY
0.4); tests compare sign-invariant quantities.  Pinned against `fastpi_oracle` by
tests/test_oracle_golden.py (torch CPU kernels, c1 / c2 / c3@50 / c3@200) and
tests/test_fullsize_gpu.py (cuBLAS / cuSOLVER, c2 and c3@200).

Never imported by the product package; none of this runs the repo's CUDA library."""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .fastpi_oracle import canonical_csr, gaussian_sketch


def _t(x, dev):
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(dev, torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(dev)


def _csr(A: sp.csr_matrix, dev):
    import torch
    A = sp.csr_matrix(A)
    return torch.sparse_csr_tensor(torch.from_numpy(A.indptr.astype(np.int64)).to(dev),
                                   torch.from_numpy(A.indices.astype(np.int64)).to(dev),
                                   torch.from_numpy(A.data.astype(np.float64)).to(dev),
                                   size=A.shape, dtype=torch.float64)


def _spmm(S, X):
    """S (torch sparse CSR) @ X (dense); a 0-column operand short-circuits."""
    import torch
    if S.shape[1] == 0 or X.shape[1] == 0:
        return torch.zeros((S.shape[0], X.shape[1]), dtype=X.dtype, device=X.device)
    return torch.sparse.mm(S, X)


def column_update(U, sigma, Vt_prev, T, r: int, thr: float = 0.3, seed: int = 0, device="cuda"):
    """pinv.py:174-208 (column_update) with the inner SVD of pinv.py:115-128 / svd.py:120-138.

    U (m x s, dense), sigma (s,), Vt_prev (s x n1, dense): the row-update factors; T = [A12; A22]
    (scipy CSR, m x n2).  Returns (U m x r, sigma (r,), Vt r x (n1 + n2), engine) as torch tensors
    on `device` (engine: "randomized" / "dense")."""
    import torch
    dev = torch.device(device)
    T = canonical_csr(T)
    m, n2 = T.shape
    U = _t(U, dev)
    sig = _t(np.asarray(sigma), dev)
    Vt_prev = _t(Vt_prev, dev)
    s_prev = int(sig.numel())
    if U.shape[0] != m:
        raise ValueError("dimension mismatch")
    if not 1 <= r <= min(s_prev + n2, m):
        raise ValueError("target rank out of range")
    # inner = [U diag(sigma) | T] (pinv.py:202-203); the dense half's products are taken as
    # U (diag(sigma) X) and diag(sigma) (U^T Q) -- the same products, reassociated (rounding-level),
    # so the m x s panel U diag(sigma) (15 GB at c5) is never formed next to B and Q
    q = s_prev + n2
    if r < thr * q:                                    # pinv.py:122
        engine = "randomized"
        X = _t(gaussian_sketch(seed, q, 2 * r), dev)   # svd.py:131-132 (numpy PCG64 stream)
        Ts = _csr(T, dev)
        B = U @ (sig[:, None] * X[:s_prev]) + _spmm(Ts, X[s_prev:])  # svd.py:133  inner @ X
        del X
        Q = torch.linalg.qr(B, mode="reduced").Q       # svd.py:134  Householder (geqrf + orgqr)
        del B
        Tt = _csr(T.T.tocsr(), dev)
        Yt = torch.cat([sig[:, None] * (U.t() @ Q), _spmm(Tt, Q)], 0)   # svd.py:135  inner^T Q
        del Tt, Ts
        Us, s, Vti = torch.linalg.svd(Yt.t(), full_matrices=False)  # svd.py:136
        del Yt
        Uo = Q @ Us[:, :r]                             # svd.py:137
        del Q
        so, Vto = s[:r].clone(), Vti[:r].contiguous()
    else:
        engine = "dense"
        D = torch.cat([U * sig, _t(T.toarray(), dev)], 1)   # pinv.py:126-128 densified pieces
        Ud, s, Vtd = torch.linalg.svd(D, full_matrices=False)  # svd.py:105 (dense_svd) + truncate
        Uo, so, Vto = Ud[:, :r].contiguous(), s[:r].clone(), Vtd[:r].contiguous()
    Vt = torch.cat([Vto[:, :s_prev] @ Vt_prev, Vto[:, s_prev:]], 1)   # pinv.py:205-207
    return Uo, so, Vt, engine
