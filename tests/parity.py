"""Parity helpers shared by the GPU tests (test infrastructure; never imported by the product).

The singular-value bar of BASELINE.json's north star is a relative error of <= 1e-9 on EACH
singular value.  `assert_sigma` checks exactly that, value by value, for every sigma_i at or
above SIG_FLOOR * sigma_max.  Below that floor LAPACK's own sigma_i (dgesdd, the reference's
engine) is only normwise accurate -- its error is ~eps * sigma_max, which exceeds 1e-9 * sigma_i
once sigma_i < ~1e-7 sigma_max -- so those values are held to the absolute bound
SIG_TOL * SIG_FLOOR * sigma_max, the same bound the relative test gives at the floor.
The normwise figure max_i |d sigma_i| / sigma_max is printed beside the per-value one.

Low-rank comparisons (reconstruction U S Vt against the oracle's) are computed without the
cancellation of ||A||^2 + ||B||^2 - 2<A, B>: A - B = [Ua Sa, -Ub Sb] [Vta; Vtb] and the norm is
taken through the QR of the short stacked factor.
"""
from __future__ import annotations

import numpy as np

SIG_TOL = 1e-9
REC_TOL = 1e-8
SIG_FLOOR = 1e-4


def sigma_errors(got, want, floor: float = SIG_FLOOR):
    """(max per-value relative error over sigma_i >= floor*sigma_max,
        max |d sigma_i| / sigma_max over the values below the floor,
        normwise max |d sigma_i| / sigma_max, number of values checked per value)."""
    got = np.asarray(got, dtype=np.float64).ravel()
    want = np.asarray(want, dtype=np.float64).ravel()
    assert got.shape == want.shape, (got.shape, want.shape)
    if want.size == 0:
        return 0.0, 0.0, 0.0, 0
    smax = float(np.abs(want).max())
    if smax == 0.0:
        d = float(np.abs(got).max())
        return d, d, d, 0
    d = np.abs(got - want)
    big = want >= floor * smax
    per = float((d[big] / want[big]).max()) if big.any() else 0.0
    small = float(d[~big].max() / smax) if (~big).any() else 0.0
    return per, small, float(d.max() / smax), int(big.sum())


def assert_sigma(got, want, tol: float = SIG_TOL, label: str = "", floor: float = SIG_FLOOR):
    per, small, nw, n = sigma_errors(got, want, floor)
    print(f"[sigma] {label}: per-value rel {per:.3e} over {n} values, below-floor {small:.3e}, "
          f"normwise {nw:.3e}")
    assert per <= tol, f"{label}: per-value relative sigma error {per:.3e} > {tol:.1e}"
    assert small <= tol * floor, f"{label}: sub-floor sigma error {small:.3e} > {tol * floor:.1e}"
    return per, nw


def assert_block_sigma(got, want, spans, alpha: float, tol: float = SIG_TOL, label: str = ""):
    """P2: per block (svd.py:154-178), every kept sigma against LAPACK's, relative to itself (block
    floor = SIG_FLOOR * that block's sigma_max).  Returns (worst per-value, worst normwise,
    number of non-degenerate blocks)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    spans = np.asarray(spans, dtype=np.int64).reshape(-1, 4)
    h, w = spans[:, 1], spans[:, 3]
    nd = (h > 0) & (w > 0)
    keep = np.ceil(alpha * np.minimum(h[nd], w[nd])).astype(np.int64)
    assert keep.sum() == want.size
    if want.size == 0:
        return 0.0, 0.0, 0
    start = np.concatenate([[0], np.cumsum(keep)[:-1]])
    bmax = np.maximum.reduceat(np.abs(want), start)
    bmax_e = np.repeat(bmax, keep)
    d = np.abs(got - want)
    big = want >= SIG_FLOOR * bmax_e
    safe = np.where(bmax_e > 0, bmax_e, 1.0)
    per = float((d[big] / want[big]).max()) if big.any() else 0.0
    small = float((d[~big] / safe[~big]).max()) if (~big).any() else 0.0
    nw = float((d / safe).max())
    worst = int(np.repeat(np.arange(keep.size), keep)[np.argmax(np.where(big, d / np.where(big, want, 1), 0))])
    print(f"[sigma] {label}: {keep.size} blocks, per-value rel {per:.3e} (worst block {worst}: "
          f"{tuple(spans[nd][worst])}), below-floor {small:.3e}, normwise {nw:.3e}")
    assert per <= tol, f"{label}: per-value block sigma error {per:.3e} > {tol:.1e}"
    assert small <= tol * SIG_FLOOR
    return per, nw, int(keep.size)


def lowrank_rel_factored(Ua, sa, Vta, Ub, sb, Vtb) -> float:
    """||Ua Sa Vta - Ub Sb Vtb||_F / ||sb|| (B's factors orthonormal), numpy, via a QR of the tall
    left factor [Ua Sa, -Ub Sb]."""
    Ua, Vta, Ub, Vtb = (np.asarray(x) for x in (Ua, Vta, Ub, Vtb))
    M = np.hstack([Ua * sa, -(Ub * sb)])
    _, R = np.linalg.qr(M)
    D = R @ np.vstack([Vta, Vtb])
    return float(np.linalg.norm(D) / np.linalg.norm(sb))


def lowrank_rel_factored_gpu(Ua, sa, Vta, Ub, sb, Vtb, chunk_rows: int = 1 << 18) -> float:
    """Same quantity for factors too large for the host QR (c5: m = 2M rows), on the GPU with
    torch as the checker: QR of the short right factor N^T = [Vta; Vtb]^T (n x 2s), then
    ||A - B|| = ||[Ua Sa, -Ub Sb] R^T||, accumulated over row chunks (a direct difference, no
    squared-norm cancellation)."""
    import torch
    dev = torch.device("cuda")

    def t(x):
        return x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))

    Vta, Vtb = t(Vta).to(dev), t(Vtb).to(dev)
    sa_t, sb_t = t(np.asarray(sa)).to(dev), t(np.asarray(sb)).to(dev)
    s_a = Vta.shape[0]
    N = torch.cat([Vta, Vtb], 0)
    _, R = torch.linalg.qr(N.t().contiguous(), mode="reduced")     # N^T = Q R
    Rt = R.t()                                                      # (sa+sb) x (sa+sb)
    Ra = sa_t[:, None] * Rt[:s_a]
    Rb = sb_t[:, None] * Rt[s_a:]
    m = Ua.shape[0]
    acc = torch.zeros((), dtype=torch.float64, device=dev)
    for lo in range(0, m, chunk_rows):
        hi = min(m, lo + chunk_rows)
        ua = t(Ua[lo:hi]).to(dev)
        ub = t(Ub[lo:hi]).to(dev)
        D = ua @ Ra - ub @ Rb
        acc += (D * D).sum()
    return float(acc.sqrt().item() / float(np.linalg.norm(np.asarray(sb))))
