"""GPU: the largest BASELINE config (c5: 2M x 200k, 30M nnz, r = 1000, 3000 labels) at full size,
checked through size-independent properties (the CPU oracle needs hours here):
  * the permutations are bijections, the spans tile the spoke region, T / m1 / n1 are consistent;
  * sigma is positive and sorted, r = min(ceil(alpha n), s + n2, m) (pinv.py:336);
  * U and V have orthonormal columns (1e-9: the small SVD of Y goes through its Gram, so the
    right vectors of the smallest kept singular values carry ~eps cond(Y)^2; the parity bar on
    reconstruction / Z is 1e-8);
  * Z = pinv(A) Y agrees with V diag(sigma+) (U^T (Y x)) on random probes x (1e-10): the apply path
    against an independent small-product route."""
import math

import numpy as np
import pytest

from conftest import problem

pytestmark = pytest.mark.gpu


def test_c5_fullsize_properties():
    import torch
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    from paper_2011_04235_b200.pinv import fastpi_device
    p = problem("c5")
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    A = DeviceCSR.from_host(p.A)
    stats = {}
    res = fastpi_device(A, cfg, stats=stats)
    m, n = p.A.shape
    o = res.reordering
    rf, cf = o.row_perm.forward, o.col_perm.forward
    assert np.array_equal(np.sort(rf), np.arange(m)) and np.array_equal(np.sort(cf), np.arange(n))
    sp = np.asarray(o.spans)
    assert sp[:, 1].sum() == o.n_spoke_rows and sp[:, 3].sum() == o.n_spoke_cols
    assert np.all(sp[1:, 0] == sp[:-1, 0] + sp[:-1, 1]) and np.all(sp[1:, 2] == sp[:-1, 2] + sp[:-1, 3])
    assert o.n_spoke_rows + o.n_hub_rows == m and o.n_spoke_cols + o.n_hub_cols == n

    d = res.factors.device()
    r = res.factors.rank
    s = stats["s"]
    assert r == min(math.ceil(w.alpha * n), s + o.n_hub_cols, m)
    sig = d2h(d.sigma)
    assert np.all(sig > 0) and np.all(np.diff(sig) <= 0)

    U, Vt = d.U, d.Vt
    eye = torch.eye(r, dtype=torch.float64, device="cuda")
    assert (U.t() @ U - eye).abs().max().item() < 1e-9
    assert (Vt @ Vt.t() - eye).abs().max().item() < 1e-9

    Y = DeviceCSR.from_host(p.Y)
    Z = res.pseudoinverse.apply_device(Y)                       # n x L, original column order
    pv = res.pseudoinverse._device()
    Ys = torch.sparse_csr_tensor(Y.indptr, Y.indices.long(), Y.values, size=Y.shape)
    rng = np.random.default_rng(0)
    for _ in range(3):
        x = torch.from_numpy(rng.standard_normal((Y.shape[1], 1))).cuda()
        yx = torch.sparse.mm(Ys, x)                              # m x 1, original rows
        uy = pv.U.t() @ yx[torch.argsort(pv.row_fwd)]            # U in reordered rows
        zr = pv.Vt.t() @ (pv.sdag[:, None] * uy)                 # n x 1, reordered columns
        want = zr[pv.col_fwd]                                    # original column order
        got = Z @ x
        assert ((got - want).norm() / want.norm()).item() < 1e-10
