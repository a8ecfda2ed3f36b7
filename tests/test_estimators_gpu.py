"""GPU: the baselines and utilities around the hot path --
estimators.factorize / compute_pseudoinverse for "fastpi", "randpi" and "dense",
reconstruction_error, and the sklearn wrappers -- against the oracle."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2011_04235_b200 as fp
from oracle import fastpi_oracle as orc

pytestmark = pytest.mark.gpu


def _A(m=300, n=120, seed=0):
    A = sp.random(m, n, density=0.05, random_state=seed, format="csr")
    A = A + sp.csr_matrix((np.ones(n), (np.arange(n) % m, np.arange(n))), shape=(m, n))  # no empty columns
    return A.tocsr()


@pytest.mark.parametrize("method", ["randpi", "dense"])
def test_baseline_factorize_matches_oracle(method):
    A = _A()
    cfg = fp.FastpiConfig(alpha=0.2, k=0.05, seed=4)
    f, reordering, timings = fp.factorize(A, method, cfg)
    rank = int(np.ceil(cfg.alpha * min(A.shape)))
    want = orc.randomized_svd(A, rank, cfg.seed) if method == "randpi" else orc.dense_truncated_svd(A, rank)
    assert reordering is None and f.rank == rank
    np.testing.assert_allclose(f.sigma, want.sigma, rtol=1e-9, atol=1e-12 * want.sigma[0])
    U, Vt = np.asarray(f.U), np.asarray(f.Vt)
    np.testing.assert_allclose((U * f.sigma) @ Vt, (orc.dense(want.U) * want.sigma) @ orc.dense(want.Vt), atol=1e-9)


@pytest.mark.parametrize("method", ["fastpi", "randpi", "dense"])
def test_compute_pseudoinverse_moore_penrose_at_full_rank(method):
    A = _A(200, 60, seed=2)
    cfg = fp.FastpiConfig(alpha=1.0, k=0.1, seed=1)
    pv, factors, timings = fp.compute_pseudoinverse(A, method, cfg)
    Ad = A.toarray()
    X = np.asarray(pv.apply(Ad))           # pinv(A) A: the orthogonal projector onto row(A)
    assert np.abs(Ad @ X - Ad).max() <= 1e-8 * np.abs(Ad).max()      # A A+ A = A
    assert np.abs(X - X.T).max() <= 1e-8                              # (A+ A)^T = A+ A
    assert np.abs(X @ X - X).max() <= 1e-8                            # idempotent


def test_reconstruction_error_matches_oracle():
    A = _A(400, 150, seed=5)
    cfg = fp.FastpiConfig(alpha=0.1, k=0.05, seed=2)
    f, _, _ = fp.factorize(A, "randpi", cfg)
    host = orc.Factors(np.asarray(f.U), f.sigma, np.asarray(f.Vt), True)
    got = fp.reconstruction_error(A, f)
    want = orc.reconstruction_error(A, host)
    assert abs(got - want) <= 1e-10 * max(want, 1.0)


def test_lowrank_svd_estimator_roundtrip():
    A = _A(250, 80, seed=7)
    est = fp.LowRankSVD(method="dense", alpha=0.5, seed=0).fit(A)
    Z = est.transform(A)
    assert Z.shape == (250, 40)
    back = est.inverse_transform(Z)
    assert back.shape == (250, 80)
