"""GPU: the regression harness's P@k (regression.py:89-124) -- score block and
top-k hit test on the device -- against the reference's evaluate, bit for bit
when the scores are exact (integer data) and to one tie flip otherwise."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2011_04235_b200 as fp
from paper_2011_04235_b200.regression import RegressionModel, predict_matrix

pytestmark = pytest.mark.gpu


def _p_at_k_reference(X, Y, Z, ks):
    """regression.py:101-124 restated (argsort(-scores, kind='stable'))."""
    S = np.asarray(X @ Z)
    top = np.argsort(-S, axis=1, kind="stable")
    D = np.asarray(Y.todense())
    hits = np.take_along_axis(D, top[:, :max(ks)], axis=1)
    m, L = S.shape
    chunk = max(1, 1 << 22 >> max(1, L).bit_length())
    tot = {k: 0.0 for k in ks}
    for lo in range(0, m, chunk):
        for k in ks:
            tot[k] += float(hits[lo:lo + chunk, :k].sum()) / k
    return {k: tot[k] / m for k in ks}


@pytest.mark.parametrize("m,n,L,ks", [(3000, 40, 37, [1, 3, 5]), (500, 17, 4000, [1, 2, 10]), (2, 3, 1, [1])])
def test_evaluate_exact_scores_bitwise(m, n, L, ks):
    rng = np.random.default_rng(m + L)
    X = sp.csr_matrix(rng.integers(-2, 3, (m, n)) * (rng.random((m, n)) < 0.3)).astype(np.float64)
    Z = rng.integers(-3, 4, (n, L)).astype(np.float64)  # small integers: exact sums, many ties
    Y = sp.csr_matrix((rng.random((m, L)) < 0.2).astype(np.float64))
    model = RegressionModel(coefficients=Z, method="fastpi", alpha=1.0, train_seconds=0.0)
    got = fp.evaluate(model, fp.MultiLabelDataset(X, Y), ks)
    assert got == _p_at_k_reference(X, Y, Z, ks)


def test_evaluate_real_scores():
    rng = np.random.default_rng(0)
    m, n, L = 2000, 60, 300
    X = sp.random(m, n, density=0.2, random_state=3, format="csr")
    Z = rng.standard_normal((n, L))
    Y = sp.csr_matrix((rng.random((m, L)) < 0.05).astype(np.float64))
    model = RegressionModel(coefficients=Z, method="fastpi", alpha=1.0, train_seconds=0.0)
    got = fp.evaluate(model, fp.MultiLabelDataset(X, Y), [1, 5])
    want = _p_at_k_reference(X, Y, Z, [1, 5])
    for k in (1, 5):
        assert abs(got[k] - want[k]) <= 1.0 / m  # at most one near-tie resolved differently
    np.testing.assert_allclose(predict_matrix(model, X), X @ Z, rtol=1e-12, atol=1e-12)
