"""GPU: the reference's sparse.py products through the library's SpMM (sparse.py:20-39)."""
import numpy as np
import pytest
import scipy.sparse as sp

import paper_2011_04235_b200 as fp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,k", [((300, 200), 7), ((1, 50), 3), ((64, 1), 130), ((500, 40), 1)])
def test_multiply_and_transposed(shape, k):
    rng = np.random.default_rng(k)
    A = sp.random(*shape, density=0.05, random_state=k, format="csr")
    A[0, 0] = 3.0  # at least one entry
    B = rng.standard_normal((shape[1], k))
    C = rng.standard_normal((shape[0], k))
    np.testing.assert_allclose(fp.multiply(A, B), A @ B, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(fp.multiply_transposed(A, C), A.T @ C, rtol=1e-13, atol=1e-13)


def test_multiply_empty_and_errors():
    A = sp.csr_matrix((5, 4))
    np.testing.assert_array_equal(fp.multiply(A, np.ones((4, 2))), np.zeros((5, 2)))
    with pytest.raises(ValueError):
        fp.multiply(A, np.ones((3, 2)))
    with pytest.raises(ValueError):
        fp.multiply_transposed(A, np.ones((4, 2)))
