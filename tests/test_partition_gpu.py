"""GPU: permutation + 2x2 partition against the oracle (bit-exact structure and values)."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import problem
from oracle import fastpi_oracle as orc

pytestmark = pytest.mark.gpu


def _same_csr(a, b):
    a, b = sp.csr_matrix(a), sp.csr_matrix(b)
    assert a.shape == b.shape
    np.testing.assert_array_equal(a.indptr, b.indptr)
    np.testing.assert_array_equal(a.indices, b.indices)
    np.testing.assert_array_equal(a.data, b.data)


@pytest.mark.parametrize("name", ["c1", "c2", "c3r50"])
def test_partition_matches_oracle(name):
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200._device import DeviceCSR
    from paper_2011_04235_b200.reorder import partition_original
    p = problem(name)
    dev = DeviceCSR.from_host(p.A)
    r = fp.reorder(fp.to_bipartite(dev), p.workload.k)
    o = orc.reorder(*p.A.shape, p.A.indptr, p.A.indices, p.workload.k)
    Ap = orc.permute(p.A, o.row_fwd, o.col_fwd)
    spoke, A12, A21, A22 = orc.partition(Ap, o)
    part = partition_original(dev, r)
    _same_csr(part.a11.to_host(), spoke)
    _same_csr(part.T.to_host(), sp.vstack([A12, A22]).tocsr())
    _same_csr(part.Tt.to_host(), sp.vstack([A12, A22]).T.tocsr())
    _same_csr(part.a21.to_host(), A21)
    _same_csr(part.a21t.to_host(), A21.T.tocsr())
    assert part.info.nnz_a12 == A12.nnz and part.info.nnz_a22 == A22.nnz
    # public API: apply_permutation + partition on the permuted matrix
    Ap_gpu = fp.apply_permutation(p.A, r.row_perm, r.col_perm)
    _same_csr(Ap_gpu, Ap)
    blocks, g12, g21, g22 = fp.partition(Ap_gpu, r)
    _same_csr(g12, A12)
    _same_csr(g21, A21)
    _same_csr(g22, A22)
    assert len(blocks) == len(o.spans)
    assert sum(b.nnz for b in blocks) == spoke.nnz


def test_structural_violation():
    import paper_2011_04235_b200 as fp
    A = sp.csr_matrix(np.array([[1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]]))
    r = fp.reorder(fp.to_bipartite(A), 0.3)
    # corrupt: a matrix with an off-block entry in the spoke region
    B = A.tolil()
    B[0, 1] = 5.0
    Bp = fp.apply_permutation(B.tocsr(), r.row_perm, r.col_perm)
    if r.n_spoke_rows >= 2 and r.n_spoke_cols >= 2:
        with pytest.raises(fp.StructuralViolationError):
            fp.partition(Bp, r)


def test_canonicalize_sums_duplicates_drops_zeros():
    from paper_2011_04235_b200._device import DeviceCSR
    rows = np.array([0, 0, 1, 1, 2, 2, 2])
    cols = np.array([3, 1, 2, 2, 0, 4, 4])
    vals = np.array([1.0, 2.0, 3.0, 4.0, 0.0, 5.0, -5.0])
    A = sp.coo_matrix((vals, (rows, cols)), shape=(3, 5)).tocsr()
    A.has_sorted_indices = False
    dev = DeviceCSR.from_host(sp.csr_matrix((vals, cols, np.array([0, 2, 4, 7])), shape=(3, 5)))
    ref = orc.canonical_csr(sp.csr_matrix((vals, cols, np.array([0, 2, 4, 7])), shape=(3, 5)))
    _same_csr(dev.to_host(), ref)


def test_transpose():
    from paper_2011_04235_b200._device import DeviceCSR
    A = sp.random(300, 170, density=0.03, random_state=np.random.default_rng(1), format="csr")
    dev = DeviceCSR.from_host(A)
    _same_csr(dev.transpose().to_host(), orc.canonical_csr(A).T.tocsr())
