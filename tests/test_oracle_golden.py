"""CPU: the oracle (numpy restatement) against the golden fixtures written from
the unmodified reference (oracle/pin_against_reference.py).  Also pins the
seeded workload generator (input hashes)."""
import numpy as np
import pytest

from conftest import golden, problem
from oracle import fastpi_oracle as orc
from oracle.pin_against_reference import csr_hash

SMALL = ["c1", "c2", "c3r50", "c3r100", "c3r200"]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference_fixture(name):
    g = golden(name)
    p = problem(name)
    assert csr_hash(p.A) == str(g["A_sha256"]), "workload generator drifted"
    assert csr_hash(p.Y) == str(g["Y_sha256"])
    w = p.workload
    out = orc.fastpi(p.A, w.alpha, w.k, w.seed)
    o = out["ordering"]
    np.testing.assert_array_equal(o.row_fwd, g["row_fwd"])
    np.testing.assert_array_equal(o.col_fwd, g["col_fwd"])
    np.testing.assert_array_equal(o.spans, g["spans"])
    np.testing.assert_array_equal([o.m1, o.n1, o.m2, o.n2, o.n_iterations], g["sizes"])
    np.testing.assert_array_equal(o.gcc_sizes, g["gcc_sizes"])
    np.testing.assert_array_equal(out["f11"].sigma, g["f11_sigma"])
    np.testing.assert_array_equal(out["f_rows"].sigma, g["f_rows_sigma"])
    np.testing.assert_array_equal(out["factors"].sigma, g["sigma"])
    np.testing.assert_array_equal(out["pinv"].sigma_dagger, g["sigma_dagger"])
    Z = orc.apply_pinv(out["pinv"], p.Y)
    if "Z" in g:
        np.testing.assert_array_equal(Z, g["Z"])
    else:
        np.testing.assert_array_equal(Z[g["Z_rows_idx"]], g["Z_rows"])


def test_spec_examples_fixture():
    g = golden("spec_examples")
    import scipy.sparse as sp
    f = orc.block_svd(sp.block_diag([sp.csr_matrix(np.diag([3.0, 1.0])), sp.csr_matrix(np.diag([2.0, 1.0]))]).tocsr(),
                      np.array([[0, 2, 0, 2], [2, 2, 2, 2]]), 1.0)
    np.testing.assert_array_equal(f.sigma, g["spec_two_blocks_sigma"])
    np.testing.assert_array_equal(f.sigma, [3.0, 1.0, 2.0, 1.0])
    B = sp.block_diag([sp.csr_matrix(np.ones((2, 2)))] * 4).tocsr()
    o = orc.reorder(8, 8, B.indptr, B.indices, 0.1)
    assert o.n_iterations == int(g["spec_shattered_T"][0]) == 3
    np.testing.assert_array_equal(o.row_fwd, g["spec_shattered_row_fwd"])
    pv = orc.pinv_from_svd(orc.Factors(np.eye(2), np.array([2.0, 0.0]), np.eye(2), True))
    np.testing.assert_array_equal(pv.sigma_dagger, [0.5, 0.0])


def test_reorder_edge_cases_oracle():
    """Empty rows / isolated columns / single row (oracle-only structural checks)."""
    import scipy.sparse as sp
    A = sp.csr_matrix((np.ones(3), ([0, 0, 2], [1, 3, 3])), shape=(4, 5))
    o = orc.reorder(4, 5, A.indptr, A.indices, 0.3)
    assert sorted(o.row_fwd.tolist()) == list(range(4))
    assert sorted(o.col_fwd.tolist()) == list(range(5))
    with pytest.raises(ValueError):
        orc.reorder(4, 5, A.indptr, A.indices, 1.0)


@pytest.mark.parametrize("name", ["c1", "c2", "c3r50", "c3r200"])
def test_torch_oracle_column_update_matches_oracle(name):
    """Pin of oracle/torch_oracle.py (the column-update restatement the c5 GPU test runs in HBM)
    against the numpy oracle, itself pinned bit-exact to the reference: torch CPU kernels instead of
    OpenBLAS, so sigma per value and the sign-invariant product U S Vt agree to rounding."""
    from oracle import torch_oracle
    from parity import assert_sigma, lowrank_rel_factored
    p = problem(name)
    w = p.workload
    out = orc.fastpi(p.A, w.alpha, w.k, w.seed)
    fr = out["f_rows"]
    U, sig, Vt, eng = torch_oracle.column_update(orc.dense(fr.U), fr.sigma, orc.dense(fr.Vt), out["T"], out["r"],
                                                 0.3, w.seed + 2, device="cpu")
    want = out["factors"]
    assert eng == out["engines"][1]
    assert_sigma(sig.numpy(), want.sigma, tol=1e-12, label=f"{name} torch-oracle column update")
    rel = lowrank_rel_factored(U.numpy(), sig.numpy(), Vt.numpy(), orc.dense(want.U), want.sigma, orc.dense(want.Vt))
    print(f"{name}: torch oracle vs numpy oracle column update, low-rank rel {rel:.2e} ({eng})")
    assert rel <= 1e-12
