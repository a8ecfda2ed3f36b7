"""GPU: reorder (Algorithm 2) bit-exact against the oracle / golden fixtures."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, problem
from oracle import fastpi_oracle as orc

pytestmark = pytest.mark.gpu


def _gpu_reorder(A, k):
    import paper_2011_04235_b200 as fp
    return fp.reorder(fp.to_bipartite(A), k)


def _check_against_oracle(A, k):
    A = orc.canonical_csr(A)
    r = _gpu_reorder(A, k)
    o = orc.reorder(A.shape[0], A.shape[1], A.indptr, A.indices, k)
    np.testing.assert_array_equal(r.row_perm.forward, o.row_fwd)
    np.testing.assert_array_equal(r.col_perm.forward, o.col_fwd)
    np.testing.assert_array_equal(r.spans, o.spans)
    assert (r.n_spoke_rows, r.n_spoke_cols, r.n_hub_rows, r.n_hub_cols, r.n_iterations) == \
        (o.m1, o.n1, o.m2, o.n2, o.n_iterations)
    assert r.gcc_sizes == tuple(o.gcc_sizes)
    # SURVEY 8(d) work accounting of the loop (sum_t E_t, sum_t V_t) equals the oracle's
    assert (r.edges_visited, r.nodes_visited) == (o.edges_visited, o.nodes_visited)
    return r


@pytest.mark.parametrize("name", ["c1", "c2", "c3r50"])
def test_reorder_golden(name):
    g = golden(name)
    p = problem(name)
    r = _gpu_reorder(p.A, p.workload.k)
    np.testing.assert_array_equal(r.row_perm.forward, g["row_fwd"])
    np.testing.assert_array_equal(r.col_perm.forward, g["col_fwd"])
    np.testing.assert_array_equal(r.spans, g["spans"])
    np.testing.assert_array_equal([r.n_spoke_rows, r.n_spoke_cols, r.n_hub_rows, r.n_hub_cols, r.n_iterations],
                                  g["sizes"])
    np.testing.assert_array_equal(r.gcc_sizes, g["gcc_sizes"])
    # BlockSpan tuples like the reference
    assert r.blocks[0] == tuple(g["spans"][0])


def test_reorder_c4_live_oracle():
    p = problem("c4")
    _check_against_oracle(p.A, p.workload.k)


def test_reorder_spec_shattered():
    g = golden("spec_examples")
    B = sp.block_diag([sp.csr_matrix(np.ones((2, 2)))] * 4).tocsr()
    r = _gpu_reorder(B, 0.1)
    assert r.n_iterations == 3
    np.testing.assert_array_equal(r.row_perm.forward, g["spec_shattered_row_fwd"])
    np.testing.assert_array_equal(r.col_perm.forward, g["spec_shattered_col_fwd"])


@pytest.mark.parametrize("seed", range(12))
def test_reorder_random_graphs(seed):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 400))
    n = int(rng.integers(1, 300))
    dens = float(rng.choice([0.0, 0.002, 0.01, 0.05, 0.2]))
    A = sp.random(m, n, density=dens, random_state=rng, format="csr")
    if seed % 3 == 0 and m > 3:
        A = sp.vstack([A, sp.csr_matrix((3, n))]).tocsr()  # empty rows
    k = float(rng.choice([0.01, 0.05, 0.2, 0.5]))
    _check_against_oracle(A, k)


def test_reorder_domain_errors():
    A = sp.csr_matrix(np.eye(3))
    with pytest.raises(ValueError):
        _gpu_reorder(A, 0.0)
    with pytest.raises(ValueError):
        _gpu_reorder(A, 1.0)


def _skewed(m, n, nnz, seed, row_const=None):
    """Power-law bipartite graph (many isolated / small spoke components in early iterations)."""
    rng = np.random.default_rng(seed)
    if row_const:
        rows = np.repeat(np.arange(m), row_const)
    else:
        rows = np.minimum((rng.pareto(1.2, nnz) * 3).astype(np.int64), m - 1)
        rows = rng.permutation(m)[rows]
    cols = np.minimum((rng.pareto(1.0, rows.size) * 2).astype(np.int64), n - 1)
    cols = rng.permutation(n)[cols]
    return sp.csr_matrix((np.ones(rows.size), (rows, cols)), shape=(m, n))


@pytest.mark.parametrize("host_loop", [False, True])
@pytest.mark.parametrize("case", [(60000, 20000, 150000, 0.01, 0), (40000, 30000, 60000, 0.005, 1),
                                  (30000, 8000, 0, 0.05, 2), (100000, 5000, 300000, 0.02, 3)])
def test_reorder_large_paths(case, host_loop, monkeypatch):
    """Large spoke stages (grid-wide radix passes, > 8192 nodes / components per iteration), tie
    splitting at the hub threshold (constant row degrees), both device drivers."""
    m, n, nnz, k, seed = case
    if host_loop:
        monkeypatch.setenv("FPI_REORDER_HOSTLOOP", "1")
    A = _skewed(m, n, nnz, seed, row_const=3 if nnz == 0 else None)
    _check_against_oracle(A, k)
