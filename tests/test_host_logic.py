"""CPU: host-side logic of the drop-in API -- config / validation guards, the
regression harness (split, precision@k, evaluate), the status-code -> exception
mapping of the C ABI, and the host utilities of sparse.py.  Where the reference
package is importable in this container it is the oracle (compared directly);
the GPU box has no /root/reference, so those cases skip there."""
import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2011_04235_b200 as fp
from paper_2011_04235_b200 import _lib
from paper_2011_04235_b200.regression import RegressionModel
from paper_2011_04235_b200.validation import (DENSE_CAPACITY, CapacityError, StructuralViolationError, as_csr,
                                              check_dense, check_vector)

REF_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ref():
    if not (REF_SRC / "fastpi" / "__init__.py").exists():
        pytest.skip("reference package not present (GPU box)")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import fastpi
    return fastpi


def _dataset(m=57, n=13, L=9, seed=0):
    rng = np.random.default_rng(seed)
    X = sp.random(m, n, density=0.3, random_state=seed, format="csr")
    Y = sp.csr_matrix((rng.random((m, L)) < 0.25).astype(np.float64))
    return X, Y


# ---- config / validation guards (pinv.py:32-46, validation.py)

@pytest.mark.parametrize("kw", [dict(alpha=0.0), dict(alpha=1.5), dict(k=0.0), dict(k=1.0), dict(alpha=-1)])
def test_config_rejects_out_of_range(kw):
    with pytest.raises(ValueError):
        fp.FastpiConfig(**kw)


def test_config_defaults_match_reference(ref):
    a, b = fp.FastpiConfig(), ref.FastpiConfig()
    for f in ("alpha", "k", "seed", "low_rank_threshold", "pinv_cutoff_factor"):
        assert getattr(a, f) == getattr(b, f), f


def test_validation_guards():
    with pytest.raises(ValueError):
        as_csr(np.zeros(3))
    with pytest.raises(ValueError):
        check_dense(np.zeros((2, 2, 2)))
    big = sp.csr_matrix((DENSE_CAPACITY // 10 + 1, 11))
    with pytest.raises(CapacityError):
        check_dense(big)
    with pytest.raises(ValueError):
        check_vector(np.zeros(4), length=5)
    assert check_vector(sp.csr_matrix(np.ones((1, 3)))).shape == (3,)


def test_status_codes_map_to_reference_exceptions():
    _lib.raise_for_status(_lib.FPI_OK, "")
    with pytest.raises(ValueError, match="bad rank"):
        _lib.raise_for_status(_lib.FPI_EDOMAIN, "bad rank")
    with pytest.raises(CapacityError):
        _lib.raise_for_status(_lib.FPI_ECAPACITY, "too big")
    with pytest.raises(StructuralViolationError):
        _lib.raise_for_status(_lib.FPI_ESTRUCT, "spoke outside block")
    for rc in (_lib.FPI_ECUDA, _lib.FPI_ENUMERIC):
        with pytest.raises(RuntimeError, match="fpi_x"):
            _lib.raise_for_status(rc, "boom", "fpi_x")
    assert issubclass(CapacityError, RuntimeError) and not issubclass(CapacityError, ValueError)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fp.fastpi(sp.random(20, 10, density=0.3, format="csr", random_state=1))


# ---- regression harness (regression.py:37-124)

def test_split_matches_reference(ref):
    X, Y = _dataset()
    for frac, seed in [(0.9, 0), (0.5, 3), (0.25, 11)]:
        tr, te = fp.split(fp.MultiLabelDataset(X, Y), fp.SplitSpec(frac, seed))
        rtr, rte = ref.split(ref.MultiLabelDataset(X, Y), ref.SplitSpec(frac, seed))
        for a, b in [(tr, rtr), (te, rte)]:
            assert (a.features != b.features).nnz == 0
            assert (a.labels != b.labels).nnz == 0


def test_split_contract():
    X, Y = _dataset(m=10)
    tr, te = fp.split(fp.MultiLabelDataset(X, Y), fp.SplitSpec(0.9, 5))
    assert tr.n_instances == 9 and te.n_instances == 1
    with pytest.raises(ValueError):
        fp.SplitSpec(1.0)
    with pytest.raises(ValueError):
        fp.split(fp.MultiLabelDataset(X[:1], Y[:1]), fp.SplitSpec())
    with pytest.raises(ValueError):
        fp.MultiLabelDataset(X, Y[:5])
    with pytest.raises(ValueError):
        fp.MultiLabelDataset(X, Y * 2.0)


def test_precision_at_k_matches_reference_with_ties(ref):
    rng = np.random.default_rng(4)
    for _ in range(50):
        L = int(rng.integers(1, 30))
        scores = rng.integers(0, 4, L).astype(float)  # many ties: stable ascending-index order
        labels = (rng.random(L) < 0.4).astype(float)
        for k in range(1, L + 1):
            assert fp.precision_at_k(scores, labels, k) == ref.precision_at_k(scores, labels, k)
    with pytest.raises(ValueError):
        fp.precision_at_k([1.0, 2.0], [1.0, 0.0], 3)
    with pytest.raises(ValueError):
        fp.precision_at_k([1.0, 2.0], [1.0, 0.0], 0)


def test_predict_matches_reference_and_evaluate_guards(ref):
    X, Y = _dataset(m=40, n=12, L=7, seed=2)
    Z = np.random.default_rng(9).standard_normal((12, 7))
    ours = RegressionModel(coefficients=Z, method="fastpi", alpha=1.0, train_seconds=0.0)
    theirs = ref.RegressionModel(coefficients=Z, method="fastpi", alpha=1.0, train_seconds=0.0)
    a = X[3].toarray().ravel()
    np.testing.assert_array_equal(fp.predict(ours, a), ref.predict(theirs, a))
    with pytest.raises(ValueError):
        fp.predict(ours, np.zeros(5))
    test = fp.MultiLabelDataset(X, Y)
    with pytest.raises(ValueError):  # argument checks happen before any device work
        fp.evaluate(ours, test, [8])
    with pytest.raises(ValueError):
        fp.evaluate(ours, test, [0, 2])
    assert fp.evaluate(ours, test, []) == {}


# ---- sparse.py host utilities

def test_sparsity_and_frobenius_match_reference(ref):
    rng = np.random.default_rng(1)
    rows, cols = rng.integers(0, 6, 30), rng.integers(0, 5, 30)
    vals = rng.standard_normal(30)
    vals[:4] = 0.0
    A = sp.csr_matrix((vals, (rows, cols)), shape=(6, 5))  # duplicates summed, explicit zeros kept
    A_dup = sp.csr_matrix((vals, cols, np.r_[0, np.cumsum(np.bincount(rows, minlength=6))][:7]), shape=(6, 5))
    for M in (A, A_dup, A.toarray()):
        assert fp.sparsity(M) == ref.sparsity(M)
        assert fp.frobenius_norm(M) == ref.frobenius_norm(M)
    with pytest.raises(ValueError):
        fp.sparsity(sp.csr_matrix((0, 3)))


def test_public_names_cover_reference_hot_path(ref):
    # everything the reference exports except its synthetic-corpus generator (synth.py)
    out_of_scope = {"SynthSpec", "synth_generate", "make_regression_dataset"}
    missing = set(ref.__all__) - set(fp.__all__) - out_of_scope
    assert not missing, missing


# ---- artefact formats (svd.py:226-250, pinv.py:242-268, reorder.py:340-370): byte-compatible both ways

def test_factor_and_pinv_files_roundtrip_with_reference(ref, tmp_path):
    import importlib
    osvd = importlib.import_module("paper_2011_04235_b200.svd")
    opinv = importlib.import_module("paper_2011_04235_b200.pinv")
    rng = np.random.default_rng(3)
    U, s, Vt = rng.standard_normal((7, 3)), np.array([3.0, 2.0, 0.5]), rng.standard_normal((3, 5))
    ours = fp.SvdFactors(U, s, Vt, is_sorted=True)
    osvd.save_factors(ours, tmp_path / "a.bin")
    rsvd, rpinv = importlib.import_module("fastpi.svd"), importlib.import_module("fastpi.pinv")
    rsvd.save_factors(ref.SvdFactors(U, s, Vt, is_sorted=True), tmp_path / "b.bin")
    assert (tmp_path / "a.bin").read_bytes() == (tmp_path / "b.bin").read_bytes()
    back = rsvd.load_factors(tmp_path / "a.bin")
    np.testing.assert_array_equal(back.U, U)
    mine = osvd.load_factors(tmp_path / "b.bin")
    np.testing.assert_array_equal(mine.Vt, Vt)
    assert mine.is_sorted

    V, sd, Ut = rng.standard_normal((5, 3)), np.array([0.5, 1.0, 0.0]), rng.standard_normal((3, 7))
    opinv.save_pseudoinverse(fp.Pseudoinverse(V, sd, Ut, 1.25e-13, False), tmp_path / "p.bin")
    rpinv.save_pseudoinverse(ref.Pseudoinverse(V, sd, Ut, 1.25e-13, False), tmp_path / "q.bin")
    assert (tmp_path / "p.bin").read_bytes() == (tmp_path / "q.bin").read_bytes()
    pl = opinv.load_pseudoinverse(tmp_path / "q.bin")
    np.testing.assert_array_equal(pl.sigma_dagger, sd)
    assert pl.tolerance_used == 1.25e-13 and not pl.all_filtered


def test_reorder_file_roundtrip_with_reference(ref, tmp_path):
    import importlib
    oreo = importlib.import_module("paper_2011_04235_b200.reorder")  # the package name is the function
    rmod = importlib.import_module("fastpi.reorder")
    A = sp.random(30, 20, density=0.2, random_state=4, format="csr")
    res = ref.reorder(ref.to_bipartite(A), 0.1)
    rmod.save_reorder_result(res, tmp_path / "r.txt")
    mine = oreo.load_reorder_result(tmp_path / "r.txt")
    np.testing.assert_array_equal(mine.row_perm.forward, res.row_perm.forward)
    np.testing.assert_array_equal(mine.col_perm.forward, res.col_perm.forward)
    assert [tuple(b) for b in mine.blocks] == [tuple(b) for b in res.blocks]
    oreo.save_reorder_result(mine, tmp_path / "s.txt")
    assert (tmp_path / "s.txt").read_text() == (tmp_path / "r.txt").read_text()
