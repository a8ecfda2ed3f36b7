"""GPU: SVD engines against the oracle / numpy (svd.py parity)."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import problem
from oracle import fastpi_oracle as orc
from parity import assert_block_sigma, assert_sigma

pytestmark = pytest.mark.gpu


def _rel_sigma(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape
    return np.abs(a - b).max() / max(b.max(), 1e-300) if b.size else 0.0


@pytest.mark.parametrize("p,q", [(1, 1), (5, 3), (3, 5), (200, 40), (40, 200), (1000, 333)])
def test_dense_svd(p, q):
    import paper_2011_04235_b200 as fp
    rng = np.random.default_rng(p + 3 * q)
    M = rng.standard_normal((p, q)) @ np.diag(np.logspace(0, -6, q))
    f = fp.dense_svd(M)
    s = np.linalg.svd(M, compute_uv=False)
    assert _rel_sigma(f.sigma, s) < 1e-12
    assert_sigma(f.sigma, s, label=f"dense {p}x{q}")
    assert np.abs((f.U * f.sigma) @ f.Vt - M).max() < 1e-12 * s[0]
    assert f.orthonormality_defect() < 1e-10


def test_dense_svd_rank_deficient():
    import paper_2011_04235_b200 as fp
    A = np.zeros((8, 4))
    A[:4, :4] = np.diag([5.0, 4.0, 3.0, 2.0])
    A[:, 3] = 0.0
    f = fp.dense_svd(A)
    np.testing.assert_allclose(f.sigma, [5, 4, 3, 0], atol=1e-14)
    assert f.orthonormality_defect() < 1e-12


@pytest.mark.parametrize("name", ["c1", "c2", "c3r50"])
def test_block_svd_matches_oracle(name):
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200._device import DeviceCSR
    from paper_2011_04235_b200.reorder import partition_original
    from paper_2011_04235_b200.svd import block_diagonal_svd_device
    p = problem(name)
    dev = DeviceCSR.from_host(p.A)
    r = fp.reorder(fp.to_bipartite(dev), p.workload.k)
    part = partition_original(dev, r)
    alpha = p.workload.alpha
    for a in (alpha, 1.0):
        f = block_diagonal_svd_device(part.a11, r.spans_device(), a)
        fo = orc.block_svd(part.a11.to_host(), r.spans, a)
        assert f.rank == fo.rank
        # per block, per value (tests/parity.py)
        assert_block_sigma(f.sigma, fo.sigma, r.spans, a, label=f"{name} alpha={a}")
        # block-sparse structure identical, reconstruction of the kept part identical up to signs
        Ug, Vg = f.U.toarray(), f.Vt.toarray()
        Uo, Vo = fo.U.toarray(), fo.Vt.toarray()
        assert np.abs((Ug * f.sigma) @ Vg - (Uo * fo.sigma) @ Vo).max() < 1e-9 * max(1.0, fo.sigma.max())
        assert f.orthonormality_defect() < 1e-10


def test_block_svd_spec_two_blocks():
    import paper_2011_04235_b200 as fp
    f = fp.block_diagonal_svd([np.diag([3.0, 1.0]), np.diag([2.0, 1.0])], 1.0)
    np.testing.assert_allclose(f.sigma, [3.0, 1.0, 2.0, 1.0], rtol=0, atol=1e-15)
    assert not f.is_sorted


@pytest.mark.parametrize("seed,rank", [(1, 10), (7, 40)])
def test_randomized_svd_matches_oracle(seed, rank):
    """Same sketch bits -> same subspace: sigma and U S Vt agree to rounding."""
    import paper_2011_04235_b200 as fp
    rng = np.random.default_rng(seed)
    A = sp.random(3000, 400, density=0.02, random_state=rng, format="csr") + \
        sp.csr_matrix(rng.standard_normal((3000, 1)) @ rng.standard_normal((1, 400)))
    A = sp.csr_matrix(A)
    f = fp.randomized_svd(A, rank, seed)
    fo = orc.randomized_svd(A, rank, seed)
    assert _rel_sigma(f.sigma, fo.sigma) < 1e-10
    assert_sigma(f.sigma, fo.sigma, label=f"randomized seed {seed} rank {rank}")
    Bg = (f.U * f.sigma) @ f.Vt
    Bo = (fo.U * fo.sigma) @ fo.Vt
    assert np.linalg.norm(Bg - Bo) <= 1e-9 * np.linalg.norm(Bo)
    assert f.orthonormality_defect() < 1e-10


@pytest.mark.parametrize("case", ["graded_1e6", "graded_1e14", "rank_deficient"])
def test_randomized_svd_ill_conditioned_sketch(case):
    """svd.py:120-138 on inputs whose sketch B = A X is ill conditioned or rank deficient: the
    reference orthonormalises with Householder QR (stable at any condition number), this engine
    with CholeskyQR (cond(B)^2) plus its fallbacks (explicit Y^T when the Cholesky factor is ill
    conditioned, an eigen-based factor when B^T B is not numerically positive definite).  Every
    singular value above the floor to <= 1e-9 of itself, U S Vt to <= 1e-8, against the oracle on
    the same sketch."""
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200 import _lib
    rng = np.random.default_rng(5)
    p, q, rank = 2500, 320, 30
    U, _ = np.linalg.qr(rng.standard_normal((p, q)))
    V, _ = np.linalg.qr(rng.standard_normal((q, q)))
    if case == "graded_1e6":
        sig = np.logspace(0, -6, q)          # cond(B) ~ sigma_1 / sigma_60 ~ 13
        sig[:60] = np.logspace(0, -6, 60)    # ... made 1e6 inside the sketch's reach
        sig[60:] = 1e-6 * np.logspace(0, -3, q - 60)
    elif case == "graded_1e14":
        sig = np.concatenate([np.logspace(0, -14, 60), 1e-14 * np.logspace(0, -2, q - 60)])
    else:
        sig = np.concatenate([np.linspace(3.0, 1.0, 20), np.zeros(q - 20)])   # rank 20 < 2 * rank
    A = sp.csr_matrix((U * sig) @ V.T)
    f = fp.randomized_svd(A, rank, 9)
    diag = _lib.svd_diag()
    fo = orc.randomized_svd(A, rank, 9)
    print(f"[ill-conditioned sketch] {case}: diag {diag}")
    assert_sigma(f.sigma, fo.sigma, label=f"randomized {case}")
    Bg = (f.U * f.sigma) @ f.Vt
    Bo = (fo.U * fo.sigma) @ fo.Vt
    assert np.linalg.norm(Bg - Bo) <= 1e-8 * np.linalg.norm(Bo)
    keep = fo.sigma > 1e-6 * fo.sigma[0]
    Ug, Vg = f.U[:, keep], f.Vt[keep]
    assert np.abs(Ug.T @ Ug - np.eye(keep.sum())).max() < 1e-8
    assert np.abs(Vg @ Vg.T - np.eye(keep.sum())).max() < 1e-8


def test_block_svd_large_tier_batched():
    """Blocks too large for shared memory (both orientations) go through the batched Gram path."""
    import paper_2011_04235_b200 as fp
    rng = np.random.default_rng(11)
    blocks = [sp.random(600, 90, density=0.3, random_state=rng, format="csr"),
              sp.random(80, 700, density=0.3, random_state=rng, format="csr"),
              sp.csr_matrix(rng.standard_normal((5, 4))),
              sp.random(450, 120, density=0.5, random_state=rng, format="csr")]
    for alpha in (0.03, 0.5):
        f = fp.block_diagonal_svd(blocks, alpha)
        spoke = sp.block_diag(blocks).tocsr()
        spans, ro, co = [], 0, 0
        for b in blocks:
            spans.append((ro, b.shape[0], co, b.shape[1]))
            ro += b.shape[0]
            co += b.shape[1]
        fo = orc.block_svd(spoke, np.array(spans), alpha)
        assert f.rank == fo.rank
        assert_block_sigma(f.sigma, fo.sigma, np.array(spans), alpha, label=f"large tier alpha={alpha}")
        Ug, Vg = f.U.toarray(), f.Vt.toarray()
        Uo, Vo = fo.U.toarray(), fo.Vt.toarray()
        assert np.abs((Ug * f.sigma) @ Vg - (Uo * fo.sigma) @ Vo).max() < 1e-9 * fo.sigma.max()
        assert f.orthonormality_defect() < 1e-10
