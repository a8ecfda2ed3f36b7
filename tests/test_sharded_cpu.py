"""CPU: the row-sharded column update (paper_2011_04235_b200/sharded.py) over
gloo with world size 2, against world size 1 and against the oracle.

The sharded algorithm is written against an ``ops`` interface; here it runs on
``TorchCpuOps`` (torch CPU / numpy stand-ins for the library kernels, test-only)
so the decomposition itself -- what is local, what is all-reduced, what is
replicated -- is checked without a GPU.  The GPU kernels behind ``GpuOps`` are
checked against the same quantities in tests/test_sharded_gpu.py."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle import fastpi_oracle as orc
from paper_2011_04235_b200.sharded import Comm, column_update_shard, shard_bounds


class TorchCpuOps:
    """Host stand-ins for GpuOps (test infrastructure only)."""

    def zeros(self, shape):
        return torch.zeros(shape, dtype=torch.float64)

    def sketch(self, seed, rows, cols):
        return torch.from_numpy(np.random.default_rng(seed).standard_normal((rows, cols)))

    def gemm(self, A, B, ta=False, tb=False, out=None, beta=0.0):
        R = (A.T if ta else A) @ (B.T if tb else B)
        if out is None:
            return R.contiguous()
        out.copy_(R + (beta * out if beta else 0.0))
        return out

    def gram(self, B):
        return (B.T @ B).contiguous()

    def spmm(self, A, X, out, beta=0.0):
        R = torch.from_numpy(np.asarray(A @ X.numpy()))
        out.copy_(R + (beta * out if beta else 0.0))
        return out

    def scale_rows(self, A, s):
        A.mul_(s[:, None])
        return A

    def orth_factor(self, G):
        L = torch.linalg.cholesky(G)
        return torch.linalg.inv(L)

    def dense_svd(self, M, rank):
        U, s, Vt = torch.linalg.svd(M, full_matrices=False)
        U, s, Vt = U[:, :rank].contiguous(), s[:rank].contiguous(), Vt[:rank].contiguous()
        self.canonical_signs(U, Vt)
        return U, s, Vt

    def transpose(self, A):
        return A.T.contiguous()

    def canonical_signs(self, U, Vt):
        idx = Vt.abs().argmax(dim=1)
        sg = torch.sign(Vt[torch.arange(Vt.shape[0]), idx])
        sg[sg == 0] = 1.0
        Vt.mul_(sg[:, None])
        U.mul_(sg[None, :])

    def slice_rows(self, A, r0, r1):
        return A[r0:r1]

    def csr_rows(self, A, r0, r1):
        return A[r0:r1].tocsr()

    def csr_transpose(self, A):
        return A.T.tocsr()

    def copy(self, A):
        return A.clone()

    def hstack_lift(self, Vt, Vt_prev, s, n1, n2):
        return torch.cat([Vt[:, :s] @ Vt_prev, Vt[:, s:]], dim=1)


def _problem(m=240, s=18, n1=35, n2=30, seed=5):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, s)))
    sigma = np.sort(rng.uniform(1.0, 10.0, s))[::-1].copy()
    Vt = np.linalg.qr(rng.standard_normal((n1, s)))[0].T.copy()
    T = sp.random(m, n2, density=0.08, random_state=seed, format="csr")
    return U, sigma, Vt, T


def _run_shard(rank, world, U, sigma, Vt_prev, T, r, seed):
    comm = Comm()
    r0, r1 = shard_bounds(U.shape[0], world)[rank]
    ops = TorchCpuOps()
    T_i = T[r0:r1].tocsr()
    Ui, sig, Vt = column_update_shard(ops, comm, torch.from_numpy(U[r0:r1].copy()), torch.from_numpy(sigma),
                                      torch.from_numpy(Vt_prev), T_i, T_i.T.tocsr(), U.shape[0], r, seed)
    return Ui.numpy(), sig.numpy(), Vt.numpy()


def _worker(rank, world, port, out_dir, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Ui, sig, Vt = _run_shard(rank, world, *args)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), U=Ui, sig=sig, Vt=Vt)
    finally:
        torch.distributed.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_bounds():
    assert shard_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert shard_bounds(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    for m in (0, 1, 17, 1000):
        for w in (1, 2, 3, 8):
            b = shard_bounds(m, w)
            assert b[0][0] == 0 and b[-1][1] == m
            assert all(x[1] == y[0] for x, y in zip(b, b[1:]))


def test_world1_matches_oracle_column_update():
    U, sigma, Vt_prev, T = _problem()
    r, seed = 12, 7   # r < 0.3 (s + n2) -> randomized engine
    Ui, sig, Vt = _run_shard(0, 1, U, sigma, Vt_prev, T, r, seed)
    f = orc.Factors(U, sigma, Vt_prev, True)
    ref, eng = orc.column_update(f, T, r, 0.3, seed)
    assert eng == "randomized"
    np.testing.assert_allclose(sig, ref.sigma, rtol=1e-10)
    # the low-rank reconstruction is basis/sign invariant
    np.testing.assert_allclose((Ui * sig) @ Vt, (orc.dense(ref.U) * ref.sigma) @ orc.dense(ref.Vt), atol=1e-9)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_world_matches_world1(tmp_path, world):
    U, sigma, Vt_prev, T = _problem()
    r, seed = 12, 7
    U1, s1, Vt1 = _run_shard(0, 1, U, sigma, Vt_prev, T, r, seed)
    torch.multiprocessing.spawn(_worker, args=(world, _free_port(), str(tmp_path), (U, sigma, Vt_prev, T, r, seed)),
                                nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{i}.npz") for i in range(world)]
    for p in parts[1:]:  # replicated outputs agree bit for bit across ranks
        np.testing.assert_array_equal(p["sig"], parts[0]["sig"])
        np.testing.assert_array_equal(p["Vt"], parts[0]["Vt"])
    Uw = np.vstack([p["U"] for p in parts])
    np.testing.assert_allclose(parts[0]["sig"], s1, rtol=1e-12)
    np.testing.assert_allclose(parts[0]["Vt"], Vt1, atol=1e-11)
    np.testing.assert_allclose(Uw, U1, atol=1e-11)
