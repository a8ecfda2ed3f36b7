"""GPU: the row-sharded multi-GPU path (sharded.py) on one device -- world size 1
against the single-GPU pipeline, shard-wise projection identities of the
apply, and two ranks sharing the device over gloo (functional check of the
exchange pattern; the kernels never wait on each other)."""
import os
import socket

import numpy as np
import pytest
import torch

from conftest import problem

pytestmark = pytest.mark.gpu


def _cfg(name):
    import paper_2011_04235_b200 as fp
    w = problem(name).workload
    return fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)


@pytest.mark.parametrize("name", ["c2", "c3r50", "c3r200"])
def test_world1_sharded_matches_single_gpu(name):
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    from paper_2011_04235_b200.pinv import fastpi_device
    from paper_2011_04235_b200.sharded import fastpi_sharded
    p = problem(name)
    A, Y = DeviceCSR.from_host(p.A), DeviceCSR.from_host(p.Y)
    ref = fastpi_device(A, _cfg(name))
    res = fastpi_sharded(A, _cfg(name))
    s_ref = ref.factors.sigma
    np.testing.assert_allclose(d2h(res.sigma), s_ref, rtol=1e-10, atol=1e-12 * s_ref[0])
    np.testing.assert_allclose(res.pseudoinverse.sigma_dagger, ref.pseudoinverse.sigma_dagger, rtol=1e-9)
    Z_ref = d2h(ref.pseudoinverse.apply_device(Y))
    Z = d2h(res.pseudoinverse.apply_device(Y))
    assert np.abs(Z - Z_ref).max() <= 1e-8 * np.abs(Z_ref).max()


def test_projection_shards_sum_to_full():
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import DeviceCSR, d2h, empty, h2d
    rng = np.random.default_rng(0)
    import scipy.sparse as sp
    m, r, L, n = 400, 9, 23, 50
    U = h2d(rng.standard_normal((m, r)))
    row_fwd = h2d(rng.permutation(m).astype(np.int64))
    Y = DeviceCSR.from_host(sp.random(m, L, density=0.1, random_state=1, format="csr"))
    Wfull = empty((L, r))
    _lib.call("fpi_pinv_project_csr", 0, m, r, _lib.ptr(U), _lib.ptr(row_fwd), m, L, Y.nnz, _lib.ptr(Y.indptr),
              _lib.ptr(Y.indices), _lib.ptr(Y.values), _lib.ptr(Wfull))
    acc = np.zeros((L, r))
    for r0, r1 in [(0, 130), (130, 131), (131, 131), (131, 400)]:
        Wi = empty((L, r))
        Ui = U[r0:r1].contiguous()
        _lib.call("fpi_pinv_project_csr", r0, r1 - r0, r, _lib.ptr(Ui), _lib.ptr(row_fwd), m, L, Y.nnz,
                  _lib.ptr(Y.indptr), _lib.ptr(Y.indices), _lib.ptr(Y.values), _lib.ptr(Wi))
        acc += d2h(Wi)
    Yh = Y.to_host().toarray()
    Wref = Yh.T @ d2h(U)[d2h(row_fwd)]
    np.testing.assert_allclose(d2h(Wfull), Wref, atol=1e-12)
    np.testing.assert_allclose(acc, Wref, atol=1e-12)
    # lift: Z = V diag(s+) W^T in original column order
    sdag = h2d(rng.uniform(0.5, 2.0, r))
    Vt = h2d(rng.standard_normal((r, n)))
    col_fwd = h2d(rng.permutation(n).astype(np.int64))
    Z = empty((n, L))
    W = h2d(Wref.copy())
    _lib.call("fpi_pinv_lift", n, r, _lib.ptr(sdag), _lib.ptr(Vt), _lib.ptr(col_fwd), L, _lib.ptr(W), _lib.ptr(Z))
    Zref = (d2h(Vt).T * d2h(sdag)) @ Wref.T
    np.testing.assert_allclose(d2h(Z), Zref[d2h(col_fwd)], atol=1e-11)


def _worker(rank, world, port, out_dir, name):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2011_04235_b200._device import DeviceCSR, d2h
        from paper_2011_04235_b200.sharded import fastpi_sharded
        p = problem(name)
        A, Y = DeviceCSR.from_host(p.A), DeviceCSR.from_host(p.Y)
        res = fastpi_sharded(A, _cfg(name))
        Z = d2h(res.pseudoinverse.apply_device(Y))
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), sig=d2h(res.sigma), Z=Z)
    finally:
        torch.distributed.destroy_process_group()


def test_two_ranks_one_device_gloo(tmp_path):
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    from paper_2011_04235_b200.sharded import fastpi_sharded
    name = "c2"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.multiprocessing.spawn(_worker, args=(2, port, str(tmp_path), name), nprocs=2, join=True)
    r0, r1 = np.load(tmp_path / "rank0.npz"), np.load(tmp_path / "rank1.npz")
    np.testing.assert_array_equal(r0["sig"], r1["sig"])
    np.testing.assert_array_equal(r0["Z"], r1["Z"])
    p = problem(name)
    single = fastpi_sharded(DeviceCSR.from_host(p.A), _cfg(name))
    s1 = d2h(single.sigma)
    np.testing.assert_allclose(r0["sig"], s1, rtol=1e-11, atol=1e-13 * s1[0])
    Z1 = d2h(single.pseudoinverse.apply_device(DeviceCSR.from_host(p.Y)))
    assert np.abs(r0["Z"] - Z1).max() <= 1e-9 * np.abs(Z1).max()


def _bsvd_worker(rank, world, port, out_dir, name):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2011_04235_b200._device import DeviceCSR, d2h
        from paper_2011_04235_b200.reorder import partition_original, reorder_device
        from paper_2011_04235_b200.sharded import Comm
        from paper_2011_04235_b200.svd import block_diagonal_svd_device
        p = problem(name)
        A = DeviceCSR.from_host(p.A)
        o = reorder_device(A, p.workload.k)
        part = partition_original(A, o, transposes=False)
        f = block_diagonal_svd_device(part.a11, o.spans_device(), p.workload.alpha, Comm()).device()
        np.savez(os.path.join(out_dir, f"bsvd{rank}.npz"), sig=d2h(f.sigma), u=d2h(f.U.values), v=d2h(f.Vt.values))
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("name,world", [("c2", 2), ("c2", 3), ("c4", 2)])
def test_block_svd_sharded_gloo(tmp_path, name, world):
    """A11 blocks dealt over `world` ranks (fpi_block_svd_shard) + one all-reduce = the single-rank
    block SVD, bit for bit (every block is factored by the same kernel on whichever rank owns it)."""
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    from paper_2011_04235_b200.reorder import partition_original, reorder_device
    from paper_2011_04235_b200.svd import block_diagonal_svd_device
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.multiprocessing.spawn(_bsvd_worker, args=(world, port, str(tmp_path), name), nprocs=world, join=True)
    p = problem(name)
    A = DeviceCSR.from_host(p.A)
    o = reorder_device(A, p.workload.k)
    part = partition_original(A, o, transposes=False)
    f = block_diagonal_svd_device(part.a11, o.spans_device(), p.workload.alpha).device()
    ref = (d2h(f.sigma), d2h(f.U.values), d2h(f.Vt.values))
    for r in range(world):
        got = np.load(tmp_path / f"bsvd{r}.npz")
        for key, want in zip(("sig", "u", "v"), ref):
            np.testing.assert_array_equal(got[key], want)
