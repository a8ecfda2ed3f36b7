"""GPU: the sharded multi-GPU engine (csrc/sharded.cu, sharded.py) on one device -- world size 1
against the single-GPU pipeline, shard-wise projection identities of the apply, the NCCL
communicator on a world of one, and 2 / 3 ranks sharing the device over the callback
communicator (gloo: a functional check of the exchange pattern; the kernels never wait on each
other)."""
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


@pytest.mark.parametrize("name", ["c2", "c3r50", "c3r200", "c4"])
def test_world1_sharded_matches_single_gpu(name):
    """The sharded engine (csrc/sharded.cu) with a world-of-one communicator against the single-GPU
    pipeline: every singular value to 1e-10 relative (the engines take different but equivalent
    routes: B-route Gram / left finish vs the cost-model choices), Z to 1e-9.  c3r200 takes the
    dense column engine: the replicated fallback."""
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    from paper_2011_04235_b200.pinv import fastpi_device
    from paper_2011_04235_b200.sharded import fastpi_sharded
    p = problem(name)
    A, Y = DeviceCSR.from_host(p.A), DeviceCSR.from_host(p.Y)
    ref = fastpi_device(A, _cfg(name))
    st = {}
    res = fastpi_sharded(A, _cfg(name), stats=st)
    assert st["sharded"] == (name != "c3r200")
    s_ref = ref.factors.sigma
    s_got = d2h(res.sigma)
    assert np.max(np.abs(s_got - s_ref) / s_ref) <= 1e-10
    np.testing.assert_allclose(res.pseudoinverse.sigma_dagger, ref.pseudoinverse.sigma_dagger, rtol=1e-9)
    Z_ref = d2h(ref.pseudoinverse.apply_device(Y))
    Z = res.pseudoinverse.apply(Y)
    assert np.linalg.norm(Z - Z_ref) <= 1e-9 * np.linalg.norm(Z_ref)


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
        from paper_2011_04235_b200.sharded import Comm, fastpi_sharded
        p = problem(name)
        A, Y = DeviceCSR.from_host(p.A), DeviceCSR.from_host(p.Y)
        comm = Comm()
        st = {}
        res = fastpi_sharded(A, _cfg(name), comm, stats=st)
        assert comm.kind == "callback" and st["sharded"]
        cols, Zl = res.pseudoinverse.apply_local(Y)
        Z = res.pseudoinverse.apply(Y)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), sig=d2h(res.sigma), Z=Z, cols=cols, Zl=d2h(Zl),
                 plan=st["plan"])
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("name,world", [("c2", 2), ("c2", 3), ("c4", 2)])
def test_ranks_one_device_gloo(tmp_path, name, world):
    """`world` ranks sharing the one GPU, exchanges over the callback communicator (gloo): sigma and
    the gathered Z bit-identical on every rank; every rank's Z rows are exactly its columns; against
    one rank: sigma to 1e-12 relative, Z to 1e-9.  (A functional check of the exchange pattern;
    the ranks' kernels never wait on one another.)"""
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    from paper_2011_04235_b200.sharded import fastpi_sharded
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    torch.multiprocessing.spawn(_worker, args=(world, port, str(tmp_path), name), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for q in parts[1:]:
        np.testing.assert_array_equal(q["sig"], parts[0]["sig"])
        np.testing.assert_array_equal(q["Z"], parts[0]["Z"])
    cols = np.concatenate([q["cols"] for q in parts])
    p = problem(name)
    assert np.array_equal(np.sort(cols), np.arange(p.A.shape[1]))  # the ranks' columns tile Z
    for q in parts:
        np.testing.assert_array_equal(q["Zl"], q["Z"][q["cols"]])
    plan = parts[0]["plan"]
    assert plan[0, 0] == 0 and all(plan[i, 1] == plan[i + 1, 0] for i in range(world - 1))
    single = fastpi_sharded(DeviceCSR.from_host(p.A), _cfg(name))
    s1 = d2h(single.sigma)
    assert np.max(np.abs(parts[0]["sig"] - s1) / s1) <= 1e-12
    Z1 = single.pseudoinverse.apply(DeviceCSR.from_host(p.Y))
    assert np.linalg.norm(parts[0]["Z"] - Z1) <= 1e-9 * np.linalg.norm(Z1)


@pytest.mark.parametrize("name,world", [("c2", 3), ("c4", 4)])
def test_block_svd_ranges_tile_the_full_factorization(name, world):
    """The ranks' block ranges (fpi_shard_plan) factored separately (fpi_block_svd_range) give,
    value for value, the single-rank block SVD: each block is factored by the same kernel
    whichever rank owns it; outside its range a rank's values are zero and its keep range is
    exactly the kept ranks of its blocks."""
    import ctypes as C
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import DeviceCSR, d2h, empty
    from paper_2011_04235_b200.reorder import partition_original, reorder_device
    from paper_2011_04235_b200.sharded import shard_plan
    from paper_2011_04235_b200.svd import block_diagonal_svd_device
    p = problem(name)
    A = DeviceCSR.from_host(p.A)
    o = reorder_device(A, p.workload.k)
    part = partition_original(A, o, transposes=False)
    full = block_diagonal_svd_device(part.a11, o.spans_device(), p.workload.alpha).device()
    ref = [d2h(full.sigma), d2h(full.U.values), d2h(full.Vt.values)]
    plan = shard_plan(o, part.T, world)
    spans = o.spans_device()
    nsp = int(spans.numel() // 4)
    m1, n1 = part.a11.shape
    acc = [np.zeros_like(x) for x in ref]
    kr_all = []
    for i in range(world):
        bp = _lib.BlockPlan()
        _lib.call("fpi_block_svd_plan", nsp, _lib.ptr(spans), float(p.workload.alpha), C.byref(bp))
        U = DeviceCSR.empty(m1, bp.rank11, bp.nnz_u11)
        Vt = DeviceCSR.empty(bp.rank11, n1, bp.nnz_vt11)
        sig = empty(bp.rank11)
        kr = (C.c_int64 * 2)()
        _lib.call("fpi_block_svd_range", m1, n1, _lib.ptr(part.a11.indptr), _lib.ptr(part.a11.indices),
                  _lib.ptr(part.a11.values), nsp, _lib.ptr(spans), float(p.workload.alpha), int(plan[i, 0]),
                  int(plan[i, 1]), _lib.ptr(sig), _lib.ptr(U.indptr), _lib.ptr(U.indices), _lib.ptr(U.values),
                  _lib.ptr(Vt.indptr), _lib.ptr(Vt.indices), _lib.ptr(Vt.values), C.byref(bp), kr)
        kr_all.append((kr[0], kr[1]))
        got = [d2h(sig), d2h(U.values), d2h(Vt.values)]
        sl = d2h(sig)
        assert not sl[:kr[0]].any() and not sl[kr[1]:].any()
        np.testing.assert_array_equal(sl[kr[0]:kr[1]], ref[0][kr[0]:kr[1]])
        for a_, g in zip(acc, got):
            a_ += g
    for a_, want in zip(acc, ref):
        np.testing.assert_array_equal(a_, want)
    assert kr_all[0][0] == 0 and kr_all[-1][1] == len(ref[0])
    assert all(kr_all[i][1] == kr_all[i + 1][0] for i in range(world - 1))


def test_nccl_library_communicator_world1(tmp_path):
    """The library's NCCL loader and a single-rank communicator built from an NCCL unique id
    (the box has one GPU: NCCL cannot put two ranks on it)."""
    from paper_2011_04235_b200 import _lib
    import ctypes as C
    uid, err = C.create_string_buffer(128), C.create_string_buffer(256)
    assert _lib.load().fpi_comm_nccl_id(uid, err, len(err)) == 0, err.value
    h = _lib.handle()
    lib = _lib.load()
    assert lib.fpi_comm_init_nccl(h, uid.raw, 0, 1) == 0, lib.fpi_last_error(h)
    from paper_2011_04235_b200._device import d2h, h2d
    x = h2d(np.arange(10, dtype=np.float64))
    _lib.call("fpi_comm_allreduce", _lib.ptr(x), 10)
    np.testing.assert_array_equal(d2h(x), np.arange(10))
    rk, wd = C.c_int(), C.c_int()
    _lib.call("fpi_comm_info", C.byref(rk), C.byref(wd))
    assert (rk.value, wd.value) == (0, 1)
    assert lib.fpi_comm_free(h) == 0
