"""GPU: FastPI pipeline parity.

P3 stage-wise: the oracle's row_update / column_update are fed the GPU's own
upstream factors (removing LAPACK's arbitrary singular-vector signs) and must
agree with the GPU stage: every singular value to <= 1e-9 relative to itself
(tests/parity.py), reconstruction and U S Vt <= 1e-8 relative.
P4 end-to-end on the dense-column-update configs (c1, c3r200): sigma <= 1e-9,
Z <= 1e-8 against the golden fixtures written from the reference.
P5 randomized-column configs: end-to-end quality is reported, not bit-level.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, problem
from oracle import fastpi_oracle as orc
from parity import REC_TOL, assert_block_sigma, assert_sigma, lowrank_rel_factored

pytestmark = pytest.mark.gpu


def _run(name):
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200._device import DeviceCSR
    from paper_2011_04235_b200.pinv import fastpi_device
    p = problem(name)
    w = p.workload
    stats = {}
    res = fastpi_device(DeviceCSR.from_host(p.A), fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed), stats=stats)
    return p, res, stats


def _host_factors(f):
    return orc.Factors(f.U, f.sigma.copy(), f.Vt, f.is_sorted)


def _lowrank_rel(fa, fb):
    A = (np.asarray(fa.U) * fa.sigma) @ np.asarray(fa.Vt)
    B = (np.asarray(fb.U) * fb.sigma) @ np.asarray(fb.Vt)
    return np.linalg.norm(A - B) / np.linalg.norm(B)


@pytest.mark.parametrize("name", ["c1", "c2", "c3r50", "c3r100", "c3r200"])
def test_stagewise_parity(name):
    _check_stagewise(name)


@pytest.mark.parametrize("heavy", ["0", "16", "256"])
@pytest.mark.parametrize("name", ["c2", "c3r50", "c3r100"])
def test_stagewise_parity_gram_route(name, heavy, monkeypatch):
    """The column update's Z = H X route (gram_route.cu) forced on the small randomized-column
    configs, with no / some / all-qualifying heavy (densified) columns of T."""
    monkeypatch.setenv("FPI_GRAM_ROUTE", "1")
    monkeypatch.setenv("FPI_GRAM_HEAVY", heavy)
    _check_stagewise(name)


@pytest.mark.parametrize("gram", [False, True])
@pytest.mark.parametrize("name", ["c2", "c3r50", "c3r100"])
def test_stagewise_parity_sparse_core(name, gram, monkeypatch):
    """The dense core of T (sparse_core.cu: heavy rows x heavy columns on DMMA, the rest as a
    gather SpMM) forced on the small randomized-column configs, through the B route and -- with
    the inner-Gram route forced -- through the lift alone."""
    from paper_2011_04235_b200 import _lib
    monkeypatch.setenv("FPI_SPMM_CORE", "force")
    if gram:
        monkeypatch.setenv("FPI_GRAM_ROUTE", "1")
    _check_stagewise(name)
    info = _lib.sparse_core_info()
    assert info["rows"] > 0 and info["cols"] > 0 and info["core_nnz"] > 0, info
    monkeypatch.setenv("FPI_SPMM_CORE", "0")
    _run(name)
    assert _lib.sparse_core_info()["core_nnz"] == 0


def test_gram_route_h11_shortcut_declined_for_scaled_factor(monkeypatch):
    """The inner-Gram route takes H11 = Sigma^2 when its probe finds D^T D = I (the row update's U).
    column_update(2 U, Sigma / 2, Vt) is the same inner matrix [U Sigma | T] with a D that is not
    orthonormal: the probe must decline the shortcut and the factors must agree with the unscaled
    call (pinv.py:174-208 computes with the U it is given)."""
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200.pinv import column_update
    monkeypatch.setenv("FPI_GRAM_ROUTE", "1")
    p, res, st = _run("c2")
    fr = st["f_rows"]
    T = st["part"].T.to_host()
    w = p.workload
    U, sig, Vt = np.asarray(fr.U), np.asarray(fr.sigma), np.asarray(fr.Vt)
    fa = column_update(fp.SvdFactors(U, sig, Vt, True), T, st["r"], seed=w.seed + 2)
    fb = column_update(fp.SvdFactors(2.0 * U, 0.5 * sig, Vt, True), T, st["r"], seed=w.seed + 2)
    assert_sigma(fb.sigma, fa.sigma, tol=1e-11, label="scaled-U column update")
    assert _lowrank_rel(fb, fa) <= 1e-10
    monkeypatch.setenv("FPI_GRAM_H11_GEMM", "1")
    fc = column_update(fp.SvdFactors(U, sig, Vt, True), T, st["r"], seed=w.seed + 2)
    assert_sigma(fc.sigma, fa.sigma, tol=1e-11, label="H11 shortcut vs Gram")
    assert _lowrank_rel(fc, fa) <= 1e-10


def _check_stagewise(name):
    p, res, st = _run(name)
    g = golden(name)
    w = p.workload
    # reorder-derived quantities exact
    assert (st["m1"], st["n1"], st["m2"], st["n2"], st["T"]) == tuple(g["sizes"])
    assert (st["s"], st["r"]) == tuple(g["s_r"])
    assert list(st["engines"]) == [1 if e == "randomized" else 2 for e in g["engines"]]
    # block stage vs reference fixture: every kept sigma of every block
    assert_block_sigma(st["f11"].sigma, g["f11_sigma"], g["spans"], w.alpha, label=f"{name} f11")
    part = st["part"]
    A21 = part.a21.to_host()
    T = part.T.to_host()
    # row update fed with the GPU's f11
    fo_rows, _ = orc.row_update(_host_factors(st["f11"]), A21, st["s"], 0.3, w.seed + 1)
    fr = st["f_rows"]
    assert_sigma(fr.sigma, fo_rows.sigma, label=f"{name} row update")
    assert _lowrank_rel(fr, fo_rows) <= REC_TOL
    # column update fed with the GPU's row-update factors
    fo_full, _ = orc.column_update(_host_factors(fr), T, st["r"], 0.3, w.seed + 2)
    ff = res.factors
    assert_sigma(ff.sigma, fo_full.sigma, label=f"{name} column update")
    assert _lowrank_rel(ff, fo_full) <= REC_TOL
    assert ff.orthonormality_defect() < 1e-8
    # sign-invariant reconstruction of the reordered matrix
    Ap = orc.permute(p.A, res.reordering.row_perm.forward, res.reordering.col_perm.forward)
    rec_gpu = orc.reconstruction_error(Ap, _host_factors(ff))
    rec_ref = orc.reconstruction_error(Ap, fo_full)
    assert abs(rec_gpu - rec_ref) <= REC_TOL * rec_ref
    # Z from the GPU pseudoinverse vs the oracle's Z of the same (GPU-fed) factors
    pv_o = orc.pinv_from_svd(orc.unfold(fo_full, orc.Ordering(res.reordering.row_perm.forward,
                                                              res.reordering.col_perm.forward, 0, 0, 0, 0,
                                                              np.zeros((0, 4), np.int64), 0, ())))
    Zo = orc.apply_pinv(pv_o, p.Y)
    Zg = res.pseudoinverse.apply(p.Y)
    assert np.linalg.norm(Zg - Zo) <= REC_TOL * np.linalg.norm(Zo)


@pytest.mark.parametrize("name", ["c1", "c3r200"])
def test_end_to_end_dense_column_configs(name):
    p, res, st = _run(name)
    g = golden(name)
    assert_sigma(res.factors.sigma, g["sigma"], label=f"{name} end to end")
    Z = res.pseudoinverse.apply(p.Y)
    if "Z" in g:
        assert np.linalg.norm(Z - g["Z"]) <= REC_TOL * np.linalg.norm(g["Z"])
    else:
        assert np.linalg.norm(Z[g["Z_rows_idx"]] - g["Z_rows"]) <= REC_TOL * np.linalg.norm(g["Z_rows"])
    assert abs(np.linalg.norm(Z) - g["Z_fro"][0]) <= REC_TOL * g["Z_fro"][0]
    Ap = orc.permute(p.A, res.reordering.row_perm.forward, res.reordering.col_perm.forward)
    rec = orc.reconstruction_error(Ap, _host_factors(res.factors))
    assert abs(rec - g["recon"][0]) <= REC_TOL * g["recon"][0]


@pytest.mark.parametrize("name", ["c2", "c3r50", "c3r100"])
def test_end_to_end_randomized_column_configs_quality(name):
    """P5: sign-dependent configs -- report the end-to-end gap, require equal approximation quality."""
    p, res, st = _run(name)
    g = golden(name)
    rel = np.abs(res.factors.sigma - g["sigma"]).max() / g["sigma"][0]
    Ap = orc.permute(p.A, res.reordering.row_perm.forward, res.reordering.col_perm.forward)
    rec = orc.reconstruction_error(Ap, _host_factors(res.factors))
    print(f"{name}: end-to-end sigma gap {rel:.3e}, recon {rec:.6g} vs reference {g['recon'][0]:.6g}")
    assert rel < 5e-2
    assert rec <= 1.02 * g["recon"][0]


def test_public_api_fit_and_spec_examples():
    import paper_2011_04235_b200 as fp
    # diag(5,4,3,2) padded to 8x4, alpha=1 -> A+ A = I
    A = np.zeros((8, 4))
    A[:4, :4] = np.diag([5.0, 4.0, 3.0, 2.0])
    res = fp.fastpi(sp.csr_matrix(A), fp.FastpiConfig(alpha=1.0))
    P = fp.materialize(res.pseudoinverse)
    assert np.abs(P @ A - np.eye(4)).max() < 1e-10
    # pinv(diag(2,0)) -> sigma_dagger (0.5, 0)
    pv = fp.pinv_from_svd(fp.SvdFactors(np.eye(2), np.array([2.0, 0.0]), np.eye(2), True))
    np.testing.assert_array_equal(pv.sigma_dagger, [0.5, 0.0])
    # random 400x100 at alpha=1: Moore-Penrose identities, sigma vs dense
    rng = np.random.default_rng(7)
    R = sp.random(400, 100, density=0.05, random_state=rng, format="csr")
    res = fp.fastpi(R, fp.FastpiConfig(alpha=1.0, seed=3))
    Ad = R.toarray()
    P = fp.materialize(res.pseudoinverse)
    nA = np.linalg.norm(Ad)
    assert np.linalg.norm(Ad @ P @ Ad - Ad) <= 1e-8 * nA
    assert np.linalg.norm(P @ Ad @ P - P) <= 1e-8 * np.linalg.norm(P)
    sd = np.linalg.svd(Ad, compute_uv=False)
    k = min(len(sd), res.factors.rank)
    assert np.abs(res.factors.sigma[:k] - sd[:k]).max() <= 1e-7 * sd[0]
    # wide input runs on the transpose: tested stage by stage in test_wide_input_transpose_branch
    # regression fit through the public API
    p = problem("c1")
    w = p.workload
    res = fp.fastpi(p.A, fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed))
    model = fp.fit(fp.MultiLabelDataset(p.A, p.Y), res.pseudoinverse)
    g1 = golden("c1")
    assert np.linalg.norm(model.coefficients - g1["Z"]) <= REC_TOL * np.linalg.norm(g1["Z"])
    # estimator front-end
    reg = fp.PseudoinverseRegressor(alpha=w.alpha, k=w.k, seed=w.seed).fit(p.A, p.Y)
    assert np.linalg.norm(reg.coef_ - g1["Z"]) <= REC_TOL * np.linalg.norm(g1["Z"])


def _lowrank_rel_factored(fa, fb):
    return lowrank_rel_factored(fa.U, fa.sigma, fa.Vt, fb.U, fb.sigma, fb.Vt)


@pytest.mark.parametrize("route", ["auto", "gram"])
def test_stagewise_parity_c4(route, monkeypatch):
    """P3 at the benchmark size (c4, 200k x 50k): oracle row / column updates fed the GPU's own
    upstream factors; the reorder sizes against the live oracle.  route=gram forces the column
    update's Z = H X route (gram_route.cu), which the cost model leaves off at c4."""
    if route == "gram":
        monkeypatch.setenv("FPI_GRAM_ROUTE", "1")
    p, res, st = _run("c4")
    w = p.workload
    Ac = orc.canonical_csr(p.A)
    o = orc.reorder(Ac.shape[0], Ac.shape[1], Ac.indptr, Ac.indices, w.k)
    assert (st["m1"], st["n1"], st["m2"], st["n2"], st["T"]) == (o.m1, o.n1, o.m2, o.n2, o.n_iterations)
    np.testing.assert_array_equal(res.reordering.row_perm.forward, o.row_fwd)
    part = st["part"]
    fo_rows, _ = orc.row_update(_host_factors(st["f11"]), part.a21.to_host(), st["s"], 0.3, w.seed + 1)
    fr = st["f_rows"]
    assert_sigma(fr.sigma, fo_rows.sigma, label="c4 row update")
    assert _lowrank_rel_factored(fr, fo_rows) <= REC_TOL
    fo_full, _ = orc.column_update(_host_factors(fr), part.T.to_host(), st["r"], 0.3, w.seed + 2)
    ff = res.factors
    assert_sigma(ff.sigma, fo_full.sigma, label="c4 column update")
    assert _lowrank_rel_factored(ff, fo_full) <= REC_TOL
    if route == "auto":
        # c4's T has a dense heavy-row x heavy-column core (Zipf x Zipf): the cost rule takes it
        from paper_2011_04235_b200 import _lib
        info = _lib.sparse_core_info()
        assert info["core_nnz"] > 0.3 * (info["core_nnz"] + info["rem_nnz"]), info


def test_apply_to_host_matches_device_apply():
    """Pseudoinverse.apply on a sparse operand (chunked lift with overlapped device->host copies)
    agrees with the device-resident apply."""
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    p = problem("c2")
    w = p.workload
    res = fp.fastpi(p.A, fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed))
    Zh = res.pseudoinverse.apply(p.Y)
    Zd = d2h(res.pseudoinverse.apply_device(DeviceCSR.from_host(p.Y)))
    assert Zh.shape == Zd.shape and Zh.dtype == np.float64
    np.testing.assert_allclose(Zh, Zd, rtol=0, atol=1e-13 * np.abs(Zd).max())


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_c_abi_fastpi_matches_python_pipeline(name):
    """fpi_fastpi (Algorithm 1 in one C call) runs the same stages as the stage-by-stage Python mirror:
    identical sigma, sigma+, factors and permutations -- through the handle-owned result
    (fpi_fastpi_get) and through the default fastpi() path (fpi_fastpi_ex + fpi_fastpi_take)."""
    import ctypes as C
    import torch
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import DeviceCSR, d2h
    from paper_2011_04235_b200.pinv import fastpi_device
    p = problem(name)
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    res = fastpi_device(DeviceCSR.from_host(p.A), cfg, stagewise=True)
    A = DeviceCSR.from_host(p.A, canonicalize=False)  # fpi_fastpi runs check_csr itself
    info = _lib.FastpiInfo()
    _lib.call("fpi_fastpi", A.shape[0], A.shape[1], A.nnz, _lib.ptr(A.indptr), _lib.ptr(A.indices),
              _lib.ptr(A.values), float(w.alpha), float(w.k), int(w.seed), float(cfg.low_rank_threshold),
              float(cfg.pinv_cutoff_factor), C.byref(info))
    ptrs = [C.c_void_p() for _ in range(6)]
    _lib.call("fpi_fastpi_get", *[C.byref(x) for x in ptrs])
    m, n, r = info.m, info.n, info.rank
    assert r == res.factors.rank
    assert (info.m1, info.n1, info.m2, info.n2, info.n_iterations, info.n_gcc) == (
        res.reordering.n_spoke_rows, res.reordering.n_spoke_cols, res.reordering.n_hub_rows,
        res.reordering.n_hub_cols, res.reordering.n_iterations, len(res.reordering.gcc_sizes))
    assert (info.edges_visited, info.nodes_visited) == (res.reordering.edges_visited, res.reordering.nodes_visited)

    from cuda.bindings import runtime as rt
    d = res.pseudoinverse._device()
    fd = res.factors.device()
    torch.cuda.synchronize()
    for ptr, ref in ((ptrs[1], fd.sigma), (ptrs[3], d.sdag), (ptrs[0], fd.U), (ptrs[2], fd.Vt),
                     (ptrs[4], d.row_fwd), (ptrs[5], d.col_fwd)):
        out = torch.empty(ref.numel(), dtype=ref.dtype, device="cuda")
        err, = rt.cudaMemcpy(out.data_ptr(), ptr.value, out.numel() * out.element_size(),
                             rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
        assert int(err) == 0
        np.testing.assert_array_equal(d2h(out), d2h(ref.reshape(-1)))
    _lib.call("fpi_fastpi_release")

    # default public path: one C call, buffers adopted by torch
    one = fp.fastpi(p.A, cfg)
    d1, f1 = one.pseudoinverse._device(), one.factors.device()
    for a, b in ((f1.sigma, fd.sigma), (d1.sdag, d.sdag), (f1.U, fd.U), (f1.Vt, fd.Vt), (d1.row_fwd, d.row_fwd),
                 (d1.col_fwd, d.col_fwd), (one.reordering.spans_device(), res.reordering.spans_device())):
        np.testing.assert_array_equal(d2h(a), d2h(b))
    assert one.reordering.gcc_sizes == res.reordering.gcc_sizes
    assert one.reordering.n_iterations == res.reordering.n_iterations
    assert one.pseudoinverse.tolerance_used == res.pseudoinverse.tolerance_used
    assert [(t.stage, t.rank) for t in one.timings] == [(t.stage, t.rank) for t in res.timings]
    assert all(t.seconds > 0 for t in one.timings)
    del one, d1, f1
    import gc
    gc.collect()
    torch.cuda.synchronize()  # the adopted buffers were returned through fpi_device_free


def test_wide_input_transpose_branch():
    """pinv.py:291-303: an m < n input is solved as fastpi(A^T) and the results are swapped.
    The SPEC wide example (60 x 150, alpha 0.5, k 0.05, seed 5; the generator sequence of
    oracle/pin_against_reference.py) is checked stage by stage against the oracle's own transposed
    run -- reorder of A^T bit-exact, block sigma per value, row / column updates fed the GPU's
    upstream factors -- and the swap itself: factors transposed, the pseudoinverse of A equal to
    the transpose of the pseudoinverse of A^T.  End to end the column update of this example takes
    the randomized engine, so its sigma depend on LAPACK's singular-vector signs; the
    golden end-to-end sigma are reported, not asserted."""
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200._device import DeviceCSR
    from paper_2011_04235_b200.pinv import fastpi_device
    rng = np.random.default_rng(7)
    sp.random(400, 100, density=0.05, random_state=rng, format="csr")
    R2 = sp.random(60, 150, density=0.08, random_state=rng, format="csr")
    alpha, k, seed = 0.5, 0.05, 5
    cfg = fp.FastpiConfig(alpha=alpha, k=k, seed=seed)
    res = fp.fastpi(R2, cfg)
    st = {}
    res_t = fastpi_device(DeviceCSR.from_host(R2).transpose(), cfg, stats=st)
    ref = orc.fastpi(R2, alpha, k, seed)
    assert ref["transposed"]
    # the swap (pinv.py:297-303)
    assert res.factors.shape == (60, 150) and res.pseudoinverse.shape == (150, 60)
    np.testing.assert_array_equal(res.factors.sigma, res_t.factors.sigma)
    np.testing.assert_array_equal(res.factors.U, res_t.factors.Vt.T)
    np.testing.assert_array_equal(res.factors.Vt, res_t.factors.U.T)
    P, Pt = fp.materialize(res.pseudoinverse), fp.materialize(res_t.pseudoinverse)
    # same factors; only the side diag(sigma+) is multiplied onto differs (rounding)
    np.testing.assert_allclose(P, Pt.T, rtol=0, atol=1e-13 * np.abs(P).max())
    # reorder of A^T: bit-exact against the oracle's transposed run
    o = ref["ordering"]
    np.testing.assert_array_equal(res_t.reordering.row_perm.forward, o.row_fwd)
    np.testing.assert_array_equal(res_t.reordering.col_perm.forward, o.col_fwd)
    np.testing.assert_array_equal(res_t.reordering.spans, o.spans)
    assert (st["m1"], st["n1"], st["m2"], st["n2"], st["T"]) == (o.m1, o.n1, o.m2, o.n2, o.n_iterations)
    assert (st["s"], st["r"]) == (ref["s"], ref["r"])
    # block stage (sign-free): per block, per value
    assert_block_sigma(st["f11"].sigma, ref["f11"].sigma, o.spans, alpha, label="wide f11")
    # updates fed the GPU's own upstream factors
    fo_rows, _ = orc.row_update(_host_factors(st["f11"]), ref["A21"], st["s"], 0.3, seed + 1)
    assert_sigma(st["f_rows"].sigma, fo_rows.sigma, label="wide row update")
    assert _lowrank_rel(st["f_rows"], fo_rows) <= REC_TOL
    fo_full, eng = orc.column_update(_host_factors(st["f_rows"]), ref["T"], st["r"], 0.3, seed + 2)
    assert_sigma(res.factors.sigma, fo_full.sigma, label="wide column update")
    assert _lowrank_rel(res_t.factors, fo_full) <= REC_TOL
    # pseudoinverse of A from the GPU-fed oracle factors, swapped back as pinv.py:297-301 does
    pv_t = orc.pinv_from_svd(orc.unfold(fo_full, o))
    P_o = (pv_t.Ut.T * pv_t.sigma_dagger) @ pv_t.V.T
    assert np.linalg.norm(P - P_o) <= REC_TOL * np.linalg.norm(P_o)
    g = golden("spec_examples")
    gap = np.abs(res.factors.sigma - g["spec_wide_sigma"]).max() / g["spec_wide_sigma"][0]
    print(f"wide example: end-to-end sigma gap vs the reference {gap:.3e} (column engine {eng})")


def test_block_sigma_c4_against_lapack():
    """P2 at the benchmark size: every non-degenerate c4 block (incl. the min-dim >= 48 blocks of the
    batched Gram path, block_svd.cu) against LAPACK dgesdd, per value (svd.py:154-178)."""
    p, res, st = _run("c4")
    part = st["part"]
    spans = res.reordering.spans
    fo = orc.block_svd(part.a11.to_host(), spans, p.workload.alpha)
    assert st["f11"].rank == fo.rank
    assert_block_sigma(st["f11"].sigma, fo.sigma, spans, p.workload.alpha, label="c4 f11")
    fo1 = orc.block_svd(part.a11.to_host(), spans, 1.0)
    from paper_2011_04235_b200.svd import block_diagonal_svd_device
    f1 = block_diagonal_svd_device(part.a11, res.reordering.spans_device(), 1.0)
    assert_block_sigma(f1.sigma, fo1.sigma, spans, 1.0, label="c4 f11 alpha=1")


def _result_arrays(res):
    from paper_2011_04235_b200._device import d2h
    d = res.pseudoinverse._device()
    fd = res.factors.device()
    return [d2h(x) for x in (fd.U, fd.sigma, fd.Vt, d.sdag, d.row_fwd, d.col_fwd)]


@pytest.mark.parametrize("name", ["c2", "c3r100"])
def test_deferred_values_upload_same_bits(name, monkeypatch):
    """fastpi(host CSR) hides the upload of A's values behind the reorder (fpi_fastpi_ex with
    FPI_FASTPI_DEFERRED_VALUES + fpi_fastpi_values_hook): the factors, sigma+, and permutations are
    bit-identical to the plain upload-then-solve path, and so is apply()."""
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200 import pinv as pinv_mod
    p = problem(name)
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    monkeypatch.setattr(pinv_mod, "_NO_DEFER", True)
    plain = fp.fastpi(p.A, cfg)
    ref = _result_arrays(plain)
    Zp = plain.pseudoinverse.apply(p.Y)
    monkeypatch.setattr(pinv_mod, "_NO_DEFER", False)
    monkeypatch.setattr(pinv_mod, "_DEFER_MIN_NNZ", 0)
    calls = []
    orig = pinv_mod._fastpi_host_overlapped
    monkeypatch.setattr(pinv_mod, "_fastpi_host_overlapped", lambda A, c: calls.append(1) or orig(A, c))
    for _ in range(3):  # repeated: the side-stream copy and the worker thread must not race the solve
        got = fp.fastpi(p.A, cfg)
        for a, b in zip(_result_arrays(got), ref):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(got.pseudoinverse.apply(p.Y), Zp)
    assert len(calls) == 3


@pytest.mark.parametrize("defect", ["unsorted", "duplicates", "explicit_zero"])
def test_deferred_values_upload_falls_back_on_non_canonical_input(defect, monkeypatch):
    """A CSR that check_csr (validation.py:38-55) would rewrite -- unsorted indices, duplicate entries
    or explicit zeros -- fails one half of the deferred path's canonical-form test (FPI_ERETRY) and
    takes the plain path: same bits as with the deferred upload disabled."""
    import scipy.sparse as sp
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200 import _lib, pinv as pinv_mod
    p = problem("c2")
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    A = p.A.copy()
    ip, ix, dv = A.indptr.copy(), A.indices.copy(), A.data.copy()
    r = int(np.argmax(np.diff(ip) >= 3))
    b = ip[r]
    if defect == "unsorted":
        ix[b], ix[b + 1] = ix[b + 1], ix[b]
        dv[b], dv[b + 1] = dv[b + 1], dv[b]
    elif defect == "duplicates":
        ix[b + 1] = ix[b]
    else:
        dv[b + 2] = 0.0
    B = sp.csr_matrix((dv, ix, ip), shape=A.shape)
    B.has_sorted_indices = True  # keep scipy from repairing it
    monkeypatch.setattr(pinv_mod, "_NO_DEFER", True)
    ref = _result_arrays(fp.fastpi(B, cfg))
    monkeypatch.setattr(pinv_mod, "_NO_DEFER", False)
    monkeypatch.setattr(pinv_mod, "_DEFER_MIN_NNZ", 0)
    seen = []
    orig = pinv_mod._fastpi_host_overlapped

    def spy(M, c):
        out = orig(M, c)
        seen.append(out[0] is None)
        return out
    monkeypatch.setattr(pinv_mod, "_fastpi_host_overlapped", spy)
    got = _result_arrays(fp.fastpi(B, cfg))
    assert seen == [True]
    for a, b_ in zip(got, ref):
        np.testing.assert_array_equal(a, b_)


def test_deferred_values_flag_needs_hook():
    """FPI_FASTPI_DEFERRED_VALUES without a registered hook (or without FPI_FASTPI_CANONICAL) is a
    domain error, not a solve on half-uploaded values."""
    import ctypes as C
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import DeviceCSR
    p = problem("c1")
    A = DeviceCSR.from_host(p.A)
    info = _lib.FastpiInfo()
    for flags in (_lib.FASTPI_DEFERRED_VALUES, _lib.FASTPI_DEFERRED_VALUES | _lib.FASTPI_CANONICAL):
        with pytest.raises(ValueError):
            _lib.call("fpi_fastpi_ex", A.shape[0], A.shape[1], A.nnz, _lib.ptr(A.indptr), _lib.ptr(A.indices),
                      _lib.ptr(A.values), 0.5, 0.01, 0, 0.3, 1.0, flags, C.byref(info))
