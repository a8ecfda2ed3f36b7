"""Pin the oracle against the unmodified reference and write golden fixtures.

TEST INFRASTRUCTURE.  Runs only in the build container, where the reference
is importable from ``/root/reference/pkg/src`` (read-only, never copied).

1. For each small workload (c1, c2, c3r50/100/200) and the SPEC.md examples,
   run the reference ``fastpi.fastpi`` and the oracle, and require every
   stage to agree bit-for-bit: permutations, spans, iteration count, GCC
   sizes, block sigma, U11/Vt11, row/column-update factors, the
   pseudoinverse and Z = pinv @ Y.
2. Write ``tests/golden/<name>.npz`` with the reference's outputs (the
   fixtures travel to the GPU box; the reference does not).

Usage:  python oracle/pin_against_reference.py [names...]
"""

from __future__ import annotations

import hashlib
import json
import sys
import warnings
from pathlib import Path

import numpy as np
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = Path("/root/reference/pkg/src")

from oracle import fastpi_oracle as orc  # noqa: E402
from paper_2011_04235_b200 import workloads  # noqa: E402


def _ref():
    if not REF.exists():
        raise SystemExit("reference not present; pinning runs only in the build container")
    sys.path.insert(0, str(REF))
    import fastpi  # noqa: F401
    return fastpi


def csr_hash(A) -> str:
    A = sp.csr_matrix(A)
    h = hashlib.sha256()
    for arr in (np.asarray(A.indptr, np.int64), np.asarray(A.indices, np.int64), np.asarray(A.data, np.float64)):
        h.update(arr.tobytes())
    h.update(np.asarray(A.shape, np.int64).tobytes())
    return h.hexdigest()


def _same(a, b, what):
    a = np.asarray(a.todense() if sp.issparse(a) else a)
    b = np.asarray(b.todense() if sp.issparse(b) else b)
    if a.shape != b.shape or not np.array_equal(a, b):
        diff = np.abs(a - b).max() if a.shape == b.shape else "shape"
        raise AssertionError(f"oracle != reference at {what}: {diff}")


def pin_one(fastpi, A, Y, alpha, k, seed):
    cfg = fastpi.FastpiConfig(alpha=alpha, k=k, seed=seed)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ref = fastpi.fastpi(A, cfg)
        ours = orc.fastpi(A, alpha, k, seed)
    ro, oo = ref.reordering, ours["ordering"]
    if not ours["transposed"]:
        _same(ro.row_perm.forward, oo.row_fwd, "row_perm")
        _same(ro.col_perm.forward, oo.col_fwd, "col_perm")
        _same(np.asarray([tuple(b) for b in ro.blocks], np.int64).reshape(-1, 4), oo.spans, "spans")
        assert (ro.n_spoke_rows, ro.n_spoke_cols, ro.n_hub_rows, ro.n_hub_cols, ro.n_iterations) == \
            (oo.m1, oo.n1, oo.m2, oo.n2, oo.n_iterations), "sizes"
        assert tuple(ro.gcc_sizes) == tuple(oo.gcc_sizes), "gcc sizes"
    _same(ref.factors.U, ours["factors"].U, "factors.U")
    _same(ref.factors.sigma, ours["factors"].sigma, "factors.sigma")
    _same(ref.factors.Vt, ours["factors"].Vt, "factors.Vt")
    pv, po = ref.pseudoinverse, ours["pinv"]
    _same(pv.V, po.V, "pinv.V")
    _same(pv.Ut, po.Ut, "pinv.Ut")
    _same(pv.sigma_dagger, po.sigma_dagger, "sigma_dagger")
    assert pv.tolerance_used == po.tolerance_used
    Zr = None
    if Y is not None:
        Zr = pv.apply(Y)
        _same(Zr, orc.apply_pinv(po, Y), "Z")
    return ref, ours, Zr


def stage_checks(fastpi, ours, alpha, seed):
    """Stage-level agreement: block SVD, row update, column update called directly."""
    from fastpi import reorder as R, svd as S, pinv as P
    o = ours["ordering"]
    blocks = [ours["spoke"][rs:rs + h, cs:cs + w].tocsr() for rs, h, cs, w in o.spans]
    f11r = S.block_diagonal_svd(blocks, alpha)
    _same(f11r.sigma, ours["f11"].sigma, "f11.sigma")
    _same(f11r.U, ours["f11"].U, "f11.U")
    _same(f11r.Vt, ours["f11"].Vt, "f11.Vt")
    fr = P.row_update(f11r, ours["A21"], ours["s"], seed=seed + 1)
    _same(fr.sigma, ours["f_rows"].sigma, "f_rows.sigma")
    _same(fr.U, ours["f_rows"].U, "f_rows.U")


def spec_examples(fastpi):
    """SPEC.md examples the code honours."""
    out = {}
    # two diagonal blocks -> sigma (3,1,2,1) unsorted
    blocks = [sp.csr_matrix(np.diag([3.0, 1.0])), sp.csr_matrix(np.diag([2.0, 1.0]))]
    f = fastpi.block_diagonal_svd(blocks, 1.0)
    spoke = sp.block_diag(blocks).tocsr()
    fo = orc.block_svd(spoke, np.array([[0, 2, 0, 2], [2, 2, 2, 2]]), 1.0)
    _same(f.sigma, fo.sigma, "spec two blocks")
    out["spec_two_blocks_sigma"] = f.sigma
    # pinv(diag(2,0)) -> sigma_dagger (0.5, 0)
    fd = fastpi.SvdFactors(np.eye(2), np.array([2.0, 0.0]), np.eye(2), True)
    pv = fastpi.pinv_from_svd(fd)
    _same(pv.sigma_dagger, orc.pinv_from_svd(orc.Factors(np.eye(2), np.array([2.0, 0.0]), np.eye(2), True)).sigma_dagger, "spec diag(2,0)")
    out["spec_diag20_sigma_dagger"] = pv.sigma_dagger
    # diag(5,4,3,2) padded to 8x4, alpha=1 -> A+A = I
    A = np.zeros((8, 4))
    A[:4, :4] = np.diag([5.0, 4.0, 3.0, 2.0])
    ref, ours, _ = pin_one(fastpi, sp.csr_matrix(A), None, 1.0, 0.01, 0)
    out["spec_diag_padded_sigma"] = ref.factors.sigma
    # 4 disjoint 2x2 components, k=0.1: the code gives T=3
    B = sp.block_diag([sp.csr_matrix(np.ones((2, 2)))] * 4).tocsr()
    g = fastpi.to_bipartite(B)
    r = fastpi.reorder(g, 0.1)
    o = orc.reorder(8, 8, B.indptr, B.indices, 0.1)
    _same(r.row_perm.forward, o.row_fwd, "spec shattered rows")
    _same(r.col_perm.forward, o.col_fwd, "spec shattered cols")
    assert r.n_iterations == o.n_iterations
    out["spec_shattered_T"] = np.array([r.n_iterations])
    out["spec_shattered_row_fwd"] = r.row_perm.forward
    out["spec_shattered_col_fwd"] = r.col_perm.forward
    # random 400x100 at alpha=1, wide 60x150 (transpose branch)
    rng = np.random.default_rng(7)
    R1 = sp.random(400, 100, density=0.05, random_state=rng, format="csr")
    ref, ours, _ = pin_one(fastpi, R1, None, 1.0, 0.01, 3)
    out["spec_rand400_sigma"] = ref.factors.sigma
    R2 = sp.random(60, 150, density=0.08, random_state=rng, format="csr")
    ref, ours, _ = pin_one(fastpi, R2, None, 0.5, 0.05, 5)
    out["spec_wide_sigma"] = ref.factors.sigma
    return out


def sketch_vectors(names):
    """Hashes + leading values of every (seed, shape) Gaussian sketch the configs use."""
    rows = []
    for seed, r, c in names:
        X = np.random.default_rng(seed).standard_normal((r, c))
        rows.append({"seed": seed, "rows": r, "cols": c,
                     "sha256": hashlib.sha256(X.tobytes()).hexdigest(),
                     "head": X.ravel()[:8].tolist(), "sum": float(X.sum())})
    return rows


def main(names):
    fastpi = _ref()
    gold = ROOT / "tests" / "golden"
    gold.mkdir(parents=True, exist_ok=True)
    sketches = []
    for name in names:
        prob = workloads.make_problem(name)
        w = prob.workload
        ref, ours, Z = pin_one(fastpi, prob.A, prob.Y, w.alpha, w.k, w.seed)
        stage_checks(fastpi, ours, w.alpha, w.seed)
        ro = ref.reordering
        f = ref.factors
        recon = orc.reconstruction_error(ours["A_perm"], ours["factors"])
        s, r = ours["s"], ours["r"]
        n1, n2 = ro.n_spoke_cols, ro.n_hub_cols
        sketches += [(w.seed + 1, n1, 2 * s), (w.seed + 2, ours["f_rows"].rank + n2, 2 * r)]
        payload = dict(
            A_sha256=np.array(csr_hash(prob.A)), Y_sha256=np.array(csr_hash(prob.Y)),
            row_fwd=ro.row_perm.forward, col_fwd=ro.col_perm.forward,
            spans=np.asarray([tuple(b) for b in ro.blocks], np.int64).reshape(-1, 4),
            sizes=np.array([ro.n_spoke_rows, ro.n_spoke_cols, ro.n_hub_rows, ro.n_hub_cols, ro.n_iterations]),
            gcc_sizes=np.asarray(ro.gcc_sizes, np.int64),
            f11_sigma=ours["f11"].sigma, f_rows_sigma=ours["f_rows"].sigma,
            sigma=f.sigma, s_r=np.array([s, r]), engines=np.array(list(ours["engines"])),
            recon=np.array([recon]), tol=np.array([ref.pseudoinverse.tolerance_used]),
            sigma_dagger=ref.pseudoinverse.sigma_dagger,
            Z_fro=np.array([np.linalg.norm(Z)]),
        )
        if Z.size <= 400_000:
            payload["Z"] = Z
        else:
            sel = np.random.default_rng(0).choice(Z.shape[0], 64, replace=False)
            payload["Z_rows_idx"] = np.sort(sel)
            payload["Z_rows"] = Z[np.sort(sel)]
        np.savez_compressed(gold / f"{name}.npz", **payload)
        print(f"pinned {name}: T={ro.n_iterations} m1={ro.n_spoke_rows} n1={n1} m2={ro.n_hub_rows} n2={n2} "
              f"s={s} r={r} engines={ours['engines']} recon={recon:.6g}")
    spec = spec_examples(fastpi)
    np.savez_compressed(gold / "spec_examples.npz", **spec)
    print("pinned SPEC examples")
    (gold / "sketches.json").write_text(json.dumps(sketch_vectors(sketches), indent=1))
    print("wrote sketch vectors")


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3r50", "c3r100", "c3r200"])
