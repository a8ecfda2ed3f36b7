"""CSR x dense-panel throughput (fpi_spmm) on c4-shaped operands, against cuSPARSE (torch.sparse.mm).

Operands: the c4 feature matrix A (200,000 x 50,000, Zipf columns) restricted to its 10,130
highest-degree columns -- the shape of the column-update block [A12; A22] -- with k = 1000
(= 2 r) columns, both as M X and as M^T B (long rows: the segmented path), plus the whole A
with k = 500.  Reports ms, gathered GB/s (nnz * k * 8 / t) and the max relative error."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_04235_b200 import _lib  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def case(name, Mh, k, odd_ld=False):
    M = DeviceCSR.from_host(Mh)
    p, q = Mh.shape
    ldx = k + 1 if odd_ld else k
    Xfull = torch.randn((q, ldx), dtype=torch.float64, device="cuda")
    Y = torch.empty((p, k), dtype=torch.float64, device="cuda")

    def run():
        _lib.call("fpi_spmm", p, q, k, _lib.ptr(M.indptr), _lib.ptr(M.indices), _lib.ptr(M.values), 1.0,
                  _lib.ptr(Xfull), ldx, 0.0, _lib.ptr(Y), k)

    ms = timed(run)
    X = Xfull[:, :k]
    ts = torch.sparse_csr_tensor(M.indptr, M.indices.long(), M.values, size=(p, q))
    ref = torch.sparse.mm(ts, X.contiguous())
    err = ((Y - ref).abs().max() / ref.abs().max()).item()
    ms_ref = timed(lambda: torch.sparse.mm(ts, X.contiguous()))
    nnz = Mh.nnz
    lens = np.diff(Mh.indptr)
    print(f"{name:22s} p={p} q={q} k={k} nnz={nnz} maxrow={lens.max()} rows>512={int((lens > 512).sum())}: "
          f"{ms:.3f} ms  {nnz * k * 8 / ms / 1e6:.0f} GB/s gathered  relerr {err:.1e}  "
          f"(cuSPARSE {ms_ref:.3f} ms)", flush=True)


def main():
    only = sys.argv[1:]
    A = bench.load_problem("c4").A.tocsc()
    deg = np.diff(A.indptr)
    hub = np.sort(np.argsort(-deg, kind="stable")[:10130])
    M = A[:, hub].tocsr()
    cases = [("colblock_MX_k1000", M, 1000, False), ("colblock_MtB_k1000", M.T.tocsr(), 1000, False),
             ("A_X_k500", A.tocsr(), 500, False), ("At_B_k500", A.T.tocsr(), 500, False),
             ("colblock_MX_k999_odd", M, 999, True)]
    for name, Mh, k, odd in cases:
        if only and name not in only:
            continue
        case(name, Mh, k, odd)


if __name__ == "__main__":
    main()
