"""Where the end-to-end apply(Y) -> numpy Z goes: Y upload, pinned allocation, the chunked lift + D2H
(fpi_pinv_apply_csr_host), against the raw D2H bandwidth of the same bytes."""
import statistics
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200 import _lib  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
p = bench.load_problem(name)
w = p.workload
cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
res = fp.fastpi(p.A, cfg)
pv = res.pseudoinverse
d = pv._device()
L = p.Y.shape[1]
T = {k: [] for k in ("upload Y", "pinned alloc", "lift + D2H call", "apply total", "raw D2H one copy",
                     "raw D2H 64MB chunks", "lift only (device)")}


def now():
    torch.cuda.synchronize()
    return time.perf_counter()


Zd = torch.empty((d.n, L), dtype=torch.float64, device="cuda")
for i in range(2 + reps):
    t0 = now()
    Yd = DeviceCSR.from_host(p.Y)
    t1 = now()
    Zh = torch.empty((d.n, L), dtype=torch.float64, pin_memory=True)
    t2 = now()
    _lib.call("fpi_pinv_apply_csr_host", d.m, d.n, d.r, _lib.ptr(d.U), _lib.ptr(d.sdag), _lib.ptr(d.Vt),
              _lib.ptr(d.row_fwd), _lib.ptr(d.col_fwd), L, Yd.nnz, _lib.ptr(Yd.indptr), _lib.ptr(Yd.indices),
              _lib.ptr(Yd.values), Zh.data_ptr())
    t3 = now()
    Z2 = pv.apply(p.Y)
    t4 = now()
    Zh.copy_(Zd, non_blocking=True)
    t5 = now()
    rows = max(256, (64 << 20) // (8 * L))
    for a in range(0, d.n, rows):
        Zh[a:a + rows].copy_(Zd[a:a + rows], non_blocking=True)
    t6 = now()
    Zdev = pv.apply_device(Yd)
    t7 = now()
    if i >= 2:
        for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6)):
            T[k].append(v)
    del Zh, Z2, Zdev, Yd
gb = d.n * L * 8 / 1e9
for k, v in T.items():
    extra = f"  ({gb / statistics.median(v):.1f} GB/s)" if "D2H" in k else ""
    print(f"{name} {k}: median {1e3 * statistics.median(v):.2f} ms  min {1e3 * min(v):.2f}  max {1e3 * max(v):.2f}{extra}")
