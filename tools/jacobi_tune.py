"""Time the c4 (or --workload=c5) solve under eigensolver environment settings (one process; env read per call).

usage: python tools/jacobi_tune.py "FPI_JACOBI_JOIN=1" "FPI_JACOBI_CHUNKS=4,3 FPI_JACOBI_SPREAD=4" ...
An empty string is the default configuration."""
import os
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402
from paper_2011_04235_b200.pinv import fastpi_device  # noqa: E402

WORKLOAD = "c4"
if len(sys.argv) > 1 and sys.argv[1].startswith("--workload="):
    WORKLOAD = sys.argv.pop(1).split("=", 1)[1]
p = bench.load_problem(WORKLOAD)
w = p.workload
cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
A = DeviceCSR.from_host(p.A)
Y = DeviceCSR.from_host(p.Y)
for _ in range(2):
    fastpi_device(A, cfg).pseudoinverse.apply_device(Y)
torch.cuda.synchronize()
keys = ("FPI_JACOBI_PREFETCH", "FPI_JACOBI_JOIN", "FPI_JACOBI_CHUNKS", "FPI_JACOBI_SPREAD", "FPI_JACOBI_GRID")
for rep in range(2):
    for spec in sys.argv[1:] or [""]:
        for k in keys:
            os.environ.pop(k, None)
        for kv in spec.split():
            k, v = kv.split("=", 1)
            os.environ[k] = v
        ts, st = [], {}
        for i in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fastpi_device(A, cfg)
            res.pseudoinverse.apply_device(Y)
            torch.cuda.synchronize()
            ts.append(1e3 * (time.perf_counter() - t0))
            for s in res.timings:
                st.setdefault(s.stage, []).append(s.seconds * 1e3)
        print(f"[{spec or 'default'}] median {statistics.median(ts):.2f} ms | row_update="
              f"{statistics.median(st['row_update']):.2f} column_update={statistics.median(st['column_update']):.2f}",
              flush=True)
