"""Per-step wall times of fastpi + apply over many steps (outlier hunting)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402
from paper_2011_04235_b200.pinv import fastpi_device  # noqa: E402

p = bench.load_problem("c4")
w = p.workload
cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
A = DeviceCSR.from_host(p.A)
Y = DeviceCSR.from_host(p.Y)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for i in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fastpi_device(A, cfg)
    t1 = time.perf_counter()
    res.pseudoinverse.apply_device(Y)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = " ".join(f"{s.stage[:6]}={s.seconds * 1e3:.1f}" for s in res.timings)
    print(f"step {i}: total {1e3 * (t2 - t0):.1f} ms  fastpi {1e3 * (t1 - t0):.1f}  apply {1e3 * (t2 - t1):.1f} | {st}",
          flush=True)
