"""Break the public-API end-to-end solve into host<->device and compute pieces."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR, d2h  # noqa: E402
from paper_2011_04235_b200.pinv import fastpi_device  # noqa: E402

p = bench.load_problem(sys.argv[1] if len(sys.argv) > 1 else "c4")
w = p.workload
cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    t0 = t()
    A = DeviceCSR.from_host(p.A)
    t1 = t()
    res = fastpi_device(A, cfg)
    t2 = t()
    Y = DeviceCSR.from_host(p.Y)
    t3 = t()
    Z = res.pseudoinverse.apply_device(Y)
    t4 = t()
    Zh = d2h(Z)
    t5 = t()
    t6 = t()
    res2 = fp.fastpi(p.A, cfg)
    Zh2 = res2.pseudoinverse.apply(p.Y)
    t7 = t()
    print(f"upload A {1e3*(t1-t0):.1f}  fastpi {1e3*(t2-t1):.1f}  upload Y {1e3*(t3-t2):.1f}  apply {1e3*(t4-t3):.1f}  "
          f"d2h Z {1e3*(t5-t4):.1f} ({Zh.nbytes/1e9:.2f} GB)  | public API total {1e3*(t7-t6):.1f} ms", flush=True)
    del res, res2, Z, Zh, Zh2
