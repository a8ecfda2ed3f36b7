"""A/B of the deferred values upload (pinv._fastpi_host_overlapped): fastpi(host CSR) wall time with the
upload hidden behind the reorder vs. upload-then-solve, interleaved."""
import statistics
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200 import pinv as pinv_mod  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
p = bench.load_problem(name)
w = p.workload
cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
times = {True: [], False: [], "upload": [], "solve": [], "e2e deferred": [], "e2e plain": [],
         "apply after deferred": [], "apply after plain": []}
for i in range(3 + reps):
    for defer in (False, True):
        pinv_mod._NO_DEFER = not defer
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fp.fastpi(p.A, cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if i >= 3:
            times[defer].append(dt)
        del res
    for defer in (False, True):  # the bench's e2e step: fastpi + apply -> numpy Z, no sync between
        pinv_mod._NO_DEFER = not defer
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fp.fastpi(p.A, cfg)
        t1 = time.perf_counter()
        Z = res.pseudoinverse.apply(p.Y)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        if i >= 3:
            times["e2e deferred" if defer else "e2e plain"].append(t2 - t0)
            times["apply after deferred" if defer else "apply after plain"].append(t2 - t1)
        del res, Z
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A = DeviceCSR.from_host(p.A)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = pinv_mod.fastpi_device(A, cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if i >= 3:
        times["upload"].append(t1 - t0)
        times["solve"].append(t2 - t1)
    del res, A
for k, v in times.items():
    print(f"{name} {k}: mean {1e3 * statistics.mean(v):.2f} ms  median {1e3 * statistics.median(v):.2f}  min {1e3 * min(v):.2f}")
