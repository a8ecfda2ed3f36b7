"""Per-iteration wall-clock trace of the device reorder on a workload (FPI_TRACE_REORDER=0 prints
every iteration with its host sync wait)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    import torch
    import bench
    from paper_2011_04235_b200._device import DeviceCSR
    from paper_2011_04235_b200.reorder import reorder_device
    p = bench.load_problem(name)
    A = DeviceCSR.from_host(p.A)
    for i in range(reps):
        if i == reps - 1:
            os.environ["FPI_REORDER_PROFILE"] = "1"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = reorder_device(A, p.workload.k)
        torch.cuda.synchronize()
        print(f"rep {i}: {1e3 * (time.perf_counter() - t0):.2f} ms, T={r.n_iterations}", flush=True)
