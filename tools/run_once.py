"""Run one FastPI solve (+ apply) on a workload; the second call is wrapped in
cudaProfilerStart/Stop so `ncu --profile-from-start off` captures exactly one solve."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import torch
    import bench
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200._device import DeviceCSR
    from paper_2011_04235_b200.pinv import fastpi_device
    p = bench.load_problem(args.workload)
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    A = DeviceCSR.from_host(p.A)
    Y = DeviceCSR.from_host(p.Y)
    res = fastpi_device(A, cfg)
    res.pseudoinverse.apply_device(Y)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.reps):
        t0 = time.perf_counter()
        res = fastpi_device(A, cfg)
        Z = res.pseudoinverse.apply_device(Y)
        torch.cuda.synchronize()
        print(f"solve {time.perf_counter() - t0:.3f}s", [f"{s.stage}={s.seconds*1e3:.1f}" for s in res.timings],
              file=sys.stderr)
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
