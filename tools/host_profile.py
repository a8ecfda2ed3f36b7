"""Host-side (Python + ctypes) time of one c4 solve + apply, by function (cProfile): the part of
the step where the GPU may sit idle waiting for the next submission.

    python tools/host_profile.py [c4]
"""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402
from paper_2011_04235_b200.pinv import fastpi_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    torch.cuda.set_device(0)
    p = bench.load_problem(name)
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    A, Y = DeviceCSR.from_host(p.A), DeviceCSR.from_host(p.Y)
    for _ in range(3):
        fastpi_device(A, cfg).pseudoinverse.apply_device(Y)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    res = fastpi_device(A, cfg)
    res.pseudoinverse.apply_device(Y)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
