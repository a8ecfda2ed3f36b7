"""A/B of the bench step's surroundings: L2 flush before each step, nvidia-smi clock sampler."""
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
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
for _ in range(2):
    fastpi_device(A, cfg).pseudoinverse.apply_device(Y)
torch.cuda.synchronize()
for do_flush in (False, True):
    for sampler in (False, True):
        cs = bench.ClockSampler(0) if sampler else None
        if cs:
            cs.__enter__()
        ts, st = [], {}
        for i in range(5):
            if do_flush:
                flush.fill_(float(i))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = fastpi_device(A, cfg)
            res.pseudoinverse.apply_device(Y)
            torch.cuda.synchronize()
            ts.append(1e3 * (time.perf_counter() - t0))
            for s in res.timings:
                st.setdefault(s.stage, []).append(s.seconds * 1e3)
        if cs:
            cs.__exit__(None, None, None)
        print(f"flush={do_flush} sampler={sampler}: " + " ".join(f"{t:.1f}" for t in ts) + " | " +
              " ".join(f"{k}={sum(v) / len(v):.1f}" for k, v in st.items()), flush=True)
