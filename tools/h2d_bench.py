"""Host->device upload variants for the CSR arrays of c4 (pin-copy, pageable, cudaHostRegister)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402

p = bench.load_problem("c4")
arrs = [p.A.indptr.astype(np.int64), p.A.indices.astype(np.int32), p.A.data.astype(np.float64)]
torch.zeros(1, device="cuda")


def t(f, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


def pin_copy():
    return [torch.from_numpy(a).pin_memory().to("cuda", non_blocking=True) for a in arrs]


def pageable():
    return [torch.from_numpy(a).to("cuda") for a in arrs]


def registered():
    cr = torch.cuda.cudart()
    outs = []
    for a in arrs:
        cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        outs.append(torch.from_numpy(a).to("cuda", non_blocking=True))
    torch.cuda.synchronize()
    for a in arrs:
        cr.cudaHostUnregister(a.ctypes.data)
    return outs


print(f"bytes {sum(a.nbytes for a in arrs) / 1e6:.1f} MB")
for name, f in (("pin_copy", pin_copy), ("pageable", pageable), ("registered", registered)):
    print(f"{name:12s} {t(f):.2f} ms", flush=True)
