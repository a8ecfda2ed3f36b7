"""Time fpi_orth_factor (Cholesky + inverse) on a c4-like Gram; FPI_CHOL_PROFILE=1 prints the task timeline."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

if __name__ == "__main__":
    import torch
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import empty, h2d
    for n in [int(x) for x in (sys.argv[1:] or ["798", "1000"])]:
        rng = np.random.default_rng(n)
        B = rng.standard_normal((4 * n, n))
        dG = h2d(B.T @ B)
        Li = empty((n, n))
        cond = C.c_double(0.0)
        for rep in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.call("fpi_orth_factor", n, _lib.ptr(dG), _lib.ptr(Li), C.byref(cond))
            torch.cuda.synchronize()
            print(f"n={n} rep {rep}: {1e3 * (time.perf_counter() - t0):.3f} ms", flush=True)
