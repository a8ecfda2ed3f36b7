"""Time the block-Jacobi eigensolver on Gram matrices like the randomized SVD's."""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import d2h, empty, h2d
    rng = np.random.default_rng(0)
    for n in [int(x) for x in (sys.argv[1:] or ["800", "1000"])]:
        Y = rng.standard_normal((n, 4 * n)) * np.logspace(0, -2, n)[:, None]
        G = Y @ Y.T
        dG = h2d(G)
        w = empty(n)
        V = empty((n, n))
        sw = C.c_int32(0)
        for mixed in ("0", "1"):
          os.environ["FPI_JACOBI_MIXED"] = mixed
          for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.call("fpi_sym_eig", n, _lib.ptr(dG), n, _lib.ptr(w), _lib.ptr(V), n, C.byref(sw))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
          wr = np.linalg.eigvalsh(G)[::-1]
          err = np.abs(d2h(w) - wr).max() / wr[0]
          Vh = d2h(V)
          orth = np.abs(Vh.T @ Vh - np.eye(n)).max()
          res = np.abs(G @ Vh - Vh * d2h(w)).max() / wr[0]
          print(f"n={n} mixed={mixed} sweeps={sw.value} {dt*1e3:.2f} ms "
                f"eig err {err:.2e} orth {orth:.2e} resid {res:.2e}", flush=True)


if __name__ == "__main__":
    main()
