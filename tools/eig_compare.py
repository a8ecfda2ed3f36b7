"""Time the block-Jacobi eigensolver against torch.linalg.eigh (cuSOLVER) on captured Gram matrices."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import d2h, empty, h2d
    for f in sys.argv[1:]:
        G = np.load(f)
        n = G.shape[0]
        dG = h2d(G)
        w = empty(n)
        V = empty((n, n))
        sw = C.c_int32(0)
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.call("fpi_sym_eig", n, _lib.ptr(dG), n, _lib.ptr(w), _lib.ptr(V), n, C.byref(sw))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"{f} n={n} jacobi sweeps={sw.value} {dt * 1e3:.2f} ms", flush=True)
        tG = torch.from_numpy(G).cuda()
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ev, evec = torch.linalg.eigh(tG)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"{f} n={n} torch.linalg.eigh {dt * 1e3:.2f} ms", flush=True)
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ev = torch.linalg.eigvalsh(tG)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"{f} n={n} torch.linalg.eigvalsh {dt * 1e3:.2f} ms", flush=True)
        wr = np.linalg.eigvalsh(G)[::-1]
        print("jacobi eig err", np.abs(d2h(w) - wr).max() / wr[0], "eigh err",
              np.abs(ev.cpu().numpy()[::-1] - wr).max() / wr[0])


if __name__ == "__main__":
    main()
