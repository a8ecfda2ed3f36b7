"""One eigensolve of an n x n Gram matrix (for ncu)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2011_04235_b200 import _lib  # noqa: E402
from paper_2011_04235_b200._device import empty, h2d  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
rng = np.random.default_rng(0)
Y = rng.standard_normal((n, 4 * n)) * np.logspace(0, -2, n)[:, None]
G = h2d(Y @ Y.T)
w, V = empty(n), empty((n, n))
sw = C.c_int32(0)
_lib.call("fpi_sym_eig", n, _lib.ptr(G), n, _lib.ptr(w), _lib.ptr(V), n, C.byref(sw))
torch.cuda.synchronize()
print("sweeps", sw.value)
