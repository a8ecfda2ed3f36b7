"""Bit-equality of the deferred-values fastpi(host CSR) against the plain path at full size (c4, c5)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200 import pinv as pinv_mod  # noqa: E402

for name in sys.argv[1:] or ["c4"]:
    p = bench.load_problem(name)
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    outs = {}
    for defer in (False, True, True):
        pinv_mod._NO_DEFER = not defer
        res = fp.fastpi(p.A, cfg)
        d, fd = res.pseudoinverse._device(), res.factors.device()
        cur = [x.clone() for x in (fd.U, fd.sigma, fd.Vt, d.sdag, d.row_fwd, d.col_fwd)]
        torch.cuda.synchronize()
        if not defer:
            outs["plain"] = cur
        else:
            same = all(torch.equal(a, b) for a, b in zip(cur, outs["plain"]))
            print(f"{name}: deferred upload bit-identical to the plain path: {same} "
                  f"(U {tuple(cur[0].shape)}, Vt {tuple(cur[2].shape)})", flush=True)
            assert same
        del res
