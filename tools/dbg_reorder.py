import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from conftest import golden, problem
import paper_2011_04235_b200 as fp
from paper_2011_04235_b200._device import DeviceCSR, d2h
from paper_2011_04235_b200.reorder import reorder_device
for name in ["c1"]:
    g = golden(name); p = problem(name)
    r = reorder_device(DeviceCSR.from_host(p.A), p.workload.k)
    rf = r.row_perm.forward; cf = r.col_perm.forward
    print(name, "sizes", [r.n_spoke_rows, r.n_spoke_cols, r.n_hub_rows, r.n_hub_cols, r.n_iterations], "golden", g["sizes"].tolist())
    print("gcc", list(r.gcc_sizes[:8]), list(g["gcc_sizes"][:8]))
    dr = np.nonzero(rf != g["row_fwd"])[0]; dc = np.nonzero(cf != g["col_fwd"])[0]
    print("row mismatches", len(dr), dr[:10], rf[dr[:10]], g["row_fwd"][dr[:10]])
    print("col mismatches", len(dc), dc[:10], cf[dc[:10]], g["col_fwd"][dc[:10]])
    print("spans", len(r.spans), len(g["spans"]), (r.spans[:5]).tolist(), g["spans"][:5].tolist())
