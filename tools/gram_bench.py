import sys, os
sys.path.insert(0, '/root/repo')
import torch
from paper_2011_04235_b200 import _lib
for name, n, k in [("HH", 256, 2000000), ("H11", 940, 349000), ("GramB_row", 1878, 133722), ("GramZ_row", 1878, 187726)]:
    A = torch.randn((k, n), dtype=torch.float64, device="cuda")
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    args = (1, n, k, _lib.ptr(A), n, _lib.ptr(C), n)
    _lib.call("fpi_gram", *args); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): _lib.call("fpi_gram", *args)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{name} n={n} k={k} sym: {ms:.3f} ms {n*n*k/ms/1e9:.2f} TFLOP/s", flush=True)
    del A, C
