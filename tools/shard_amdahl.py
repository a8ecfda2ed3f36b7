"""Stage-time Amdahl bound of the sharded solve (csrc/sharded.cu) from a world-of-one run.

    python tools/shard_amdahl.py [c4|c5] [steps]

Runs fastpi_sharded + apply_local with the world-of-one communicator and splits the step's kernel
time (instrumented, CUDA events per kernel class) into what every rank repeats at any world size
(reorder + partition, the 2r x 2r eigensolves and Cholesky factors, the sketch generation) and
what divides over the ranks (everything indexed by the rows of U / T / A21 / Y or by the columns of
Vt / Z).  Prints one JSON line: per-class ms, replicated ms, the N-GPU time bound
T_rep + (T_1 - T_rep) / N and T_1 / that for N = 2, 4, 8 (exchange time not included; the
exchanged volumes are printed beside it)."""
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2011_04235_b200 import FastpiConfig, _lib  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402
from paper_2011_04235_b200.sharded import Comm, fastpi_sharded  # noqa: E402

REPLICATED = ("reorder_loop", "permute_partition", "sym_eig", "cholesky", "sketch", "inner_gram_route")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    torch.cuda.set_device(0)
    p = bench.load_problem(name)
    w = p.workload
    cfg = FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    A, Y = DeviceCSR.from_host(p.A), DeviceCSR.from_host(p.Y)
    comm = Comm()
    st = {}
    for _ in range(2):
        res = fastpi_sharded(A, cfg, comm, stats=st)
        res.pseudoinverse.apply_local(Y)
    torch.cuda.synchronize()
    times = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = fastpi_sharded(A, cfg, comm, stats=st)
        res.pseudoinverse.apply_local(Y)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    _lib.timing_enable(True)
    res = fastpi_sharded(A, cfg, comm, stats=st)
    res.pseudoinverse.apply_local(Y)
    torch.cuda.synchronize()
    rep = _lib.timing_report(reset=True)
    _lib.timing_enable(False)
    t1 = statistics.mean(times)
    ktot = sum(v["ms"] for v in rep.values())
    rep_ms = sum(v["ms"] for k, v in rep.items() if k.startswith(REPLICATED))
    other = t1 - ktot  # host gaps and untimed kernels, counted as replicated (conservative)
    t_rep = rep_ms + max(other, 0.0)
    s, r, n1, n2, L = st["s"], st["r"], st["n1"], st["n2"], p.Y.shape[1]
    out = {"workload": name, "sharded": st.get("sharded"), "t1_ms": round(t1, 2),
           "kernel_ms": {k: round(v["ms"], 2) for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])},
           "replicated_ms": round(t_rep, 2),
           "bound": {N: {"ms": round(t_rep + (t1 - t_rep) / N, 2), "speedup": round(t1 / (t_rep + (t1 - t_rep) / N), 2)}
                     for N in (2, 4, 8)},
           "exchange_bytes": {"row_grams": 2 * 8 * (2 * s) ** 2, "row_reduce_scatter": 8 * n1 * 2 * s,
                              "col_allreduce_MtB": 8 * (s + n2) * 2 * r, "col_grams": 2 * 8 * (2 * r) ** 2,
                              "apply_allreduce_W": 8 * L * r},
           "stages_ms": {t.stage: round(t.seconds * 1e3, 2) for t in res.timings}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
