#!/usr/bin/env python
"""FastPI pinv + regression solve on B200 -- the driver's benchmark contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c4]

A step is one full FastPI solve on one synthetic problem: reorder + permute /
partition + block SVD + row update + column update + pseudoinverse assembly
(``fastpi``, reference pinv.py:278-347) followed by the regression solve
Z = pinv @ Y (``Pseudoinverse.apply`` / ``fit``, pinv.py:72-81,
regression.py:50-70).  The metric is seconds per solve (lower is better).

* ``value``  -- device-resident inputs, CUDA events around each step, L2 flushed
  (512 MB write) before every timed step, mean over K steps, max over ranks.
* ``e2e``    -- the public API on host scipy inputs: fastpi(A) + apply(Y) -> numpy
  Z, host->device copies of A and Y and the device->host copy of Z inside.
* ``roofline`` -- the dominant kernel class of the step, timed live with CUDA
  events on the library stream (a separate instrumented pass after the timed
  region), algorithmic flops / bytes per SURVEY.md section 8(d).
* ``cpu_baseline`` -- the oracle port (numpy/scipy restatement of the reference,
  bit-identical to it on this image) timed on the host cores, rank 0, N=1.
* ``--impl reference`` -- the reference's CPU path (the oracle port; the
  Python reference itself cannot travel to the GPU box) on the same workload.

Multi-GPU (torchrun, or `--gpus N` which spawns the ranks itself; one rank per
GPU, NCCL inside the library): the same problem is solved by all ranks together
(strong scaling) -- A11 blocks, U rows and Vt / Z columns owned per rank, NCCL
reductions of the small Grams and projections (csrc/sharded.cu, SURVEY.md
section 8(e)); the reorder and the 2r x 2r eigensolves are replicated.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FastPI pinv+solve sec & FP64 TFLOP/s|HBM GB/s frac at 1/2/4/8 B200 vs CPU ref"
CACHE = Path(os.environ.get("FASTPI_BENCH_CACHE", "/tmp/fastpi_b200_cache"))


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_problem(name):
    from paper_2011_04235_b200 import workloads
    import scipy.sparse as sp
    CACHE.mkdir(parents=True, exist_ok=True)
    f = CACHE / f"{name}.npz"
    w = workloads.WORKLOADS[name]
    if f.exists():
        z = np.load(f)
        A = sp.csr_matrix((z["Av"], z["Ai"], z["Ap"]), shape=(w.m, w.n))
        Y = sp.csr_matrix((z["Yv"], z["Yi"], z["Yp"]), shape=(w.m, w.n_labels))
        return workloads.Problem(w, A, Y)
    t0 = time.time()
    p = workloads.make_problem(name)
    log(f"[bench] generated {name} in {time.time() - t0:.1f}s (nnz={p.A.nnz}, nnz_Y={p.Y.nnz})")
    # atomic publish: concurrent ranks never read a partially written cache file
    tmp = CACHE / f".{name}.{os.getpid()}.npz"
    np.savez(tmp, Av=p.A.data, Ai=p.A.indices, Ap=p.A.indptr, Yv=p.Y.data, Yi=p.Y.indices, Yp=p.Y.indptr)
    os.replace(tmp, f)
    return p


def measured_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        return json.loads(f.read_text()), "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("FPI_CLOCK_MS", "50")],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # one rank per GPU over NCCL; FPI_DIST_BACKEND=gloo is a functional check of the multi-rank
        # path on a box with fewer GPUs than ranks (never a measurement)
        backend = os.environ.get("FPI_DIST_BACKEND", "nccl")
        dev = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_oracle_solve(p):
    """One reference-path solve (oracle port) -> seconds."""
    from oracle import fastpi_oracle as orc
    w = p.workload
    t0 = time.perf_counter()
    out = orc.fastpi(p.A, w.alpha, w.k, w.seed, keep_stages=False)
    orc.apply_pinv(out["pinv"], p.Y)
    return time.perf_counter() - t0, out["timings"]


def reference_arm(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return 0
    from threadpoolctl import threadpool_limits
    cores = cpu_cores()
    p = load_problem(args.workload)
    small = load_problem("c1")
    with threadpool_limits(cores):
        for _ in range(args.warmup):
            run_oracle_solve(small)
        times = []
        budget = args.ref_budget
        t_start = time.time()
        for i in range(args.steps):
            dt, stages = run_oracle_solve(p)
            times.append(dt)
            log(f"[bench:reference] step {i}: {dt:.2f}s {stages}")
            if time.time() - t_start > budget:
                break
    v = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": args.gpus,
        "steps": len(times), "steps_requested": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator of the BASELINE.json configs)",
        "config": workload_config(p, world),
        "cpu_baseline": {"value": v, "unit": "s", "cores": cores, "kind": "port",
                         "sample": f"full {args.workload} solve (fastpi + apply) per step; warm-up on c1; "
                                   f"{len(times)} of {args.steps} steps within a {budget:.0f}s budget"},
        "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(p, world=1):
    w = p.workload
    return {"workload": w.name, "m": w.m, "n": w.n, "nnz": int(p.A.nnz), "n_labels": w.n_labels,
            "nnz_Y": int(p.Y.nnz), "rank": w.rank, "alpha": w.alpha, "k": w.k, "seed": w.seed,
            "l2_flush": "512MB write before every timed step",
            "parallelism": "1 GPU" if world == 1 else
            f"{world} ranks (csrc/sharded.cu): A11 blocks, U rows and Vt / Z columns owned per rank; "
            "NCCL all-reduce of the k x k Grams, of the column update's M^T B and of U^T Y, ncclReduce of "
            "the row update's inner^T B onto column owners; reorder and the small eigensolves replicated"}


def _ncu_traffic():
    """DRAM bytes of one representative launch of the dominant kernel, from the committed
    `ncu --set full` capture summary (profiles/); None when absent."""
    g = None
    for name, key in (("r02_s6_ncu_summary.json", "gemm_c4_apply_lift"),
                      ("r02_ncu_full_summary.json", "r02_gemm_c4_apply_lift")):
        f = Path(__file__).resolve().parent / "profiles" / name
        try:
            g = json.loads(f.read_text())[key]
            break
        except (OSError, KeyError, ValueError):
            continue
    if g is None:
        return None
    return {"source": f"profiles/{f.name}", "launch": g.get("launch"), "traffic_bytes": g.get("traffic_bytes"),
            "algorithmic_bytes": g.get("algorithmic_bytes"), "dmma_pipe_active": g.get("dmma_pipe_active_pct"),
            "ncu_duration": g.get("duration")}


def arm_watchdog(world, rank, seconds):
    """Multi-rank runs only: a collective that one rank never joins (a crashed peer, a communicator
    that failed to form) would hang the job.  After `seconds` the rank reports where it stands on
    stderr and exits non-zero, so torchrun tears the job down instead of waiting out its own limit."""
    if world <= 1 or seconds <= 0:
        return None
    import threading

    def fire():
        log(f"[bench] rank {rank}/{world}: no result after {seconds:.0f}s -- a collective is stuck; aborting")
        import faulthandler
        faulthandler.dump_traceback(file=sys.stderr)
        os._exit(3)
    t = threading.Timer(seconds, fire)
    t.daemon = True
    t.start()
    return t


def ours_arm(args):
    import torch
    world, rank, local = dist_setup()
    arm_watchdog(world, rank, args.dist_timeout)
    import paper_2011_04235_b200 as fp
    from paper_2011_04235_b200 import _lib
    from paper_2011_04235_b200._device import DeviceCSR
    from paper_2011_04235_b200.pinv import fastpi_device

    if world > 1 and rank != 0:
        barrier(world)  # rank 0 generates (or loads) the cached problem first
    p = load_problem(args.workload)
    if world > 1 and rank == 0:
        barrier(world)
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    stream = torch.cuda.current_stream()
    A_dev = DeviceCSR.from_host(p.A)
    Y_dev = DeviceCSR.from_host(p.Y)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MB > L2 (126 MB)
    stats = {}

    if world > 1:
        from paper_2011_04235_b200.sharded import Comm, apply_local, fastpi_distributed, fastpi_sharded
        comm = Comm()
        comm.bind()
        log(f"[bench] rank {rank}/{world}: communicator {comm.kind}")

    def step(collect=False):
        if world > 1:
            res = fastpi_sharded(A_dev, cfg, comm, stats=stats)
            return res, res.pseudoinverse.apply_local(Y_dev)[1]   # this rank's rows of Z
        # timed steps: the public one-call path (fpi_fastpi_ex); the structure record comes from one
        # warm-up pass through the stage-by-stage mirror (same kernels, same bits)
        res = fastpi_device(A_dev, cfg, stats=stats if collect else None)
        return res, res.pseudoinverse.apply_device(Y_dev)

    for i in range(max(args.warmup, 1)):
        t0 = time.perf_counter()
        res, Z = step(collect=(i == 0))
        torch.cuda.synchronize()
        log(f"[bench] warmup {i}: {time.perf_counter() - t0:.3f}s "
            + " ".join(f"{s.stage}={s.seconds * 1e3:.1f}ms" for s in res.timings))
    del res, Z
    launches0 = _lib.kernel_launches()
    times = []
    stage_ms = {}
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res, Z = step()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            for s in res.timings:
                stage_ms.setdefault(s.stage, []).append(s.seconds * 1e3)
            del res, Z
    barrier(world)
    torch.cuda.synchronize()
    launches = _lib.kernel_launches() - launches0
    ms = statistics.mean(times)
    ms_max = max_over_ranks(ms, world)
    clocks = clk.summary()

    # ---- roofline: instrumented pass (per kernel class, CUDA events on the library stream)
    _lib.timing_enable(True)
    flush.fill_(0.0)
    res, Z = step()
    rep = _lib.timing_report(reset=True)
    _lib.timing_enable(False)
    del res, Z
    peaks, peak_src = measured_peaks()
    fp64_peak = _lib.dmma_peak_tflops()
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    torch.matmul(a, a)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(3):
        torch.matmul(a, a)
    t1.record()
    torch.cuda.synchronize()
    cublas_dgemm = 3 * 2 * 8192 ** 3 / (t0.elapsed_time(t1) * 1e-3) / 1e12
    del a
    total_k = sum(v["ms"] for v in rep.values()) or 1.0
    kernels = {k: {"launches": v["launches"], "ms": round(v["ms"], 3), "share_of_step": round(v["ms"] / ms, 4),
                   "gflop": round(v["flops"] / 1e9, 3), "gbytes": round(v["bytes"] / 1e9, 4)}
               for k, v in sorted(rep.items(), key=lambda kv: -kv[1]["ms"])}
    # every class against its own roofline: FP64 tensor for the DMMA GEMM, HBM for the
    # byte-counted classes (SpMM, reorder, permute/partition, sketch); latency-bound classes carry none
    peaks0, _ = measured_peaks()
    fp64_ref = max(_lib.dmma_peak_tflops(), 1e-9)
    for k, v in rep.items():
        if v["ms"] <= 0:
            continue
        if "gemm" in k and v["flops"] > 0:
            kernels[k]["tflops"] = round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 2)
            kernels[k]["roofline_frac"] = round(kernels[k]["tflops"] / fp64_ref, 4)
        elif v["bytes"] > 0:
            kernels[k]["gbs"] = round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1)
            kernels[k]["roofline_frac"] = round(kernels[k]["gbs"] / peaks0["hbm_gbs"], 4)
            if k.startswith("spmm") and v["flops"] > 0:
                # each FMA gathers one 8-byte operand element through L1 / L2 (16 B per 2 flops):
                # the gather stream the kernel actually moves, against which HBM is not the bound
                kernels[k]["gathered_gbs"] = round(4.0 * v["flops"] / (v["ms"] * 1e-3) / 1e9, 1)
    dom_name, dom = max(((k, v) for k, v in rep.items() if v["flops"] > 0 or v["bytes"] > 0),
                        key=lambda kv: kv[1]["ms"], default=(None, None))
    roofline = None
    ncu_traffic = _ncu_traffic()
    if dom is not None:
        avg_ms = dom["ms"] / max(dom["launches"], 1)
        if "gemm" in dom_name:
            ach = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
            peak = max(cublas_dgemm, fp64_peak)
            roofline = {"kernel": dom_name, "bound": "tensor", "achieved": round(ach, 3), "peak": round(peak, 3),
                        "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                        "traffic": ncu_traffic.get("traffic_bytes") if ncu_traffic else None,
                        "traffic_launch": ncu_traffic,
                        "avg_launch_ms": round(avg_ms, 4), "launches": dom["launches"],
                        "share_of_step": round(dom["ms"] / ms, 4),
                        "peak_source": f"measured FP64 on this GPU: max(cuBLAS DGEMM 8192^3 = {cublas_dgemm:.1f}, "
                                       f"DMMA issue-rate microbench = {fp64_peak:.1f}) TFLOP/s"}
        else:
            ach = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
            peak = peaks["hbm_gbs"]
            roofline = {"kernel": dom_name, "bound": "hbm", "achieved": round(ach, 1), "peak": peak,
                        "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": None,
                        "avg_launch_ms": round(avg_ms, 4), "launches": dom["launches"],
                        "share_of_step": round(dom["ms"] / ms, 4), "peak_source": peak_src}

    # the largest kernel class by time when it is not the roofline one (the latency-bound eigensolver
    # carries no algorithmic flop count of its own)
    largest = None
    if rep:
        big_name, big = max(rep.items(), key=lambda kv: kv[1]["ms"])
        if big_name != dom_name:
            largest = {"kernel": big_name, "share_of_step": round(big["ms"] / ms, 4), "launches": big["launches"],
                       "bound": "latency",
                       "note": "two-sided block Jacobi: sequential rotation chains + one grid barrier per round; "
                               "ncu: DMMA sub-pipe 27% active on the c4 n = 1000 launch (29% of the stall samples "
                               "wait at the grid barrier for the pair CTAs' sub-solves), 40% on the c5 n = 2000 "
                               "launch (profiles/r02_s5_ncu_jacobi_c5.json, r02_s5_ncu_jacobi_c5_source_after.txt)"}
        if roofline is not None:
            roofline["largest_kernel"] = largest

    # ---- e2e through the public API with host inputs
    e2e = None
    if not args.no_e2e:
        h2d_bytes = (p.A.indptr.size * 8 + p.A.indices.size * 4 + p.A.data.size * 8
                     + p.Y.indptr.size * 8 + p.Y.indices.size * 4 + p.Y.data.size * 8)
        e2e_t = []
        d2h_bytes = 0
        def e2e_step():
            if world > 1:
                # every rank uploads A and Y and copies ITS rows of Z back (the per-GPU copies run in
                # parallel); the job's Z is the union of the ranks' slices
                res = fastpi_distributed(p.A, cfg, comm)
                return res, apply_local(res.pseudoinverse, p.Y)[1], int(res.sigma.shape[0])
            res = fp.fastpi(p.A, cfg)
            return res, res.pseudoinverse.apply(p.Y), res.factors.rank

        for i in range(args.warmup):  # first calls allocate the pinned host staging buffers
            res, Zh, _ = e2e_step()
            del res, Zh
        for i in range(max(1, args.steps)):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            barrier(world)
            t0 = time.perf_counter()
            res, Zh, rk = e2e_step()
            torch.cuda.synchronize()
            e2e_t.append(time.perf_counter() - t0)
            d2h_bytes = Zh.nbytes + 8 * (3 * rk + 16)
            del res, Zh
        e2e = {"value": max_over_ranks(statistics.mean(e2e_t), world), "unit": "s",
               "h2d_bytes_per_step": int(h2d_bytes), "d2h_bytes_per_step": int(d2h_bytes),
               "note": "fastpi(A scipy) + pseudoinverse.apply(Y scipy) -> numpy Z; pinned staging inside, the upload of "
                       "A's values overlaps the reorder (FPI_NO_DEFERRED_UPLOAD=1 disables it)"}

    # ---- CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from threadpoolctl import threadpool_limits
        cores = cpu_cores()
        with threadpool_limits(cores):
            dt, _ = run_oracle_solve(p)
        cpu = {"value": dt, "unit": "s", "cores": cores, "kind": "port",
               "sample": f"one full {w.name} solve (oracle port: fastpi + apply), {cores} BLAS threads"}

    # ---- the largest config (configs[4], c5) as a second record, measured in a child process
    c5 = None
    if rank == 0 and world == 1 and args.workload == "c4" and not args.no_c5:
        c5 = c5_record(args)

    cpu_partial = None
    if rank == 0 and world == 1 and args.cpu_partial:
        cpu_partial = cpu_partial_c5(p, {k: statistics.mean(v) for k, v in stage_ms.items()})

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms_max / 1e3, "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator of the BASELINE.json configs; paper corpora unavailable)",
            "config": workload_config(p, world), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clocks,
            "stages_ms": {k: round(statistics.mean(v), 3) for k, v in stage_ms.items()},
            "step_ms_all": [round(t, 3) for t in times],
            "kernels": kernels,
            "structure": {k: stats[k] for k in ("m1", "n1", "m2", "n2", "T", "s", "r", "rank11", "engines",
                                                 "svd_diag_row", "svd_diag_col", "sparse_core") if k in stats},
            "fp64_peaks_tflops": {"cublas_dgemm_8192": round(cublas_dgemm, 2), "dmma_microbench": round(fp64_peak, 2)},
        }
        if c5 is not None:
            line["c5"] = c5
        if cpu_partial is not None:
            line["cpu_partial"] = cpu_partial
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def c5_record(args):
    """configs[4] (2M x 200k, 30M nnz, r = 1000, L = 3000) on this GPU: value, e2e, roofline and
    stage times, plus the oracle port's reorder / partition / block-SVD stages on the host cores
    (the full CPU solve of c5 takes tens of minutes; these three stages are the bounded sample)."""
    cmd = [sys.executable, str(Path(__file__).resolve()), "--workload", "c5", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--cpu-partial"]
    log(f"[bench] c5 record: {' '.join(cmd)}")
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=args.c5_timeout)
    except subprocess.TimeoutExpired:
        return {"unavailable": f"c5 run exceeded {args.c5_timeout:.0f}s"}
    sys.stderr.write(out.stderr[-3000:])
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode != 0 or not lines:
        return {"unavailable": f"c5 run failed (exit {out.returncode})"}
    rec = json.loads(lines[-1])
    keep = ("value", "unit", "ms_per_step", "e2e", "roofline", "stages_ms", "kernels", "structure", "clocks",
            "gpu_launches", "config", "cpu_partial", "step_ms_all")
    return {k: rec[k] for k in keep if k in rec}


def cpu_partial_c5(p, gpu_stages):
    """The oracle port's reorder (+ permute / partition) and block SVD on the host cores."""
    from threadpoolctl import threadpool_limits
    from oracle import fastpi_oracle as orc
    w = p.workload
    cores = cpu_cores()
    with threadpool_limits(cores):
        A = orc.canonical_csr(p.A)
        t0 = time.perf_counter()
        o = orc.reorder(*A.shape, A.indptr, A.indices, w.k)
        Ap = orc.permute(A, o.row_fwd, o.col_fwd)
        spoke, _, _, _ = orc.partition(Ap, o)
        t1 = time.perf_counter()
        orc.block_svd(spoke, o.spans, w.alpha)
        t2 = time.perf_counter()
    cpu = {"reorder": t1 - t0, "block_svd": t2 - t1}
    return {"kind": "port", "cores": cores, "unit": "s",
            "sample": "c5 stages reorder + permute/partition and block SVD (oracle port); the row / column "
                      "updates are not run on the host (minutes to hours)",
            "stages_s": {k: round(v, 3) for k, v in cpu.items()},
            "gpu_stages_s": {k: round(gpu_stages[k] / 1e3, 5) for k in cpu if k in gpu_stages},
            "speedup": {k: round(cpu[k] / (gpu_stages[k] / 1e3), 1) for k in cpu if gpu_stages.get(k)}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=240.0, help="seconds of reference steps before stopping")
    ap.add_argument("--no-c5", action="store_true", help="skip the configs[4] (c5) record of the c4 run")
    ap.add_argument("--c5-timeout", type=float, default=600.0)
    ap.add_argument("--dist-timeout", type=float, default=1800.0,
                    help="multi-rank runs: abort a rank that has no result after this many seconds")
    ap.add_argument("--cpu-partial", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    return ours_arm(args)


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: launch the N ranks ourselves (one process per GPU,
    torch.distributed.run on 127.0.0.1) with this command line; rank 0 prints the JSON line.
    NCCL's communicator log (NCCL_DEBUG=INFO unless set) stays on stderr."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    log(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.run(cmd, env=env).returncode


if __name__ == "__main__":
    sys.exit(main())
