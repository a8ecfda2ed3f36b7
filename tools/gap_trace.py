"""GPU idle gaps inside one c4 solve + apply (torch.profiler / CUPTI kernel timeline): where the
device waits on the host (stream syncs for data-dependent sizes, Python between stages).

    python tools/gap_trace.py [c4] [min_gap_us] [capi|stagewise]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2011_04235_b200 as fp  # noqa: E402
from paper_2011_04235_b200._device import DeviceCSR  # noqa: E402
from paper_2011_04235_b200.pinv import fastpi_device  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    min_gap = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
    torch.cuda.set_device(0)
    p = bench.load_problem(name)
    w = p.workload
    cfg = fp.FastpiConfig(alpha=w.alpha, k=w.k, seed=w.seed)
    A, Y = DeviceCSR.from_host(p.A), DeviceCSR.from_host(p.Y)
    use_c = len(sys.argv) > 3 and sys.argv[3] == "capi"
    stagewise = len(sys.argv) > 3 and sys.argv[3] == "stagewise"
    import ctypes as C
    from paper_2011_04235_b200 import _lib

    def solve():
        if use_c:  # Algorithm 1 in one C call (fpi_fastpi): no Python between the stages
            info = _lib.FastpiInfo()
            _lib.call("fpi_fastpi", A.shape[0], A.shape[1], A.nnz, _lib.ptr(A.indptr), _lib.ptr(A.indices),
                      _lib.ptr(A.values), float(cfg.alpha), float(cfg.k), int(cfg.seed),
                      float(cfg.low_rank_threshold), float(cfg.pinv_cutoff_factor), C.byref(info))
            return
        res = fastpi_device(A, cfg, stagewise=stagewise)
        res.pseudoinverse.apply_device(Y)

    for _ in range(3):
        solve()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=True) as prof:
        solve()
        torch.cuda.synchronize()
    allev = prof.events()
    cpu = sorted([e for e in allev if e.device_type == torch.autograd.DeviceType.CPU],
                 key=lambda e: e.time_range.start)
    ev = [e for e in allev if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    spans = [(e.time_range.start, e.time_range.end, e.name) for e in ev]
    busy = sum(e - s for s, e, _ in spans)
    total = spans[-1][1] - spans[0][0]
    gaps = []
    end = spans[0][1]
    for i in range(1, len(spans)):
        s, e, n = spans[i]
        if s - end > min_gap:
            ctx = " < ".join(x[2][:40] for x in spans[max(0, i - 3):i])
            gaps.append((s - end, ctx, n[:50], i))
        end = max(end, e)
    gaps.sort(reverse=True)
    print(f"{len(spans)} device events, span {total / 1e3:.2f} ms, busy {busy / 1e3:.2f} ms, "
          f"gaps > {min_gap:.0f} us: {len(gaps)} totalling {sum(g[0] for g in gaps) / 1e3:.2f} ms")
    for g, a, b, i in gaps[:40]:
        print(f"{g:8.1f} us  #{i}  [{a}]  -> {b}")
    # host activity inside the largest gaps (CUDA runtime calls and Python frames)
    for g, a, b, i in gaps[:8]:
        g0, g1 = spans[i - 1][1], spans[i][0]
        print(f"--- gap #{i} ({g:.0f} us): host events overlapping it")
        for e in cpu:
            s0, s1 = e.time_range.start, e.time_range.end
            if s1 < g0 or s0 > g1 or s1 - s0 < 8:
                continue
            stack = [f for f in (e.stack or []) if "paper_2011" in f or "bench" in f][:3]
            print(f"   {s0 - g0:8.1f} +{s1 - s0:7.1f} us  {e.name[:50]:50s} {' | '.join(stack)[:160]}")


if __name__ == "__main__":
    main()
