"""Key counters of an ncu --set full report (first kernel) as a JSON object."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dmma_pipe_active_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "wait", "math_pipe_throttle", "lg_throttle",
          "mio_throttle", "membar", "branch_resolving", "no_instruction", "sleeping", "selected"]


def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    res = {"kernel": get.get("Kernel Name", ("", ""))[0][:100]}
    for k, m in KEYS.items():
        if m in get:
            res[k] = f"{get[m][0]} {get[m][1]}".strip()
    st = []
    for s in STALLS:
        m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if m in get:
            try:
                st.append((s, round(float(get[m][0]), 2)))
            except ValueError:
                pass
    res["top_stalls_per_issue"] = sorted(st, key=lambda x: -x[1])[:6]
    return res


if __name__ == "__main__":
    print(json.dumps({p: summary(p) for p in sys.argv[1:]}, indent=1))
