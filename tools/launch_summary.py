"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per kernel name)."""
import csv
import io
import sys
from collections import defaultdict


def main(path, top=40):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    seq = []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1000.0 if unit == "nsecond" or unit == "ns" else (v if unit in ("usecond", "us") else v * 1000.0)
        name = r["Kernel Name"].split("(")[0][:90]
        agg[name][0] += 1
        agg[name][1] += us
        total += us
        seq.append((name, us))
    print(f"{len(seq)} launches, {total / 1000:.2f} ms summed kernel time")
    print("| kernel | launches | ms | share |\n|---|---:|---:|---:|")
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"| `{name}` | {n} | {us / 1000:.3f} | {100 * us / total:.1f}% |")
    return seq


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
