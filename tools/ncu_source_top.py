"""Top CUDA source lines of an ncu --set full --import-source on report: stall samples and executed
instructions per line (ncu -i REP --page source --print-source cuda,sass --csv)."""
import csv
import io
import subprocess
import sys


def main(path, top=28):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[2]
    ix = {}
    for i, h in enumerate(hdr):
        ix.setdefault(h, i)

    def gi(r, k):
        try:
            return int(r[ix[k]])
        except (ValueError, IndexError):
            return 0
    data = [r for r in rows[3:] if len(r) > ix["# Samples"] and r[0].isdigit() and r[2] == "-"]
    tot = sum(gi(r, "# Samples") for r in data) or 1
    ti = sum(gi(r, "Instructions Executed") for r in data) or 1
    print(f"{path}: {tot} samples, {ti / 1e9:.2f} G warp instructions")
    print("line  samples%  instr%  source")
    for r in sorted(data, key=lambda r: -gi(r, "# Samples"))[:top]:
        print(f"{r[0]:>5} {100 * gi(r, '# Samples') / tot:7.1f}% {100 * gi(r, 'Instructions Executed') / ti:6.1f}%  {r[1][:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 28)
