"""Golden CLI outputs from the unmodified reference (TEST INFRASTRUCTURE; build container only).

Writes tests/golden/cli_c1.txt (the c1 workload as a reference dataset file) and, from the
reference's own ``fastpi.cli.main`` on it:
  * cli_c1_bench_time.csv / cli_c1_bench_time.stages.csv  -- bench-time over fastpi, randpi,
    dense at alpha 0.2 with 2 runs; wall-clock seconds replaced by "T" (they are not reproducible),
    everything else (row order, stage names, ranks, number formatting) kept verbatim;
  * cli_c1_bench_error.csv  -- bench-error, kept verbatim (the GPU's errors are compared to 1e-8);
  * cli_c1_regress.csv      -- regress cell with train_seconds replaced by "T".

Usage: python oracle/make_cli_golden.py
"""

from __future__ import annotations

import re
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REF = Path("/root/reference/pkg/src")
GOLD = ROOT / "tests" / "golden"


def blank_seconds(text: str, cols) -> str:
    rows = text.strip().split("\n")
    out = [rows[0]]
    for r in rows[1:]:
        f = r.split(",")
        for c in cols:
            assert re.fullmatch(r"\d+\.\d{6}", f[c]), r
            f[c] = "T"
        out.append(",".join(f))
    return "\n".join(out) + "\n"


def main():
    if not REF.exists():
        raise SystemExit("reference not present; run in the build container")
    sys.path.insert(0, str(REF))
    import fastpi.cli as rcli
    from paper_2011_04235_b200 import workloads
    from paper_2011_04235_b200.datasets import save_dataset
    from paper_2011_04235_b200.regression import MultiLabelDataset

    p = workloads.make_problem("c1")
    data = GOLD / "cli_c1.txt"
    # the reference's own save_dataset writes numpy-2 scalar reprs ('np.float64(...)') that its loader
    # rejects; this writer emits the same format with plain float reprs (exact round trip)
    save_dataset(MultiLabelDataset(p.A.tocsr(), p.Y.tocsr()), data)
    with tempfile.TemporaryDirectory() as td:
        td = Path(td)
        assert rcli.main(["bench-time", "--input", str(data), "--alphas", "0.2", "--methods", "fastpi,randpi,dense",
                          "--seed", "0", "--runs", "2", "--out", str(td / "t.csv")]) == 0
        (GOLD / "cli_c1_bench_time.csv").write_text(blank_seconds((td / "t.csv").read_text(), [2]))
        (GOLD / "cli_c1_bench_time.stages.csv").write_text(blank_seconds((td / "t.stages.csv").read_text(), [4]))
        assert rcli.main(["bench-error", "--input", str(data), "--alphas", "0.1,0.2", "--methods",
                          "fastpi,randpi,dense", "--seed", "0", "--out", str(td / "e.csv")]) == 0
        (GOLD / "cli_c1_bench_error.csv").write_text((td / "e.csv").read_text())
        assert rcli.main(["regress", "--dataset", str(data), "--alpha", "0.2", "--method", "fastpi", "--seed", "0",
                          "--out", str(td / "r.csv")]) == 0
        (GOLD / "cli_c1_regress.csv").write_text(blank_seconds((td / "r.csv").read_text(), [4]))
    print("wrote", sorted(x.name for x in GOLD.glob("cli_c1*")))


if __name__ == "__main__":
    main()
