"""The experiment runner (paper_2011_04235_b200/cli.py) against the reference CLI's outputs
(reference cli.py:170-225), pinned by tests/golden/cli_c1_* (oracle/make_cli_golden.py ran the
unmodified reference CLI on the c1 workload).  Wall-clock columns are blanked to "T"."""
import re

import pytest

from conftest import GOLDEN
from paper_2011_04235_b200 import cli


def _blank(text, cols):
    rows = text.strip().split("\n")
    out = [rows[0]]
    for r in rows[1:]:
        f = r.split(",")
        for c in cols:
            assert re.fullmatch(r"\d+\.\d{6}", f[c]), r
            f[c] = "T"
        out.append(",".join(f))
    return "\n".join(out) + "\n"


def test_usage_errors_exit_2(tmp_path, capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["bench-time", "--input", "x", "--alphas", "1.5", "--methods", "fastpi", "--seed", "0", "--out", "o"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["bench-time", "--input", "x", "--alphas", "0.1", "--methods", "svd", "--seed", "0", "--out", "o"])
    assert e.value.code == 2
    # missing input file: I/O error -> 2
    assert cli.main(["pinv", "--input", str(tmp_path / "none.txt"), "--alpha", "0.2", "--k", "0.01", "--seed", "0",
                     "--out", str(tmp_path / "p")]) == 2
    assert "fastpi: error:" in capsys.readouterr().err


def test_runs_must_be_positive(tmp_path, capsys):
    assert cli.main(["bench-time", "--input", str(GOLDEN / "cli_c1.txt"), "--alphas", "0.2", "--methods", "fastpi",
                     "--seed", "0", "--runs", "0", "--out", str(tmp_path / "t.csv")]) == 3
    assert "--runs must be at least 1" in capsys.readouterr().err


def test_stage_file_name():
    assert cli.stages_path("out/t.csv").name == "t.stages.csv"
    assert cli.stages_path("out/t").name == "t.stages.csv"
    assert cli.fmt_float(0.2) == "0.20000000000000001"


@pytest.mark.gpu
def test_bench_time_matches_reference_layout(tmp_path):
    out = tmp_path / "t.csv"
    assert cli.main(["bench-time", "--input", str(GOLDEN / "cli_c1.txt"), "--alphas", "0.2", "--methods",
                     "fastpi,randpi,dense", "--seed", "0", "--runs", "2", "--out", str(out)]) == 0
    assert _blank(out.read_text(), [2]) == (GOLDEN / "cli_c1_bench_time.csv").read_text()
    assert _blank((tmp_path / "t.stages.csv").read_text(), [4]) == \
        (GOLDEN / "cli_c1_bench_time.stages.csv").read_text()


@pytest.mark.gpu
def test_bench_error_matches_reference(tmp_path):
    out = tmp_path / "e.csv"
    assert cli.main(["bench-error", "--input", str(GOLDEN / "cli_c1.txt"), "--alphas", "0.1,0.2", "--methods",
                     "fastpi,randpi,dense", "--seed", "0", "--out", str(out)]) == 0
    got = out.read_text().strip().split("\n")
    ref = (GOLDEN / "cli_c1_bench_error.csv").read_text().strip().split("\n")
    assert got[0] == ref[0] and len(got) == len(ref)
    for g, r in zip(got[1:], ref[1:]):
        gm, ga, ge = g.split(",")
        rm, ra, re_ = r.split(",")
        assert (gm, ga) == (rm, ra)
        assert abs(float(ge) - float(re_)) <= 1e-8 * float(re_), (g, r)


@pytest.mark.gpu
def test_regress_matches_reference(tmp_path):
    """Same rows, method / alpha / k / seed columns and formatting as the reference's cell.  The
    precision values are compared to 0.01: the c1 test split's top scores include near-ties at
    1e-18 (labels seen in almost no training row), so a rounding-level difference in Z may swap
    the order of two such labels (the oracle reproduces the reference's 0.57 / 0.465 / 0.377)."""
    out = tmp_path / "r.csv"
    assert cli.main(["regress", "--dataset", str(GOLDEN / "cli_c1.txt"), "--alpha", "0.2", "--method", "fastpi",
                     "--seed", "0", "--out", str(out)]) == 0
    got = _blank(out.read_text(), [4]).strip().split("\n")
    ref = (GOLDEN / "cli_c1_regress.csv").read_text().strip().split("\n")
    assert got[0] == ref[0] and len(got) == len(ref)
    for g, r in zip(got[1:], ref[1:]):
        gf, rf = g.split(","), r.split(",")
        assert gf[:3] + gf[4:] == rf[:3] + rf[4:], (g, r)
        assert abs(float(gf[3]) - float(rf[3])) <= 0.01, (g, r)
