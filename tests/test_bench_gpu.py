"""bench.py's multi-rank launch: `bench.py --gpus N` outside torchrun spawns N ranks itself and
reports n_gpus = N (the driver's scaling contract).  The box has one GPU, so the two ranks share
it over gloo -- a functional check of the launch and of the sharded solve, never a measurement."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.gpu
def test_bench_gpus_2_spawns_two_ranks():
    env = dict(os.environ, FPI_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--workload", "c1", "--steps", "1",
                          "--warmup", "1", "--no-cpu-baseline"], env=env, capture_output=True, text=True,
                         timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-4000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2
    assert rec["value"] > 0 and rec["e2e"]["value"] > 0
    assert "2 ranks" in rec["config"]["parallelism"]
