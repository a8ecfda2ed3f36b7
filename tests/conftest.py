"""Shared test setup: repo root on sys.path, the ``gpu`` marker, golden fixtures."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz", allow_pickle=False))


_PROBLEMS = {}


def problem(name):
    from paper_2011_04235_b200 import workloads
    if name not in _PROBLEMS:
        _PROBLEMS[name] = workloads.make_problem(name)
    return _PROBLEMS[name]
