"""GPU: the Gaussian sketch is bitwise numpy's default_rng(seed).standard_normal."""
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _gpu(seed, rows, cols):
    from paper_2011_04235_b200 import svd
    return svd.gaussian_sketch_device(seed, rows, cols).cpu().numpy()


@pytest.mark.parametrize("seed,rows,cols", [(0, 1, 1), (1, 7, 3), (2, 500, 200), (3, 1000, 1000),
                                            (12345, 333, 77), (2**33 + 1, 10, 1000), (7, 39870, 798)])
def test_sketch_bitwise(seed, rows, cols):
    X = _gpu(seed, rows, cols)
    ref = np.random.default_rng(seed).standard_normal((rows, cols))
    mism = np.flatnonzero(X.view(np.uint64).ravel() != ref.view(np.uint64).ravel())
    assert mism.size == 0, f"{mism.size} mismatches, first at {mism[:5]}"


def test_sketch_golden_hashes():
    vecs = json.loads((GOLDEN / "sketches.json").read_text())
    for v in vecs:
        X = _gpu(v["seed"], v["rows"], v["cols"])
        assert hashlib.sha256(X.tobytes()).hexdigest() == v["sha256"], v


def test_sketch_large_tail_coverage():
    # ~25M samples: thousands of tail and wedge branches, chunk-boundary crossings
    X = _gpu(4 + 2, 12500, 2000)
    ref = np.random.default_rng(6).standard_normal((12500, 2000))
    assert np.array_equal(X.view(np.uint64), ref.view(np.uint64))
    assert (np.abs(ref) > 3.6541528853610088).sum() > 1000  # the tail branch was exercised
