"""SVD engines (reference svd.py) on the B200 core."""

from __future__ import annotations

from . import _lib
from ._device import empty


def gaussian_sketch_device(seed: int, rows: int, cols: int):
    """svd.py:131-132 -- numpy ``default_rng(seed).standard_normal((rows, cols))``, bitwise, in HBM."""
    X = empty((rows, cols), "f64")
    _lib.call("fpi_sketch_normal", int(seed), int(rows), int(cols), _lib.ptr(X), int(cols))
    return X
