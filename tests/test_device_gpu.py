"""GPU: host <-> device transfers of the Python host layer (_device.h2d / d2h)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,dtype", [((1000,), np.float64), ((700_000,), np.float64), ((5_000_001,), np.float64),
                                         ((9_000_000,), np.int32), ((3000, 1500), np.float64),
                                         ((4_194_304,), np.float64), ((4_194_305,), np.int64), ((0,), np.float64)])
def test_h2d_round_trip(shape, dtype):
    """Small arrays go directly, arrays >= 1 MB through one page-locked block, arrays >= 32 MB in 16 MB
    chunks whose staging overlaps the previous chunk's DMA: the device copy equals the source in
    every regime (chunk boundaries, a ragged last chunk, 2-D shapes, an exact multiple of the chunk)."""
    from paper_2011_04235_b200._device import d2h, h2d
    rng = np.random.default_rng(int(np.prod(shape)) % 9973)
    if np.issubdtype(dtype, np.floating):
        a = rng.standard_normal(shape).astype(dtype)
    else:
        a = rng.integers(-2**31, 2**31 - 1, size=shape).astype(dtype)
    dev = h2d(a)
    assert tuple(dev.shape) == tuple(a.shape)
    np.testing.assert_array_equal(d2h(dev), a)


def test_h2d_casts_and_makes_contiguous():
    from paper_2011_04235_b200._device import d2h, h2d
    a = np.arange(6_000_000, dtype=np.int32).reshape(2000, 3000)[:, ::2]   # non-contiguous view
    dev = h2d(a, np.int64)
    assert dev.dtype.is_floating_point is False and dev.element_size() == 8
    np.testing.assert_array_equal(d2h(dev), a.astype(np.int64))
