"""The generators: C twin == numpy recipe; row-range independence."""
import numpy as np
import pytest

import gen


@pytest.mark.parametrize("n,rng,exact", [(3000, None, False), (20000, (777, 5100), True),
                                         (1 << 16, (0, 4096), False), (50, None, False)])
def test_powerlaw_c_equals_numpy(n, rng, exact):
    assert gen._genc() is not None, "gen/libgenc.so not built"
    a = gen.powerlaw(n, rng, exact=exact)
    b = gen.powerlaw_numpy(n, rng, exact=exact)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_row_range_independence():
    rp, col, val = gen.powerlaw(10000)
    rp2, col2, val2 = gen.powerlaw(10000, (1234, 5678))
    assert np.array_equal(col2, col[rp[1234]:rp[5678]])
    assert np.array_equal(val2, val[rp[1234]:rp[5678]])
    rp, col, val = gen.stencil("27pt", (9, 8, 7))
    rp2, col2, val2 = gen.stencil("27pt", (9, 8, 7), (100, 300))
    assert np.array_equal(col2, col[rp[100]:rp[300]])


def test_powerlaw_shape_statistics():
    rp, col, val = gen.powerlaw(1 << 18)
    L = np.diff(rp)
    assert 15.0 < L.mean() < 17.0 and L.min() >= 8 and L.max() <= 4096
    assert np.percentile(L, 50) in (10, 11, 12)
