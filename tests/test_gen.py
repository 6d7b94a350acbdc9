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


@pytest.mark.parametrize("kind,dims,pgrid", [("7pt", (8, 6, 4), (2, 3, 2)), ("27pt", (6, 6, 6), (3, 1, 2)),
                                             ("7pt", (12, 12, 12), (2, 2, 2))])
def test_blocked_stencil_is_a_symmetric_permutation(kind, dims, pgrid):
    """NEXT-4 generator: stencil_blocked = P A P^T of the natural stencil
    (y' = A' x' with x' = P x gives y' = P y exactly, integer values), the
    numbering is a bijection, and row slices match the full matrix."""
    from oracle import spmv as O1
    n = dims[0] * dims[1] * dims[2]
    rp, col, val = gen.stencil_blocked(kind, dims, pgrid)
    rn, cn, vn = gen.stencil(kind, dims)
    ni = gen.blocked_index(dims, pgrid)(np.arange(n))
    assert np.array_equal(np.sort(ni), np.arange(n))
    x = gen.x_values((0, n), exact=True)
    xp = np.empty(n)
    xp[ni] = x
    assert np.array_equal(O1.o1_spmv(rp, col, val, xp)[ni], O1.o1_spmv(rn, cn, vn, x))
    assert all(np.all(np.diff(col[rp[i]:rp[i + 1]]) > 0) for i in range(n))
    lo, hi = n // 3, 2 * n // 3
    r2, c2, v2 = gen.stencil_blocked(kind, dims, pgrid, (lo, hi))
    assert np.array_equal(c2, col[rp[lo]:rp[hi]]) and np.array_equal(r2, rp[lo:hi + 1] - rp[lo])


def test_blocked_stencil_halo_is_the_block_faces():
    """7-pt on a 2x2x2 block decomposition: every rank's peers are its face
    neighbours at rank offsets +-1, +-px, +-px*py and each receives exactly
    one block face (closed form) from each (oracle planner)."""
    from oracle import plan as O2
    dims, pg = (8, 6, 4), (2, 2, 2)
    bx, by, bz = 4, 3, 2
    n = 8 * 6 * 4
    rp, col, val = gen.stencil_blocked("7pt", dims, pg)
    plans = O2.plan_all(rp, col, n, 8)
    face = {1: by * bz, 2: bx * bz, 4: bx * by}
    for r, pl in enumerate(plans):
        for q in range(8):
            d = q - r
            c = int(pl["recv_count"][q])
            if abs(d) in face:
                bxr, byr, bzr = r % 2, (r // 2) % 2, r // 4
                bxq, byq, bzq = q % 2, (q // 2) % 2, q // 4
                neighbour = (abs(bxr - bxq) + abs(byr - byq) + abs(bzr - bzq)) == 1
                assert c == (face[abs(d)] if neighbour else 0), (r, q)
            else:
                assert c == 0, (r, q)
