"""Pins for O1 (oracle/spmv.py, oracle/o1.c): brute force, scipy, closed forms."""
import numpy as np
import pytest
import scipy.sparse as sp

import gen
from oracle import spmv as O1


def _rand_cases():
    cases = []
    for n in (1, 7, 33, 64):
        for dens in (0.0, 0.1, 0.5, 1.0):
            cases.append((n, dens, (), ()))
    cases.append((40, 0.2, (0, 5, 39), (7,)))      # empty rows + one full row
    cases.append((64, 0.05, tuple(range(0, 64, 3)), (1, 2)))
    return cases


@pytest.mark.parametrize("n,dens,empty,dense", _rand_cases())
@pytest.mark.parametrize("exact", [True, False])
def test_o1_matches_dense_bruteforce(n, dens, empty, dense, exact):
    rp, col, val = gen.random_csr(n, dens, seed=17 + n, exact=exact,
                                  empty_rows=empty, dense_rows=dense)
    x = gen.x_values((0, n), exact=exact)
    y = O1.o1_spmv(rp, col, val, x)
    yb = O1.dense_bruteforce(O1.csr_to_dense(rp, col, val, n), x)
    if exact:
        assert np.array_equal(y, yb)
    else:
        s = O1.o1_absdot(rp, col, val, x)
        assert np.all(np.abs(y - yb) <= 1e-13 * s)
    for i in empty:
        assert y[i] == 0.0 and not np.signbit(y[i])  # empty sum = +0.0 (R-Q18)


@pytest.mark.parametrize("which", ["c1", "7pt16", "27pt10", "powerlaw"])
def test_o1_matches_scipy(which):
    if which == "c1":
        n, (rp, col, val) = gen.config_matrix("c1")
    elif which == "7pt16":
        n = 16 ** 3
        rp, col, val = gen.stencil("7pt", (16, 16, 16))
    elif which == "27pt10":
        n = 10 ** 3
        rp, col, val = gen.stencil("27pt", (10, 10, 10))
    else:
        n = 1 << 14
        rp, col, val = gen.powerlaw(n)
    x = gen.x_values((0, n))
    y = O1.o1_spmv(rp, col, val, x)
    ys = sp.csr_matrix((val, col, rp), shape=(n, n)) @ x
    s = O1.o1_absdot(rp, col, val, x)
    # any two summation orders differ by <= 2*gamma_k*sum|a x| (R-Q11)
    assert np.all(np.abs(y - ys) <= 1e-12 * s)


def test_identity_returns_x():
    n = 1000
    rp = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    val = np.ones(n)
    x = gen.x_values((0, n))
    assert np.array_equal(O1.o1_spmv(rp, col, val, x), x)


def _out_of_domain(kind, dims):
    """Number of stencil neighbours of each grid point outside the grid,
    counted geometrically (independent of the CSR)."""
    mx, my, mz = dims
    offs = gen.stencil_offsets(kind)
    k, j, i = np.meshgrid(np.arange(mz), np.arange(my), np.arange(mx), indexing="ij")
    out = np.zeros((mz, my, mx), np.int64)
    for dk, dj, di in offs:
        if (dk, dj, di) == (0, 0, 0):
            continue
        inside = ((i + di >= 0) & (i + di < mx) & (j + dj >= 0) & (j + dj < my)
                  & (k + dk >= 0) & (k + dk < mz))
        out += ~inside
    return out.reshape(-1)


@pytest.mark.parametrize("kind,dims", [("5pt", (64, 64, 1)), ("7pt", (9, 7, 5)),
                                       ("27pt", (6, 5, 4)), ("7pt", (16, 16, 16))])
def test_laplacian_times_ones(kind, dims):
    """Laplacian x 1: y_i = number of out-of-domain neighbours (0 interior;
    7-pt faces/edges/corners 1/2/3) -- SURVEY §8(c) closed forms."""
    n = dims[0] * dims[1] * dims[2]
    rp, col, val = gen.stencil(kind, dims)
    y = O1.o1_spmv(rp, col, val, np.ones(n))
    assert np.array_equal(y, _out_of_domain(kind, dims).astype(np.float64))
    if kind == "7pt" and min(dims) >= 3:
        assert set(np.unique(y)) == {0.0, 1.0, 2.0, 3.0}


@pytest.mark.parametrize("kind,dims", [("7pt", (8, 9, 10)), ("27pt", (7, 6, 5)),
                                       ("5pt", (12, 11, 1))])
def test_laplacian_times_linear(kind, dims):
    """x(i,j,k) = a i + b j + c k + d is annihilated on interior rows."""
    mx, my, mz = dims
    n = mx * my * mz
    rp, col, val = gen.stencil(kind, dims)
    g = np.arange(n)
    i, j, k = g % mx, (g // mx) % my, g // (mx * my)
    x = (3 * i - 2 * j + 5 * k + 7).astype(np.float64)
    y = O1.o1_spmv(rp, col, val, x)
    interior = _out_of_domain(kind, dims) == 0
    assert interior.any()
    assert np.all(y[interior] == 0.0)


def test_absdot_bounds_y():
    rp, col, val = gen.powerlaw(4096)
    x = gen.x_values((0, 4096))
    y = O1.o1_spmv(rp, col, val, x)
    s = O1.o1_absdot(rp, col, val, x)
    assert np.all(np.abs(y) <= s * (1 + 1e-12))


def test_o1_rows_sample_equals_full():
    rp, col, val = gen.stencil("27pt", (12, 12, 12))
    x = gen.x_values((0, 12 ** 3))
    y = O1.o1_spmv(rp, col, val, x)
    rows = np.array([0, 5, 100, 1727], np.int64)
    assert np.array_equal(O1.o1_spmv_rows(rows, rp, col, val, x), y[rows])


def test_exact_mode_partial_sums_fit():
    """Exact mode (R-Q23): |partial sums| <= 4096*8*16 < 2^24, so fp32 and fp64
    are exact -- check the bound on a power-law matrix."""
    rp, col, val = gen.powerlaw(1 << 13, exact=True)
    x = gen.x_values((0, 1 << 13), exact=True)
    assert np.all(np.abs(val) <= 8) and np.all(val != 0)
    assert np.all(np.abs(x) <= 16)
    s = O1.o1_absdot(rp, col, val, x)
    assert s.max() < 2 ** 24
    y32 = O1.o1_spmv(rp, col, val.astype(np.float32).astype(np.float64), x)
    assert np.array_equal(y32, O1.o1_spmv(rp, col, val, x))


def test_o1_openmp_rows_equal_serial_bitwise():
    """The all-cores CPU baseline (the O1 loop under
    `omp parallel for schedule(static)` over rows) sums every row in one
    thread in stored order, so it equals the serial O1 bit for bit."""
    mats = [gen.powerlaw(20000), gen.stencil("27pt", (14, 14, 14)),
            gen.random_csr(300, 0.05, seed=11, empty_rows=(0, 1, 150, 299), dense_rows=(7, 200))]
    for rp, col, val in mats:
        n = len(rp) - 1
        x = gen.x_values((0, n))
        assert np.array_equal(O1.o1_spmv_omp(rp, col, val, x), O1.o1_spmv(rp, col, val, x))
    assert O1.o1_threads() >= 1


# --------------------------------------------------------------------------
# Independent pins for o1_absdot, the scale s_i = sum_j |a_ij x_j| of every
# tolerance assertion (BASELINE.json north_star).  The |y| <= s bound above is
# one-sided: an over-large s (an accumulator not reset per row, sum|a| max|x|)
# would pass it and silently loosen every parity test.  These pin s from the
# other side with a library routine and with closed forms.

def _scipy_absdot(rp, col, val, x, n):
    A = sp.csr_matrix((np.abs(val), col, rp - rp[0]), shape=(len(rp) - 1, n))
    return A @ np.abs(x)


@pytest.mark.parametrize("name", ["rand", "pl", "27pt", "5pt"])
def test_absdot_exact_mode_equals_scipy_abs_product(name):
    """Exact mode (integers, R-Q23): |A| @ |x| by scipy is exact, so O1's s
    must equal it bitwise, row by row (including empty rows, where s = 0)."""
    if name == "rand":
        n = 300
        rp, col, val = gen.random_csr(n, 0.05, seed=3, exact=True,
                                      empty_rows=(0, 17, 299), dense_rows=(5,))
    elif name == "pl":
        n = 20000
        rp, col, val = gen.powerlaw(n, exact=True)
    elif name == "27pt":
        n = 9 * 8 * 7
        rp, col, val = gen.stencil("27pt", (9, 8, 7))
    else:
        n = 33 * 31
        rp, col, val = gen.stencil("5pt", (33, 31, 1))
    x = gen.x_values((0, n), exact=True)
    s = O1.o1_absdot(rp, col, val, x)
    assert np.array_equal(s, _scipy_absdot(rp, col, val, x, n))


@pytest.mark.parametrize("n,dens", [(64, 0.5), (300, 0.05), (2000, 0.01)])
def test_absdot_float_mode_within_rounding_of_scipy(n, dens):
    """Float mode: both sides sum k nonnegative terms, so each is within
    gamma_k = k u/(1 - k u) (u = 2^-53) of the exact value; the two differ by
    at most 2 gamma_k s_i."""
    rp, col, val = gen.random_csr(n, dens, seed=23, exact=False, dense_rows=(1,))
    x = gen.x_values((0, n))
    s = O1.o1_absdot(rp, col, val, x)
    ref = _scipy_absdot(rp, col, val, x, n)
    k = np.diff(rp).astype(np.float64)
    u = 2.0 ** -53
    g = k * u / (1 - k * u)
    assert np.all(np.abs(s - ref) <= 2 * g * ref)
    assert np.all(s > 0) or np.all(s[k > 0] > 0)


def test_absdot_nonnegative_inputs_equal_y():
    """Closed form: with a_ij >= 0 and x_j >= 0, |a_ij x_j| = a_ij x_j, so s is
    the same sum in the same order as y -- bitwise equal to O1's y."""
    n = 500
    rp, col, val = gen.random_csr(n, 0.03, seed=5, exact=False, empty_rows=(3,))
    val = np.abs(val)
    x = np.abs(gen.x_values((0, n)))
    assert np.array_equal(O1.o1_absdot(rp, col, val, x), O1.o1_spmv(rp, col, val, x))


def test_absdot_cancellation_rows():
    """Closed forms: a row (+1, -1) against x = (1, 1) gives y = 0 but s = 2; an
    empty row gives s = 0; a row (2, -3, 5) against (1, -1, 2) has all products
    positive, so s = y = 15; a row (2, 3) against (1, -1) gives y = -1, s = 5."""
    rp = np.array([0, 2, 2, 5, 7], np.int64)
    col = np.array([0, 1, 0, 1, 2, 0, 1], np.int32)
    val = np.array([1.0, -1.0, 2.0, -3.0, 5.0, 2.0, 3.0])
    x = np.array([1.0, -1.0, 2.0])
    s = O1.o1_absdot(rp, col, val, np.array([1.0, 1.0, 1.0]))
    assert s[0] == 2.0 and s[1] == 0.0
    s = O1.o1_absdot(rp, col, val, x)
    y = O1.o1_spmv(rp, col, val, x)
    assert s.tolist() == [2.0, 0.0, 15.0, 5.0]
    assert y.tolist() == [2.0, 0.0, 15.0, -1.0]


def test_absdot_is_per_row_and_scales_with_x():
    """Row-locality (a sample of rows equals the same rows of the full s after
    permuting the row order) and homogeneity s(A, c x) = |c| s(A, x) for c a
    power of two (exact)."""
    n = 4096
    rp, col, val = gen.powerlaw(n)
    x = gen.x_values((0, n))
    s = O1.o1_absdot(rp, col, val, x)
    perm = np.random.default_rng(1).permutation(n)
    lens = np.diff(rp)[perm]
    rp2 = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col2 = np.concatenate([col[rp[i]:rp[i + 1]] for i in perm])
    val2 = np.concatenate([val[rp[i]:rp[i + 1]] for i in perm])
    assert np.array_equal(O1.o1_absdot(rp2, col2, val2, x), s[perm])
    assert np.array_equal(O1.o1_absdot(rp, col, val, -0.25 * x), 0.25 * s)
