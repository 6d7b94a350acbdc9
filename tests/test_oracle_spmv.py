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
