"""O1 -- the serial CSR product.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

``o1_spmv`` runs the plain C loop in ``oracle/o1.c`` (rows ascending, stored
order, fp64, product and sum rounded separately).  ``dense_bruteforce`` is the
textbook sum over a dense matrix used to pin O1 on tiny inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libo1.so")
_lib = None


def build() -> str:
    """Compile o1.c (plain -O2, no FMA contraction, no fast-math)."""
    src = os.path.join(_HERE, "o1.c")
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        for name in ("o1_spmv", "o1_absdot", "o1_spmv_omp"):
            f = getattr(lib, name)
            f.argtypes = [ctypes.c_int64, P, P, P, P, P]
            f.restype = None
        lib.o1_spmv_rows.argtypes = [ctypes.c_int64, P, P, P, P, P, P]
        lib.o1_spmv_rows.restype = None
        lib.o1_omp_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def o1_spmv(rowptr, col, val, x) -> np.ndarray:
    """y_i = sum_{p in row i} val[p] * x[col[p]] in fp64."""
    lib = _load()
    rowptr = _c(rowptr, np.int64)
    col = _c(col, np.int32)
    val = _c(val, np.float64)
    x = _c(x, np.float64)
    n = len(rowptr) - 1
    y = np.empty(n, np.float64)
    if n:
        lib.o1_spmv(n, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data,
                    x.ctypes.data, y.ctypes.data)
    return y


def o1_spmv_omp(rowptr, col, val, x) -> np.ndarray:
    """The O1 loop with its rows split over all host cores (OpenMP, static
    schedule; SURVEY 8(d) CPU baseline); bitwise equal to o1_spmv."""
    lib = _load()
    rowptr = _c(rowptr, np.int64)
    col = _c(col, np.int32)
    val = _c(val, np.float64)
    x = _c(x, np.float64)
    n = len(rowptr) - 1
    y = np.empty(n, np.float64)
    if n:
        lib.o1_spmv_omp(n, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data,
                        x.ctypes.data, y.ctypes.data)
    return y


def o1_threads() -> int:
    """Threads o1_spmv_omp uses (OpenMP max threads)."""
    return int(_load().o1_omp_threads())


def o1_spmv_rows(rows, rowptr, col, val, x) -> np.ndarray:
    """O1 on a sample of rows (same loop, same order)."""
    lib = _load()
    rows = _c(rows, np.int64)
    rowptr = _c(rowptr, np.int64)
    col = _c(col, np.int32)
    val = _c(val, np.float64)
    x = _c(x, np.float64)
    y = np.empty(len(rows), np.float64)
    if len(rows):
        lib.o1_spmv_rows(len(rows), rows.ctypes.data, rowptr.ctypes.data, col.ctypes.data,
                         val.ctypes.data, x.ctypes.data, y.ctypes.data)
    return y


def o1_absdot(rowptr, col, val, x) -> np.ndarray:
    """s_i = sum_p |val[p] x[col[p]]| -- scale of the north_star tolerance."""
    lib = _load()
    rowptr = _c(rowptr, np.int64)
    col = _c(col, np.int32)
    val = _c(val, np.float64)
    x = _c(x, np.float64)
    n = len(rowptr) - 1
    s = np.empty(n, np.float64)
    if n:
        lib.o1_absdot(n, rowptr.ctypes.data, col.ctypes.data, val.ctypes.data,
                      x.ctypes.data, s.ctypes.data)
    return s


def csr_to_dense(rowptr, col, val, ncols) -> np.ndarray:
    n = len(rowptr) - 1
    A = np.zeros((n, ncols), np.float64)
    b = int(rowptr[0])
    for i in range(n):
        for p in range(int(rowptr[i]) - b, int(rowptr[i + 1]) - b):
            A[i, col[p]] += val[p]
    return A


def dense_bruteforce(A, x) -> np.ndarray:
    """y_i = sum_j A[i][j] * x[j], pure-Python loops (tiny inputs only)."""
    n, m = A.shape
    y = np.zeros(n, np.float64)
    for i in range(n):
        acc = 0.0
        for j in range(m):
            if A[i, j] != 0.0:
                acc = acc + A[i, j] * x[j]
        y[i] = acc
    return y
