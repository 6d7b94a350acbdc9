"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no partition, no halo, no
product): it only produces global CSR matrices / vectors from a counter-based
RNG keyed by *global* row/column ids, so any rank can generate exactly its own
rows and the oracle can generate the identical global matrix with no
communication (SURVEY.md §8(d) "Generators").

Recipes (DESIGN.md §3 restates them):

* G1 ``stencil(kind, dims)`` -- graph Laplacian on a regular grid, natural
  ordering ``idx = i + mx*j + mx*my*k`` (i fastest), columns ascending in each
  row, Dirichlet-truncated (out-of-domain neighbours dropped, diagonal kept).
  Values: 5-pt 4/-1, 7-pt 6/-1, 27-pt 26/-1.
* G2 ``powerlaw(n)`` -- row length ``L_i = min(4096, floor(8.25 * u_i^-1/2))``
  (discrete Pareto alpha=2, min 8, cap 4096 per Q11); diagonal always present;
  each other entry: with prob. 0.75 ``j = clamp(i + U[-n/16, n/16])`` else
  ``j = U[0, n)``; duplicates resampled so a row has exactly ``L_i`` distinct
  sorted columns.  Float values U[-1,1); exact mode integers in [-8,8]\\{0}.
* x: float mode U[-1,1) keyed by (seed, j); exact mode integers in [-16,16]
  (Q23).

Seeds: matrix 2203, x 2530.
"""
from __future__ import annotations

import numpy as np

SEED_MATRIX = 2203
SEED_X = 2530

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_u64(seed: int, stream: int, a, b=0) -> np.ndarray:
    """Counter-based 64-bit draw keyed by (seed, stream, a, b)."""
    key = splitmix64(np.uint64((seed * 0x100000001B3 + stream * 0x9E37) & 0xFFFFFFFFFFFFFFFF))
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64(splitmix64(key ^ a) + b * np.uint64(0xD1B54A32D192ED03))


def u01(bits: np.ndarray) -> np.ndarray:
    """uint64 -> float64 uniform in [0,1) using the top 53 bits."""
    return (bits >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# --------------------------------------------------------------------------- x
def x_values(n_global_range, seed: int = SEED_X, exact: bool = False,
             dtype=np.float64) -> np.ndarray:
    """x_j for global ids j in ``range(lo, hi)`` (pass a (lo, hi) tuple)."""
    lo, hi = n_global_range
    j = np.arange(lo, hi, dtype=np.uint64)
    bits = counter_u64(seed, 1, j)
    if exact:
        v = (bits % np.uint64(33)).astype(np.int64) - 16
        return v.astype(dtype)
    return (2.0 * u01(bits) - 1.0).astype(dtype)


# ------------------------------------------------------------------- stencils
_STENCIL_DIAG = {"5pt": 4.0, "7pt": 6.0, "27pt": 26.0}


def stencil_offsets(kind: str):
    """Neighbour offsets (dk, dj, di) of a stencil, in ascending linear order."""
    if kind == "5pt":
        offs = [(0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0)]
    elif kind == "7pt":
        offs = [(-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0),
                (0, 0, 1), (0, 1, 0), (1, 0, 0)]
    elif kind == "27pt":
        offs = [(dk, dj, di) for dk in (-1, 0, 1) for dj in (-1, 0, 1) for di in (-1, 0, 1)]
    else:
        raise ValueError(f"unknown stencil kind {kind!r}")
    return offs


def stencil_dims(kind: str, m: int, mz: int | None = None):
    """Grid dims (mx, my, mz) of an m-sized stencil (2D for 5pt)."""
    if kind == "5pt":
        return (m, m if mz is None else mz, 1)
    return (m, m, m if mz is None else mz)


def stencil(kind: str, dims, row_range=None, dtype=np.float64, chunk: int = 1 << 20):
    """Rows ``row_range=(lo, hi)`` of the stencil matrix on grid ``dims``.

    Returns (rowptr int64[n_r+1] starting at 0, col int32[nnz], val dtype[nnz]).
    """
    mx, my, mz = dims
    n = mx * my * mz
    lo, hi = (0, n) if row_range is None else row_range
    offs = stencil_offsets(kind)
    lin = np.array([dk * mx * my + dj * mx + di for dk, dj, di in offs], dtype=np.int64)
    order = np.argsort(lin, kind="stable")
    offs = [offs[t] for t in order]
    lin = lin[order]
    diag = _STENCIL_DIAG[kind]
    cvals = np.array([diag if o == (0, 0, 0) else -1.0 for o in offs], dtype=np.float64)
    rowptr_parts, col_parts, val_parts = [np.zeros(1, np.int64)], [], []
    base = 0
    for c0 in range(lo, hi, chunk):
        c1 = min(hi, c0 + chunk)
        r = np.arange(c0, c1, dtype=np.int64)
        i = r % mx
        j = (r // mx) % my
        k = r // (mx * my)
        valid = np.empty((c1 - c0, len(offs)), dtype=bool)
        for t, (dk, dj, di) in enumerate(offs):
            valid[:, t] = ((i + di >= 0) & (i + di < mx) & (j + dj >= 0) & (j + dj < my)
                           & (k + dk >= 0) & (k + dk < mz))
        cnt = valid.sum(axis=1)
        cols = (r[:, None] + lin[None, :])[valid]
        vals = np.broadcast_to(cvals, valid.shape)[valid]
        rowptr_parts.append(base + np.cumsum(cnt))
        base += int(cnt.sum())
        col_parts.append(cols.astype(np.int32))
        val_parts.append(vals.astype(dtype))
    rowptr = np.concatenate(rowptr_parts)
    col = np.concatenate(col_parts) if col_parts else np.zeros(0, np.int32)
    val = np.concatenate(val_parts) if val_parts else np.zeros(0, dtype)
    return rowptr, col, val


def blocked_index(dims, pgrid):
    """3D domain decomposition numbering (NEXT-4): the grid is cut into
    px x py x pz equal blocks, rank R = bx + px*(by + py*bz) owns block
    (bx, by, bz), and its points are numbered contiguously (x fastest) from
    R * block volume.  Returns new_index(natural linear index array)."""
    mx, my, mz = dims
    px, py, pz = pgrid
    if mx % px or my % py or mz % pz:
        raise ValueError("grid dims must be divisible by the process grid")
    bx, by, bz = mx // px, my // py, mz // pz
    vol = bx * by * bz

    def new_index(nat):
        nat = np.asarray(nat, np.int64)
        i, j, k = nat % mx, (nat // mx) % my, nat // (mx * my)
        R = i // bx + px * (j // by + py * (k // bz))
        return R * vol + (i % bx) + bx * ((j % by) + by * (k % bz))

    return new_index


def stencil_blocked(kind: str, dims, pgrid, row_range=None, dtype=np.float64):
    """Rows ``row_range`` of the stencil matrix on ``dims`` renumbered by
    ``blocked_index`` (P A P^T): with the library's even row partition over
    px*py*pz ranks every rank owns one block, and its peers sit at rank
    offsets +-1 (x), +-px (y), +-px*py (z) for a 7-pt stencil -- one
    per-destination exchange vertex set per face of the block ("3D halo
    exchange ... per dimension").  Columns ascending per row."""
    mx, my, mz = dims
    px, py, pz = pgrid
    n = mx * my * mz
    bx, by, bz = mx // px, my // py, mz // pz
    vol = bx * by * bz
    new_index = blocked_index(dims, pgrid)
    lo, hi = (0, n) if row_range is None else row_range
    r = np.arange(lo, hi, dtype=np.int64)                 # new row ids
    R, loc = r // vol, r % vol
    i = (R % px) * bx + loc % bx
    j = ((R // px) % py) * by + (loc // bx) % by
    k = (R // (px * py)) * bz + loc // (bx * by)
    offs = stencil_offsets(kind)
    diag = _STENCIL_DIAG[kind]
    cols = np.full((len(r), len(offs)), -1, np.int64)
    vals = np.zeros((len(r), len(offs)), np.float64)
    for t, (dk, dj, di) in enumerate(offs):
        ok = ((i + di >= 0) & (i + di < mx) & (j + dj >= 0) & (j + dj < my) & (k + dk >= 0) & (k + dk < mz))
        nat = (i + di) + mx * ((j + dj) + my * (k + dk))
        cols[ok, t] = new_index(nat[ok])
        vals[ok, t] = diag if (dk, dj, di) == (0, 0, 0) else -1.0
    order = np.argsort(np.where(cols < 0, np.iinfo(np.int64).max, cols), axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, 1)
    vals = np.take_along_axis(vals, order, 1)
    valid = cols >= 0
    rowptr = np.concatenate([[0], np.cumsum(valid.sum(1))]).astype(np.int64)
    return rowptr, cols[valid].astype(np.int32), vals[valid].astype(dtype)


# ------------------------------------------------------------------ power-law
POWERLAW_C = 8.25
POWERLAW_CAP = 4096


def powerlaw_row_lengths(n: int, rows: np.ndarray, seed: int = SEED_MATRIX,
                         cap: int = POWERLAW_CAP) -> np.ndarray:
    u = 1.0 - u01(counter_u64(seed, 2, rows))  # (0, 1]
    L = np.floor(POWERLAW_C / np.sqrt(u))
    return np.minimum(np.minimum(L, cap), n).astype(np.int64)


_GENC = None


def _genc():
    """The C twin of powerlaw_numpy (gen/genc.c), or None if not built."""
    global _GENC
    if _GENC is None:
        import ctypes
        import os
        so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgenc.so")
        if not os.path.exists(so):
            return None
        lib = ctypes.CDLL(so)
        P, I64 = ctypes.c_void_p, ctypes.c_int64
        lib.powerlaw_lengths.argtypes = [I64, I64, I64, ctypes.c_uint64, I64, P]
        lib.powerlaw_lengths.restype = I64
        lib.powerlaw_fill.argtypes = [I64, I64, I64, ctypes.c_uint64, ctypes.c_int, P, P, P]
        lib.powerlaw_fill.restype = ctypes.c_int
        _GENC = lib
    return _GENC


def powerlaw(n: int, row_range=None, seed: int = SEED_MATRIX, exact: bool = False,
             dtype=np.float64, cap: int = POWERLAW_CAP):
    """Rows ``row_range`` of the G2 power-law matrix (module docstring); uses
    the C twin when built (identical output, tests/test_gen.py)."""
    lib = _genc()
    if lib is None:
        return powerlaw_numpy(n, row_range, seed, exact, dtype, cap)
    lo, hi = (0, n) if row_range is None else row_range
    lens = np.empty(hi - lo, np.int64)
    tot = lib.powerlaw_lengths(n, lo, hi, seed, cap, lens.ctypes.data) if hi > lo else 0
    rowptr = np.zeros(hi - lo + 1, np.int64)
    np.cumsum(lens, out=rowptr[1:])
    col = np.empty(tot, np.int32)
    val = np.empty(tot, np.float64)
    if hi > lo and lib.powerlaw_fill(n, lo, hi, seed, int(exact), rowptr.ctypes.data,
                                     col.ctypes.data, val.ctypes.data) != 0:
        raise MemoryError("powerlaw_fill")
    return rowptr, col, val.astype(dtype, copy=False)


def powerlaw_numpy(n: int, row_range=None, seed: int = SEED_MATRIX, exact: bool = False,
                   dtype=np.float64, cap: int = POWERLAW_CAP, chunk: int = 1 << 18):
    """Rows ``row_range`` of the G2 power-law matrix (see module docstring).

    Candidate slots s = 0, 1, 2, ... of row i are drawn from the counter RNG
    keyed (seed, i, s); a row keeps the first ``L_i - 1`` distinct
    off-diagonal candidates in slot order, so the result depends only on
    (seed, i), never on the chunking or the row range.
    """
    lo, hi = (0, n) if row_range is None else row_range
    rp, cp, vp = [np.zeros(1, np.int64)], [], []
    base = 0
    w = max(1, n // 16)
    for c0 in range(lo, hi, chunk):
        c1 = min(hi, c0 + chunk)
        rows = np.arange(c0, c1, dtype=np.int64)
        L = powerlaw_row_lengths(n, rows, seed, cap)
        need = L - 1  # off-diagonal entries per row
        fin_r, fin_c = [rows], [rows]  # the diagonal
        kept_r = np.zeros(0, np.int64)
        kept_c = np.zeros(0, np.int64)
        have = np.zeros(len(rows), np.int64)
        slot0 = np.zeros(len(rows), np.int64)
        active = np.nonzero(need > 0)[0]
        rnd = 0
        while len(active):
            m = need[active] - have[active]
            m = m + (m >> 1) + 4
            tot = int(m.sum())
            rr = np.repeat(active, m)
            starts = np.repeat(np.cumsum(m) - m, m)
            slot = slot0[rr] + (np.arange(tot) - starts)
            grow = rows[rr]
            b1 = counter_u64(seed, 3, grow, slot)
            b2 = counter_u64(seed, 4, grow, slot)
            near = u01(b1) < 0.75
            ub = u01(b2)
            d = np.floor(ub * (2 * w + 1)).astype(np.int64) - w
            far = np.floor(ub * n).astype(np.int64)
            cand = np.where(near, np.clip(grow + d, 0, n - 1), far)
            slot0[active] += m
            kr = np.concatenate([kept_r, grow])   # kept entries precede new slots
            kc = np.concatenate([kept_c, cand])
            nd = kc != kr
            kr, kc = kr[nd], kc[nd]
            _, first = np.unique((kr - c0) * n + kc, return_index=True)
            first.sort()
            kr, kc = kr[first], kc[first]
            ridx = kr - c0
            srt = np.argsort(ridx, kind="stable")
            rs = ridx[srt]
            bnd = np.r_[0, np.nonzero(np.diff(rs))[0] + 1] if len(rs) else np.zeros(0, np.int64)
            runlen = np.diff(np.r_[bnd, len(rs)])
            pos = np.empty(len(kr), np.int64)
            pos[srt] = np.arange(len(rs)) - np.repeat(bnd, runlen)
            keep = pos < need[ridx]
            kr, kc = kr[keep], kc[keep]
            have[active] = np.bincount(kr - c0, minlength=len(rows))[active]
            done = have[kr - c0] == need[kr - c0]
            fin_r.append(kr[done])
            fin_c.append(kc[done])
            kept_r, kept_c = kr[~done], kc[~done]
            active = np.nonzero(have < need)[0]
            rnd += 1
            if rnd > 64:
                raise RuntimeError("power-law generator failed to converge")
        allr = np.concatenate(fin_r)
        allc = np.concatenate(fin_c)
        o = np.argsort((allr - c0) * n + allc)
        allr, allc = allr[o], allc[o]
        cnt = np.bincount(allr - c0, minlength=len(rows))
        assert np.array_equal(cnt, L)
        pos_in_row = np.arange(len(allr)) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        vb = counter_u64(seed, 5, allr, pos_in_row)
        if exact:
            t = (vb % np.uint64(16)).astype(np.int64)
            vals = np.where(t < 8, t - 8, t - 7).astype(np.float64)
        else:
            vals = 2.0 * u01(vb) - 1.0
        rp.append(base + np.cumsum(cnt))
        base += int(cnt.sum())
        cp.append(allc.astype(np.int32))
        vp.append(vals.astype(dtype))
    rowptr = np.concatenate(rp)
    col = np.concatenate(cp) if cp else np.zeros(0, np.int32)
    val = np.concatenate(vp) if vp else np.zeros(0, dtype)
    return rowptr, col, val


# ------------------------------------------------------ paper replica (G3)
def banded(n: int = 150000, nnz: int = 1500000, half_bw: int | None = None,
           seed: int = SEED_MATRIX, exact: bool = False, dtype=np.float64):
    """The paper's input: band-diagonal n x n, `nnz` distinct cells
    uniform within the band |i - j| <= half_bw (reading R-Q20: "bandwidth
    150000/4" = half-bandwidth n/4), values U[-1,1) (exact: [-8,8] minus 0).
    Global generation (the whole matrix is small); slice rows per rank."""
    b = n // 4 if half_bw is None else half_bw
    cells = []
    have = 0
    draw = 0
    seen = set()
    while have < nnz:
        m = int((nnz - have) * 1.2) + 1024
        k = np.arange(draw, draw + m, dtype=np.uint64)
        draw += m
        i = (u01(counter_u64(seed, 8, k)) * n).astype(np.int64)
        d = (u01(counter_u64(seed, 9, k)) * (2 * b + 1)).astype(np.int64) - b
        j = i + d
        ok = (j >= 0) & (j < n)
        key = (i * n + j)[ok]
        _, first = np.unique(key, return_index=True)
        for kk in key[np.sort(first)]:
            if kk not in seen:
                seen.add(int(kk))
                cells.append(int(kk))
                have += 1
                if have == nnz:
                    break
    cells = np.sort(np.array(cells, np.int64))
    rows, cols = cells // n, cells % n
    rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rowptr[1:])
    vb = counter_u64(seed, 10, cells.astype(np.uint64))
    if exact:
        t = (vb % np.uint64(16)).astype(np.int64)
        vals = np.where(t < 8, t - 8, t - 7).astype(np.float64)
    else:
        vals = 2.0 * u01(vb) - 1.0
    return rowptr, cols.astype(np.int32), vals.astype(dtype)


# -------------------------------------------------------------- small randoms
def random_csr(n: int, density: float, seed: int, exact: bool = True,
               ncols: int | None = None, dtype=np.float64, empty_rows=(), dense_rows=()):
    """Small random CSR for tests (rows may be empty / dense)."""
    ncols = n if ncols is None else ncols
    rp, cols, vals = [0], [], []
    for i in range(n):
        if i in empty_rows:
            rp.append(rp[-1])
            continue
        bits = counter_u64(seed, 6, np.uint64(i), np.arange(ncols, dtype=np.uint64))
        pick = u01(bits) < density
        if i in dense_rows:
            pick[:] = True
        c = np.nonzero(pick)[0]
        vb = counter_u64(seed, 7, np.uint64(i), c.astype(np.uint64))
        if exact:
            t = (vb % np.uint64(16)).astype(np.int64)
            v = np.where(t < 8, t - 8, t - 7).astype(np.float64)
        else:
            v = 2.0 * u01(vb) - 1.0
        cols.append(c)
        vals.append(v)
        rp.append(rp[-1] + len(c))
    col = np.concatenate(cols).astype(np.int32) if cols else np.zeros(0, np.int32)
    val = np.concatenate(vals).astype(dtype) if vals else np.zeros(0, dtype)
    return np.array(rp, np.int64), col, val


# -------------------------------------------------------------- named configs
CONFIGS = {
    # name: (builder kwargs, default ranks) -- BASELINE.json configs[0..4]
    "c1": dict(kind="5pt", m=64, ranks=2),
    "c2": dict(kind="7pt", m=128, ranks=1),
    "c3": dict(kind="27pt", m=256, ranks=8),
    "c4": dict(kind="powerlaw", n=1 << 23, ranks=8),
    "c5": dict(kind="7pt", m=192, ranks=4),
    # NEXT-4: C5's grid in a 2 x 2 x 1 block decomposition
    "c5b": dict(kind="7pt", m=192, ranks=4, pgrid=(2, 2, 1)),
}


def config_matrix(name: str, row_range=None, exact: bool = False, dtype=np.float64, mz=None):
    c = CONFIGS[name]
    if c["kind"] == "powerlaw":
        return c["n"], powerlaw(c["n"], row_range, exact=exact, dtype=dtype)
    dims = stencil_dims(c["kind"], c["m"], mz)
    n = dims[0] * dims[1] * dims[2]
    if "pgrid" in c:
        return n, stencil_blocked(c["kind"], dims, c["pgrid"], row_range, dtype=dtype)
    return n, stencil(c["kind"], dims, row_range, dtype=dtype)
