"""The planner's device row layout (host-only hook): S/V split, row classes
(2^c lanes per row), windowed stable class partition, block limits, warp
bounds -- the invariants the row-block kernel relies on (K1)."""
import numpy as np
import pytest

import gen
from paper_2203_02530_b200 import dspmv as D

TILE = {0: 2048, 1: 1024, 2: 2048, 3: 1024, 4: 768, 5: 4096, 6: 4096, 7: 3072}
ROWMAX = {0: 256, 1: 128, 2: 256, 3: 128, 4: 96, 5: 256, 6: 128, 7: 96}
WARPS = {0: 8, 1: 4, 2: 8, 3: 4, 4: 3, 5: 8, 6: 4, 7: 3}
LANE_MAX = {0: 8, 1: 8, 2: 8, 3: 8, 4: 8, 5: 32, 6: 32, 7: 32}


def _cls(length, cfg):
    if length <= LANE_MAX[cfg]:
        return 0
    c = 0
    while c < 5 and length > (8 << c):
        c += 1
    return c


MATS = {
    "pl": lambda: gen.powerlaw(20000)[0],
    "7pt": lambda: gen.stencil("7pt", (20, 20, 20))[0],
    "27pt": lambda: gen.stencil("27pt", (14, 14, 14))[0],
    "rand": lambda: gen.random_csr(600, 0.05, seed=2, empty_rows=(0, 5, 599), dense_rows=(7,))[0],
    "empty": lambda: np.zeros(100, np.int64),
}


@pytest.mark.parametrize("mat", list(MATS))
@pytest.mark.parametrize("cfg", [-1, 0, 3, 5, 6])
@pytest.mark.parametrize("vthr", [-1, 0, 64])
def test_layout_invariants(mat, cfg, vthr):
    rp = MATS[mat]()
    n = len(rp) - 1
    L = np.diff(rp)
    s_rows, desc, v_rows, cu = D.dspmv_layout_host(rp, cfg=cfg, vthr=vthr)
    thr = 256 if vthr < 0 else vthr
    # S / V split and coverage (every row exactly once)
    assert sorted(np.concatenate([s_rows, v_rows]).tolist()) == list(range(n))
    assert np.all(L[s_rows] <= thr) and np.all(L[v_rows] > thr)
    assert np.all(np.diff(v_rows) > 0)
    cls = np.array([_cls(l, cu) for l in L[s_rows]])
    # windowed stable partition: inside each 4096-row window, classes ascend and
    # rows of one class keep ascending order; windows cover S rows in order
    for w0 in range(0, len(s_rows), 4096):
        w = s_rows[w0:w0 + 4096]
        c = cls[w0:w0 + 4096]
        assert np.all(np.diff(c) >= 0)
        for k in np.unique(c):
            assert np.all(np.diff(w[c == k]) > 0)
        if w0:
            assert w.min() > s_rows[:w0].max()
    # blocks: contiguous, one class, nnz <= tile, rows <= rowmax >> c, warp bounds
    prefix = np.concatenate([[0], np.cumsum(L[s_rows])])
    r_next = 0
    for d in desc:
        r0, r1, p0, p1, fl = d[:5]
        c = fl >> 8
        assert r0 == r_next and r1 > r0
        r_next = r1
        assert p0 == prefix[r0] and p1 == prefix[r1]
        assert np.all(cls[r0:r1] == c)
        assert p1 - p0 <= TILE[cu] and r1 - r0 <= max(1, ROWMAX[cu] >> c)
        W = WARPS[cu]
        wb = d[5:6 + W]
        assert wb[0] == r0 and wb[-1] == r1 and np.all(np.diff(wb) >= 0)
        assert np.all(np.diff(wb) <= max(1, 32 >> c) + (32 >> c))
    assert r_next == len(s_rows)


def test_auto_config_choice():
    assert D.dspmv_layout_host(gen.stencil("7pt", (16, 16, 16))[0])[3] == 3
    assert D.dspmv_layout_host(gen.stencil("27pt", (16, 16, 16))[0])[3] == 5
    assert D.dspmv_layout_host(gen.stencil("27pt", (16, 16, 16))[0], dtype=D.DSPMV_F32)[3] == 6
    assert D.dspmv_layout_host(gen.powerlaw(20000)[0])[3] == 3
    assert D.dspmv_layout_host(gen.stencil("7pt", (16, 16, 16))[0], dtype=D.DSPMV_F32)[3] == 0


@pytest.mark.parametrize("mat", list(MATS))
@pytest.mark.parametrize("vthr", [-1, 0, 16, 1024])
def test_stream_layout_invariants(mat, vthr):
    """CSR-stream tiles (K1b): S rows (<= min(vthr, 256) nnz) in
    matrix order, cut greedily into contiguous row-aligned tiles of <= 256
    nnz and <= 64 rows that cover every S row once; the rest are V rows."""
    rp = MATS[mat]()
    lens = np.diff(rp)
    cap = min(256 if vthr < 0 else vthr, 256)
    tiles, v_rows, _ = D.dspmv_stream_layout_host(rp, vthr=vthr)
    s_rows = np.flatnonzero(lens <= cap)
    assert np.array_equal(v_rows, np.flatnonzero(lens > cap))
    ns = len(s_rows)
    if ns == 0:
        assert len(tiles) == 0
        return
    assert tiles[0, 0] == 0 and tiles[-1, 1] == ns
    assert np.array_equal(tiles[1:, 0], tiles[:-1, 1])          # contiguous, no gap or overlap
    slen = lens[s_rows]
    cum = np.concatenate([[0], np.cumsum(slen)])
    for r0, r1 in tiles:
        assert r1 > r0 and r1 - r0 <= 64
        assert cum[r1] - cum[r0] <= 256
        if r1 < ns:  # greedy: the next row would break a limit
            assert r1 - r0 == 64 or cum[r1 + 1] - cum[r0] > 256


def test_stream_kernel_auto_choice_host():
    """Row-length coefficient of variation > 0.5 selects CSR-stream: the
    power-law generator (G2) yes, stencils no; forced choices win."""
    pick = lambda rp, k=D.DSPMV_SKERNEL_AUTO: D.dspmv_stream_layout_host(rp, s_kernel=k)[2]
    pl = MATS["pl"]()
    assert pick(pl)
    assert not pick(MATS["7pt"]()) and not pick(MATS["27pt"]())
    assert not pick(gen.stencil("7pt", (16, 16, 16))[0]) and not pick(gen.config_matrix("c1")[1][0])
    assert not pick(pl, D.DSPMV_SKERNEL_BLOCK)
    assert pick(MATS["7pt"](), D.DSPMV_SKERNEL_STREAM)
    lens = np.diff(pl).astype(float)
    lens = lens[lens <= 256]
    assert lens.std() > 0.5 * lens.mean()   # the criterion, computed independently


@pytest.mark.parametrize("name", ["pl", "7pt", "27pt"])
@pytest.mark.parametrize("window", [-1, 32, 96, 4096])
def test_sell_layout_invariants(name, window):
    """Sliced form (DSPMV_SKERNEL_SELL, K1d): every S row (<= 256
    nnz) sits in exactly one lane; within a sort window rows are longest
    first; the lanes active at entry k are a prefix 0..m_k-1 and entry k of
    the slice is stored as their m_k consecutive values, each lane's entries
    in its row's CSR order; the stored entries are a permutation of the S
    group's; the work chunks cover the slices in order."""
    rp = MATS[name]()
    lens = np.diff(rp)
    s_rows = np.nonzero(lens <= 256)[0]
    L = D.dspmv_sell_layout_host(rp, window=window)
    base, row, ln, src, ch = L["base"], L["lane_row"], L["lane_len"], L["entry_src"], L["chunks"]
    ns = len(base) - 1
    sl = lens[s_rows]
    s_start = np.concatenate([[0], np.cumsum(sl)])
    assert sorted(row[row >= 0].tolist()) == list(range(len(s_rows)))
    assert np.array_equal(ln[row >= 0], sl[row[row >= 0]]) and np.all(ln[row < 0] == 0)
    assert np.all(np.diff(ln, axis=1) <= 0)                     # longest first within a slice
    assert base[0] == 0 and base[-1] == len(src) == sl.sum()
    assert np.array_equal(np.sort(src), np.arange(len(src)))    # a permutation of the S entries
    w = 256 if window == -1 else window
    for s in range(ns):
        q = base[s]
        for k in range(int(ln[s, 0])):
            act = ln[s] > k
            m = int(act.sum())
            assert np.all(act[:m]) and not np.any(act[m:])
            want = s_start[row[s, :m]] + k                      # entry k of each active lane's row
            assert np.array_equal(src[q:q + m], want)
            q += m
        assert q == base[s + 1]
    # window order: the S rows of window j are exactly S rows [j*w, (j+1)*w)
    win_of_slice = []
    for s in range(ns):
        r = row[s][row[s] >= 0]
        assert len(set((r // w).tolist())) == 1
        win_of_slice.append(int(r[0] // w))
    assert win_of_slice == sorted(win_of_slice)
    assert ch[0] == 0 and ch[-1] == ns and np.all(np.diff(ch) > 0)
