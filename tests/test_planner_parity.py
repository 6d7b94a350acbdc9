"""The library planner (host twin of dspmv_plan_create, same C++ code) is
bit-exact against the oracle's independent O2 planner: partition, halo lists,
counts, pack maps, A_L / A_R arrays and values."""
import numpy as np
import pytest

import gen
from oracle import plan as O2
from paper_2203_02530_b200 import dspmv as D

MATS = {
    "rand50": lambda: (50, gen.random_csr(50, 0.15, seed=3, exact=False,
                                          empty_rows=(4, 9), dense_rows=(20,))),
    "rand7": lambda: (7, gen.random_csr(7, 0.5, seed=5)),
    "5pt16": lambda: (256, gen.stencil("5pt", (16, 16, 1))),
    "7pt8x8x6": lambda: (384, gen.stencil("7pt", (8, 8, 6))),
    "27pt6": lambda: (216, gen.stencil("27pt", (6, 6, 6))),
    "pl3k": lambda: (3000, gen.powerlaw(3000)),
}


@pytest.mark.parametrize("n,P", [(0, 1), (1, 1), (10, 4), (4096, 2), (3, 5), (7077888, 4),
                                 (16777216, 8), (2 ** 31 - 1, 7)])
def test_partition_matches_oracle(n, P):
    assert list(D.dspmv_partition(n, P)) == O2.partition(n, P)


@pytest.mark.parametrize("mat", list(MATS))
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_plan_bit_exact_vs_oracle(mat, P):
    n, (rp, col, val) = MATS[mat]()
    ref = O2.plan_all(rp, col, n, P)
    hp = D.dspmv_plan_build_host(P, n, rp, col, val)
    try:
        for r in range(P):
            o = ref[r]
            ex = lambda w: D.dspmv_host_plan_export(hp, r, w)
            pairs = [(D.DSPMV_HALO_GID, "halo_gid"), (D.DSPMV_RECV_COUNTS, "recv_count"),
                     (D.DSPMV_RECV_DISPL, "recv_displ"), (D.DSPMV_SEND_COUNTS, "send_count"),
                     (D.DSPMV_SEND_DISPL, "send_displ"), (D.DSPMV_PACK_MAP, "pack_map"),
                     (D.DSPMV_AL_ROWPTR, "al_rowptr"), (D.DSPMV_AL_COL, "al_col"),
                     (D.DSPMV_AR_ROWS, "ar_rows"), (D.DSPMV_AR_ROWPTR, "ar_rowptr"),
                     (D.DSPMV_AR_COL, "ar_col")]
            for w, key in pairs:
                got, want = ex(w), np.asarray(o[key], np.int32)
                assert got.dtype == np.int32 and np.array_equal(got, want), (key, r)
            # values: the oracle carries source positions; gather bitwise
            assert np.array_equal(ex(D.DSPMV_AL_VAL).view(np.uint64),
                                  val[o["al_src"]].view(np.uint64))
            assert np.array_equal(ex(D.DSPMV_AR_VAL).view(np.uint64),
                                  val[o["ar_src"]].view(np.uint64))
            info = D.dspmv_host_plan_info(hp, r)
            assert info["row_begin"] == o["row_begin"] and info["row_end"] == o["row_end"]
            assert info["nnz_local"] == len(o["al_col"]) and info["nnz_remote"] == len(o["ar_col"])
            assert info["n_halo"] == len(o["halo_gid"]) and info["n_send"] == len(o["pack_map"])
    finally:
        D.dspmv_host_plan_destroy(hp)


def test_plan_fp32_values():
    n, (rp, col, val) = MATS["pl3k"]()
    v32 = val.astype(np.float32)
    hp = D.dspmv_plan_build_host(3, n, rp, col, v32, dtype=D.DSPMV_F32)
    ref = O2.plan_all(rp, col, n, 3)
    for r in range(3):
        assert np.array_equal(D.dspmv_host_plan_export(hp, r, D.DSPMV_AL_VAL), v32[ref[r]["al_src"]])
    D.dspmv_host_plan_destroy(hp)


def test_plan_rejects_bad_input():
    rp, col, val = gen.random_csr(10, 0.3, seed=1)
    bad = col.copy()
    bad[0] = 10                                   # column id >= n_global
    with pytest.raises(D.DspmvError) as e:
        D.dspmv_plan_build_host(2, 10, rp, bad, val)
    assert e.value.status == D.DSPMV_ERR_ARG
    bad[0] = -1
    with pytest.raises(D.DspmvError):
        D.dspmv_plan_build_host(2, 10, rp, bad, val)
    with pytest.raises(D.DspmvError) as e:
        D.dspmv_plan_build_host(2, 2 ** 31, np.zeros(1, np.int64), np.zeros(0, np.int32))
    assert e.value.status == D.DSPMV_ERR_RANGE
    rp2 = rp.copy()
    rp2[3], rp2[4] = rp2[4], rp2[3] - 1           # non-monotone rowptr
    if rp2[3] > rp2[4]:
        with pytest.raises(D.DspmvError):
            D.dspmv_plan_build_host(1, 10, rp2, col, val)


def test_stencil_appendix_b_counts_library():
    """Appendix B via the library planner at a size the oracle cannot do
    quickly in pure Python: 27-pt 64^3 over 8 ranks."""
    m, P = 64, 8
    rp, col, val = gen.stencil("27pt", (m, m, m))
    hp = D.dspmv_plan_build_host(P, m ** 3, rp, col)
    for r in range(P):
        i = D.dspmv_host_plan_info(hp, r)
        nb = 1 if r in (0, P - 1) else 2
        assert (i["nnz_remote"], i["n_halo"], i["n_remote_rows"]) == (
            nb * (3 * m - 2) ** 2, nb * m * m, nb * m * m)
    D.dspmv_host_plan_destroy(hp)


def test_pack_alias_detection_host():
    """the contiguous-alias option applies exactly when every
    destination's send list is a run of consecutive rows -- stencil slabs
    (whole planes) yes, the power-law matrix no -- checked against the
    oracle planner's pack maps."""
    from oracle import plan as O2
    from paper_2203_02530_b200 import dspmv as D
    cases = [("7pt", 12 ** 3, gen.stencil("7pt", (12, 12, 12)), (2, 3, 4)),
             ("27pt", 10 ** 3, gen.stencil("27pt", (10, 10, 10)), (2, 5)),
             ("pl", 6000, gen.powerlaw(6000), (2, 3))]
    for name, n, (rp, col, _), Ps in cases:
        for P in Ps:
            hp = D.dspmv_plan_build_host(P, n, rp, col)
            try:
                plans = O2.plan_all(rp, col, n, P)
                for r in range(P):
                    pm = np.asarray(plans[r]["pack_map"])
                    sc = np.asarray(plans[r]["send_count"])
                    sd = np.concatenate([[0], np.cumsum(sc)])
                    want = int(len(pm) > 0 and all(np.all(np.diff(pm[sd[q]:sd[q + 1]]) == 1)
                                                    for q in range(P) if sc[q] > 0))
                    assert D.dspmv_host_plan_info(hp, r)["pack_alias"] == want, (name, P, r)
                    if name != "pl" and len(pm):
                        assert want == 1
            finally:
                D.dspmv_host_plan_destroy(hp)
