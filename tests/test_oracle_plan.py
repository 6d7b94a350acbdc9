"""Pins for O2 (oracle/plan.py): partition, split/halo invariants, Appendix-B
closed forms, exchange consistency, rank-count invariance, deadlock rule."""
import os

import numpy as np
import pytest

import gen
from oracle import plan as O2
from oracle import schedules as S
from oracle import spmv as O1

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_partition_examples():
    assert O2.partition(10, 4) == [0, 3, 6, 8, 10]
    assert O2.partition(4096, 2) == [0, 2048, 4096]
    assert O2.partition(3, 5) == [0, 1, 2, 3, 3, 3]
    for n in (0, 1, 7, 100, 4097):
        for P in (1, 2, 3, 8):
            rb = O2.partition(n, P)
            sizes = np.diff(rb)
            assert rb[0] == 0 and rb[-1] == n
            assert sizes.max() - sizes.min() <= 1
            assert list(sizes) == sorted(sizes, reverse=True)


def _reassemble(pl, rowptr_g, col_g):
    """Map A_L and A_R back to global columns; must equal the input rows."""
    b, e = pl["row_begin"], pl["row_end"]
    n_r = e - b
    rows = [[] for _ in range(n_r)]
    for i in range(n_r):
        for p in range(pl["al_rowptr"][i], pl["al_rowptr"][i + 1]):
            rows[i].append((int(pl["al_src"][p]), int(pl["al_col"][p]) + b))
    for k, i in enumerate(pl["ar_rows"]):
        for p in range(pl["ar_rowptr"][k], pl["ar_rowptr"][k + 1]):
            rows[i].append((int(pl["ar_src"][p]), int(pl["halo_gid"][pl["ar_col"][p]])))
    for i in range(n_r):
        got = sorted(rows[i])
        want = [(p, int(col_g[p])) for p in range(rowptr_g[b + i], rowptr_g[b + i + 1])]
        assert got == want


MATS = {
    "rand50": lambda exact=False: (50, gen.random_csr(50, 0.15, seed=3, exact=exact,
                                                      empty_rows=(4, 9), dense_rows=(20,))),
    "5pt16": lambda exact=False: (256, gen.stencil("5pt", (16, 16, 1))),
    "pl2k": lambda exact=False: (2048, gen.powerlaw(2048, exact=exact)),
}


@pytest.mark.parametrize("mat", list(MATS))
@pytest.mark.parametrize("P", [1, 2, 3, 5, 8])
def test_split_invariants(mat, P):
    n, (rp, col, val) = MATS[mat]()
    plans = O2.plan_all(rp, col, n, P)
    tot_h = tot_s = 0
    for r, pl in enumerate(plans):
        _reassemble(pl, rp, col)
        nnz_r = rp[pl["row_end"]] - rp[pl["row_begin"]]
        assert len(pl["al_col"]) + len(pl["ar_col"]) == nnz_r
        h = pl["halo_gid"]
        assert np.all(np.diff(h) > 0)                     # R-Q4 ascending unique
        assert not np.any((h >= pl["row_begin"]) & (h < pl["row_end"]))
        assert np.all(np.diff(pl["ar_rows"]) > 0)         # R-Q6 ascending
        tot_h += len(h)
        tot_s += len(pl["pack_map"])
        for p in range(P):                                 # counts agree pairwise
            assert plans[p]["send_count"][r] == pl["recv_count"][p]
    assert tot_h == tot_s                                  # conservation


def test_partition_more_ranks_than_rows():
    n, (rp, col, val) = 5, gen.random_csr(5, 0.6, seed=9)
    plans = O2.plan_all(rp, col, n, 8)
    assert [pl["row_end"] - pl["row_begin"] for pl in plans] == [1, 1, 1, 1, 1, 0, 0, 0]
    x = gen.x_values((0, n))
    y = O2.simulate(plans, val, x, [(v,) for v in O2.paper_sequence_1()])
    y1 = O1.o1_spmv(rp, col, val, x)
    assert np.all(np.abs(y - y1) <= 1e-12 * O1.o1_absdot(rp, col, val, x))


def _closed_form(kind, m, P, cls):
    """Appendix B: link nnz to an adjacent layer: 5-pt m, 7-pt m^2,
    27-pt (3m-2)^2; h = |R| = m^(d-1) per neighbour."""
    link = {"5pt": m, "7pt": m * m, "27pt": (3 * m - 2) ** 2}[kind]
    layer = m if kind == "5pt" else m * m
    nb = 1 if cls == "end" else 2
    return nb * link, nb * layer, nb * layer


@pytest.mark.parametrize("kind,m,P", [("5pt", 16, 4), ("7pt", 8, 4), ("7pt", 12, 3),
                                      ("27pt", 8, 4), ("27pt", 6, 3)])
def test_stencil_halo_closed_forms_bruteforce(kind, m, P):
    dims = gen.stencil_dims(kind, m)
    n = dims[0] * dims[1] * dims[2]
    rp, col, val = gen.stencil(kind, dims)
    plans = O2.plan_all(rp, col, n, P)
    for r, pl in enumerate(plans):
        cls = "end" if r in (0, P - 1) else "interior"
        nnzR, h, R = _closed_form(kind, m, P, cls)
        assert (len(pl["ar_col"]), len(pl["halo_gid"]), len(pl["ar_rows"])) == (nnzR, h, R)


def test_stencil_halo_golden_full_size():
    """The full-size Appendix-B table agrees with the closed forms (the
    closed forms are themselves pinned by brute force above)."""
    for line in open(os.path.join(GOLDEN, "stencil_halo.txt")):
        if line.startswith("#") or not line.strip():
            continue
        kind, m, P, cls, nnzR, h, R = line.split()
        assert _closed_form(kind, int(m), int(P), cls) == (int(nnzR), int(h), int(R))
    # and the 5-pt 64^2 / 2-rank row by brute force (C1)
    n, (rp, col, val) = gen.config_matrix("c1")
    for pl in O2.plan_all(rp, col, n, 2):
        assert (len(pl["ar_col"]), len(pl["halo_gid"]), len(pl["ar_rows"])) == (64, 64, 64)


@pytest.mark.parametrize("mat", list(MATS))
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_exchange_consistency_and_rank_invariance(mat, P):
    for exact in (True, False):
        n, (rp, col, val) = MATS[mat](exact)
        x = gen.x_values((0, n), exact=exact)
        plans = O2.plan_all(rp, col, n, P)
        # exchange consistency: recvbuf == x_global[H_r] bitwise
        st_ops = [(v,) for v in O2.paper_sequence_1()]
        y = O2.simulate(plans, val, x, st_ops)
        y1 = O1.o1_spmv(rp, col, val, x)
        if exact:
            assert np.array_equal(y, y1)
        else:
            s = O1.o1_absdot(rp, col, val, x)
            assert np.all(np.abs(y - y1) <= 1e-12 * s)
        for pl in plans:
            xs = x[pl["row_begin"]:pl["row_end"]]
            # the pack map gathers exactly what the peers' halos need
            for d in range(P):
                so, c = pl["send_displ"][d], pl["send_count"][d]
                seg = xs[pl["pack_map"][so:so + c]]
                ro = plans[d]["recv_displ"][r_of(plans, pl)]
                want = x[plans[d]["halo_gid"][ro:ro + c]]
                assert np.array_equal(seg, want)


def r_of(plans, pl):
    return next(i for i, q in enumerate(plans) if q is pl)


def test_schedule_invariance_of_y():
    n, (rp, col, val) = MATS["pl2k"]()
    x = gen.x_values((0, n))
    plans = O2.plan_all(rp, col, n, 4)
    ys = set()
    for order in S.topological_orders(S.EDGES):
        y = O2.simulate(plans, val, x, [(v,) for v in order])
        ys.add(y.tobytes())
    assert len(ys) == 1


def test_deadlock_rule_matches_simulation():
    """R-Q13 pinned dynamically: over all 280 orders of SPEC's DAG, the static
    rule (a Wait before the matching Post) is exactly the set of orders whose
    lock-step SPMD simulation deadlocks."""
    n, (rp, col, val) = gen.config_matrix("c1")
    x = gen.x_values((0, n))
    plans = O2.plan_all(rp, col, n, 2)
    n_dead = 0
    for order in S.topological_orders(S.EDGES_A):
        pos = {v: i for i, v in enumerate(order)}
        static_dead = any(pos[u] > pos[v] for (u, v) in S.DEADLOCK_EDGES)
        try:
            O2.simulate(plans, val, x, [(v,) for v in order])
            dyn_dead = False
        except O2.Deadlock:
            dyn_dead = True
        assert static_dead == dyn_dead, order
        n_dead += dyn_dead
    assert n_dead == 280 - 96
