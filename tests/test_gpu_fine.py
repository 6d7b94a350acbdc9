"""GPU parity of per-destination schedules (NEXT-3 (i), DESIGN.md
R-N4): Pack[d] / PostSend[d] / ... / Unpack[e] vertices executed through the
C ABI on LOCAL groups (both exchanges), against the oracle's lock-step
simulation of the same schedule; plus coverage errors and the PUT flag
symmetry on a one-directional pattern."""
import random

import numpy as np
import pytest
import torch

import gen
from oracle import plan as O2
from oracle import schedules as S
from oracle import spmv as O1
from paper_2203_02530_b200 import dspmv as D
from tests.gpu_helpers import LocalRun, oracle_ops_to_lib, within_tol

pytestmark = pytest.mark.gpu


def _rand_topo(V, E, rng):
    pred = {v: {u for u, w in E if w == v} for v in V}
    done, out = set(), []
    while len(out) < len(V):
        v = rng.choice([v for v in V if v not in done and pred[v] <= done])
        out.append(v)
        done.add(v)
    return out


def _offsets(plans):
    P = len(plans)
    return sorted({q - r for r in range(P) for q in range(P) if plans[r]["send_count"][q] > 0}
                  | {r - q for r in range(P) for q in range(P) if plans[r]["send_count"][q] > 0})


def _build(name, exact):
    if name == "c1-P3":
        n, (rp, col, val) = gen.config_matrix("c1", exact=exact)
        return n, rp, col, val, 3
    if name == "banded-P6":
        rp, col, val = gen.banded(3000, 30000, 750, exact=exact)
        return 3000, rp, col, val, 6
    # NEXT-4: 7-pt on a 2x2x2 block decomposition, per-dimension vertices
    rp, col, val = gen.stencil_blocked("7pt", (16, 16, 16), (2, 2, 2))
    return 16 ** 3, rp, col, val, 8


@pytest.mark.parametrize("exchange", [D.DSPMV_EXCHANGE_COPY, D.DSPMV_EXCHANGE_PUT], ids=["copy", "put"])
@pytest.mark.parametrize("name", ["c1-P3", "banded-P6", "blocked3d-P8"])
def test_fine_schedules_vs_oracle(name, exchange):
    """Random per-destination traversals on 2 streams: y bitwise identical
    across schedules (ticket combine) and equal to the oracle's simulation of
    the same per-destination schedule (exact mode bitwise, else tolerance)."""
    n, rp, col, val, P = _build(name, False)
    plans = O2.plan_all(rp, col, n, P)
    offs = _offsets(plans)
    if name.startswith("blocked"):
        assert offs == [-4, -2, -1, 1, 2, 4]
    V, E, _ = S.fine_dag(offs)
    rng = random.Random(P)
    x = gen.x_values((0, n))
    s_abs = O1.o1_absdot(rp, col, val, x)
    run = LocalRun(n, rp, col, val, P, exchange=exchange)
    try:
        first = None
        for i in range(12):
            order = _rand_topo(V, E, rng)
            ops = S.derive(order, {v: rng.randrange(2) for v in V if S.base(v) in S.GPU_VERTICES})
            yref = O2.simulate(plans, val, x, ops)
            assert not np.isnan(yref).any()
            ss = run.schedule(oracle_ops_to_lib(ops))
            y = run.apply(ss, x, reps=3)
            assert within_tol(y, yref, s_abs, 1e-12), i
            if first is None:
                first = y
            assert np.array_equal(y.view(np.uint64), first.view(np.uint64))
    finally:
        run.close()
    # exact mode: bitwise against the simulation
    n, rp, col, val, P = _build(name, True)
    xe = gen.x_values((0, n), exact=True)
    ops = S.derive(_rand_topo(V, E, rng), {v: 1 for v in V})
    run = LocalRun(n, rp, col, val, P, exchange=exchange)
    try:
        y = run.apply(run.schedule(oracle_ops_to_lib(ops)), xe, reps=2)
    finally:
        run.close()
    assert np.array_equal(y, O2.simulate(O2.plan_all(rp, col, n, P), val, xe, ops))


def test_fine_schedule_must_cover_every_peer():
    n, (rp, col, val) = gen.config_matrix("c1")
    run = LocalRun(n, rp, col, val, 3)
    try:
        V, E, _ = S.fine_dag([1])                  # no exchange with rank offset -1
        ops = oracle_ops_to_lib(S.derive(S.topological_orders(E, V)[0], {v: 0 for v in V}))
        with pytest.raises(D.DspmvError, match="offset"):
            D.dspmv_schedule_create(run.plans[1], ops, 1)
    finally:
        run.close()


@pytest.mark.parametrize("fine", [False, True])
def test_put_one_directional_pattern(fine):
    """Lower-triangular banded matrix: rank r only receives from r-1.  The PUT
    exchange still pairs the epoch flags both ways (the receiver acks), so
    results stay exact over many applies with changing x."""
    n, P = 4000, 4
    rp, col, val = gen.banded(n, 20000, 900, exact=True)
    keep_rows = []
    for i in range(n):
        a, b = rp[i], rp[i + 1]
        m = col[a:b] <= i
        keep_rows.append((col[a:b][m], val[a:b][m]))
    rp = np.concatenate([[0], np.cumsum([len(c) for c, _ in keep_rows])]).astype(np.int64)
    col = np.concatenate([c for c, _ in keep_rows]).astype(np.int32)
    val = np.concatenate([v for _, v in keep_rows])
    plans = O2.plan_all(rp, col, n, P)
    assert all(plans[r]["send_count"][q] == 0 for r in range(P) for q in range(r + 1))
    if fine:
        V, E, _ = S.fine_dag(_offsets(plans))
        ops = oracle_ops_to_lib(S.derive(S.topological_orders(E, V)[-1], {v: 0 for v in V}))
    else:
        ops = oracle_ops_to_lib(S.derive(S.topological_orders(S.EDGES)[0], dict.fromkeys(S.GPU_VERTICES, 0)))
    run = LocalRun(n, rp, col, val, P, exchange=D.DSPMV_EXCHANGE_PUT)
    try:
        ss = run.schedule(ops)
        for k in range(5):
            x = gen.x_values((0, n), exact=True) + k
            y = run.apply(ss, x)
            assert np.array_equal(y, O1.o1_spmv(rp, col, val, x)), k
    finally:
        run.close()


def test_fine_schedule_graph_mode_single_rank():
    """A per-destination schedule on one rank (no peers) runs host-driven and
    as a captured graph with the same bits."""
    n, (rp, col, val) = gen.config_matrix("c1")
    x = torch.from_numpy(gen.x_values((0, n))).cuda()
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val)
    V, E, _ = S.fine_dag([-1, 1])
    ops = oracle_ops_to_lib(S.derive(S.topological_orders(E, V)[7], {v: i % 2 for i, v in enumerate(V)}))
    s = D.dspmv_schedule_create(plan, ops, 2)
    try:
        y1 = torch.empty_like(x)
        y2 = torch.empty_like(x)
        D.dspmv_apply(s, x, y1)
        st = torch.cuda.Stream()
        D.dspmv_apply_graph(s, x, y2, st)
        st.synchronize()
        assert torch.equal(y1, y2)
        assert np.array_equal(y1.cpu().numpy(), O1.o1_spmv(rp, col, val, x.cpu().numpy()))
    finally:
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
