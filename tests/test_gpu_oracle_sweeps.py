"""GPU parity over the design spaces the bench and the MCTS actually run:
every orderable-sync schedule (R-N5, 4,780) and MCTS rollouts with real GPU
timing, each checked against the oracle O2 (P:273 y = y_L + y_R; P:430-434
syncs as insertions; P:460 SPMD), plus fp32 apply_host against O1."""
import time

import numpy as np
import pytest
import torch

import gen
from oracle import plan as O2
from oracle import schedules as S
from oracle import spmv as O1
from paper_2203_02530_b200 import dspmv as D
from paper_2203_02530_b200 import mcts as M
from paper_2203_02530_b200 import schedules as PS
from tests.gpu_helpers import LocalRun, oracle_ops_to_lib, within_tol

pytestmark = pytest.mark.gpu


def _lib_to_oracle(ops):
    """Library op array -> the oracle's tuple form (inverse of oracle_ops_to_lib)."""
    out = []
    for k, s, e, d in np.asarray(ops).tolist():
        if k == D.DSPMV_OP_EVENT_RECORD:
            out.append(("CER", s, e))
        elif k == D.DSPMV_OP_EVENT_SYNC:
            out.append(("CES", e))
        elif k == D.DSPMV_OP_STREAM_WAIT_EVENT:
            out.append(("CSWE", s, e))
        else:
            name = S.vname(S.VERTICES[k], d)
            out.append((name, s) if S.VERTICES[k] in S.GPU_VERTICES else (name,))
    return out


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "float"])
def test_every_orderable_schedule_c1_equals_o2(exact):
    """C1 (5-pt 64^2, 2 LOCAL ranks on cuda:0), all 4,780 orderable-sync
    schedules of the oracle's enumerator: the GPU y is bitwise identical
    across schedules (R-Q9) and equals O2 simulating that same schedule
    (exact mode bitwise, float mode within the north_star tolerance)."""
    n, (rp, col, val) = gen.config_matrix("c1")
    x = gen.x_values((0, n), exact=exact)
    plans = O2.plan_all(rp, col, n, 2)
    scale = O1.o1_absdot(rp, col, val, x)
    space = S.enumerate_orderable(2, S.EDGES)
    assert len(space) == 4780
    run = LocalRun(n, rp, col, val, 2)
    first = None
    try:
        for i, ops in enumerate(space):
            ss = run.schedule(oracle_ops_to_lib(ops))
            y = run.apply(ss, x)
            for s in ss:
                D.dspmv_schedule_destroy(s)
            run.scheds.pop()
            yref = O2.simulate(plans, val, x, ops)
            if exact:
                assert np.array_equal(y, yref), i
            else:
                assert within_tol(y, yref, scale, 1e-12), i
            if first is None:
                first = y
            assert np.array_equal(y.view(np.uint64), first.view(np.uint64)), i
    finally:
        run.close()


@pytest.mark.parametrize("space_name", ["coarse", "per-destination"])
def test_mcts_rollouts_on_gpu_equal_o2(space_name):
    """NEXT-1 with the real executor: 50 MCTS iterations over the orderable
    space (coarse DAG, or the per-destination DAG of offsets {-1, +1},
    P:281-284), every rollout timed on cuda:0 (2 LOCAL ranks, C1) with the
    paper's repeat-until protocol shortened to 2 ms, and every rollout's y
    checked against O2 bitwise (exact mode)."""
    n, (rp, col, val) = gen.config_matrix("c1")
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, 2)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    sp = PS.COARSE if space_name == "coarse" else PS.Space([-1, 1])
    run = LocalRun(n, rp, col, val, 2)
    xs, ys = run.xy(x)
    checked = []

    def measure(ops):
        ss = run.schedule(ops)
        try:
            for y in ys:
                y.fill_(float("nan"))
            D.dspmv_apply_group(ss, xs, ys)
            torch.cuda.synchronize()
            y = np.concatenate([t.cpu().numpy() for t in ys])
            assert np.array_equal(y, yref), PS.describe(ops)
            # the same schedule in the oracle's own executor gives the same y
            assert np.array_equal(O2.simulate(plans, val, x, _lib_to_oracle(ops)), yref)
            reps, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < 0.002:
                D.dspmv_apply_group(ss, xs, ys)
                reps += 1
            torch.cuda.synchronize()
            checked.append(1)
            return (time.perf_counter() - t0) / reps
        finally:
            for s in ss:
                D.dspmv_schedule_destroy(s)
            run.scheds.pop()
    try:
        m = M.MCTS(measure, n_streams=2, seed=3, space=sp, syncs="orderable").run(50)
    finally:
        run.close()
    assert m.iterations == 50 and len(checked) == 50
    assert len(m.dataset) >= 40              # rollouts are mostly distinct schedules
    best_ops, best_t = m.best()
    assert best_t > 0
    D.dspmv_schedule_validate(best_ops, 2)


@pytest.mark.parametrize("name", ["7pt64", "pl200k"])
def test_apply_host_fp32_vs_o1(name):
    """fp32 through the end-to-end C-ABI call with pinned host buffers, against
    O1 on the fp32 inputs upcast to fp64 (R-Q12: |y32 - y_ref| <= 1e-5 sum|a x|),
    and exact-mode inputs bitwise."""
    if name == "7pt64":
        n = 64 ** 3
        rp, col, val = gen.stencil("7pt", (64, 64, 64))
    else:
        n = 200000
        rp, col, val = gen.powerlaw(n)
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    try:
        for exact in (False, True):
            # stencil values are small integers already; the power-law matrix
            # has an exact-mode twin with the same structure (R-Q23)
            v = gen.powerlaw(n, exact=True)[2] if (exact and name == "pl200k") else val
            v32 = v.astype(np.float32)
            x32 = gen.x_values((0, n), exact=exact).astype(np.float32)
            plan = D.dspmv_plan_create(comm, n, rp, col, v32, dtype=D.DSPMV_F32)
            s = D.dspmv_schedule_create(plan, D.dspmv_schedule_derive(list(range(10)), [0] * 10, 1), 1)
            xh = torch.from_numpy(x32).pin_memory()
            yh = torch.full((n,), float("nan"), dtype=torch.float32).pin_memory()
            D.dspmv_apply_host(s, xh, yh)
            y = yh.numpy().astype(np.float64)
            xr, vr = x32.astype(np.float64), v32.astype(np.float64)
            yref = O1.o1_spmv(rp, col, vr, xr)
            if exact:
                assert np.array_equal(y, yref)
            else:
                assert within_tol(y, yref, O1.o1_absdot(rp, col, vr, xr), 1e-5)
            D.dspmv_schedule_destroy(s)
            D.dspmv_plan_destroy(plan)
    finally:
        D.dspmv_comm_destroy(comm)
