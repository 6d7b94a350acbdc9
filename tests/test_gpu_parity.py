"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element on the same seeded inputs.  Tolerance (BASELINE.json north_star):
|y_gpu - y_ref| <= 1e-12 * sum_j |a_ij x_j| (fp64), 1e-5 (fp32, R-Q12); exact
mode (integer values, R-Q23) and the row-block kernel (stored-order sums,
DESIGN.md K1) are compared bitwise."""
import numpy as np
import pytest
import torch

import gen
from oracle import plan as O2
from oracle import schedules as S
from oracle import spmv as O1
from paper_2203_02530_b200 import dspmv as D
from tests.gpu_helpers import LocalRun, derive_ops, oracle_ops_to_lib, within_tol

pytestmark = pytest.mark.gpu


def _mat(name, exact=False):
    if name == "7pt32":
        return 32 ** 3, gen.stencil("7pt", (32, 32, 32))
    if name == "27pt20":
        return 20 ** 3, gen.stencil("27pt", (20, 20, 20))
    if name == "5pt64":
        return gen.config_matrix("c1")
    if name == "pl20k":
        return 20000, gen.powerlaw(20000, exact=exact)
    if name == "rand300":
        return 300, gen.random_csr(300, 0.05, seed=11, exact=exact, empty_rows=(0, 1, 150, 299),
                                   dense_rows=(7, 200))
    raise KeyError(name)


@pytest.mark.parametrize("name", ["7pt32", "27pt20", "5pt64"])
def test_single_rank_stencil_vs_o1(name):
    """The auto-chosen configuration sums every row of these stencils in one
    lane (rows <= 8 nnz with the short-row configuration, rows <= 32 with the
    fp64 long-row one), in stored order with separate rounding: bitwise equal
    to O1.  (Multi-lane classes -- a shuffle tree, tolerance -- are covered by
    the every-configuration test.)"""
    n, (rp, col, val) = _mat(name)
    short = np.diff(rp).max() <= 32
    for exact in (False, True):
        x = gen.x_values((0, n), exact=exact)
        run = LocalRun(n, rp, col, val, 1)
        try:
            y = run.apply(run.schedule(derive_ops()), x)
        finally:
            run.close()
        y1 = O1.o1_spmv(rp, col, val, x)
        if short or exact:
            assert np.array_equal(y, y1)
        else:
            assert within_tol(y, y1, O1.o1_absdot(rp, col, val, x), 1e-12)


@pytest.mark.parametrize("name", ["pl20k", "rand300"])
@pytest.mark.parametrize("vthr", [-1, 0, 1024])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_irregular_multi_rank_vs_oracle(name, vthr, P):
    for exact in (False, True):
        n, (rp, col, val) = _mat(name, exact)
        x = gen.x_values((0, n), exact=exact)
        run = LocalRun(n, rp, col, val, P, vector_threshold=vthr)
        try:
            y = run.apply(run.schedule(derive_ops()), x)
        finally:
            run.close()
        plans = O2.plan_all(rp, col, n, P)
        yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
        if exact:
            assert np.array_equal(y, yref)
        else:
            assert within_tol(y, yref, O1.o1_absdot(rp, col, val, x), 1e-12)


def test_row_length_bins():
    """Rows of every length class: 0, 1, 2, ..., 33, 64, ..., 2048, 2049, 4096."""
    lens = list(range(0, 34)) + [63, 64, 65, 255, 256, 1000, 2047, 2048, 2049, 4095, 4096]
    n = 5000
    rps, cols, vals = [0], [], []
    for i in range(n):
        L = lens[i % len(lens)]
        c = (np.arange(L) * 7919 + i) % n
        c = np.unique(c)
        bits = gen.counter_u64(5, 9, np.uint64(i), np.arange(len(c), dtype=np.uint64))
        cols.append(c)
        vals.append(2.0 * gen.u01(bits) - 1.0)
        rps.append(rps[-1] + len(c))
    rp = np.array(rps, np.int64)
    col = np.concatenate(cols).astype(np.int32)
    val = np.concatenate(vals)
    x = gen.x_values((0, n))
    yref = O1.o1_spmv(rp, col, val, x)
    s = O1.o1_absdot(rp, col, val, x)
    for vthr in (-1, 0, 1, 32, 1024):
        for P in (1, 4):
            run = LocalRun(n, rp, col, val, P, vector_threshold=vthr)
            try:
                y = run.apply(run.schedule(derive_ops()), x)
            finally:
                run.close()
            assert within_tol(y, yref, s, 1e-12), (vthr, P)


def test_every_schedule_same_bits_c1():
    """C1 (BASELINE configs[0]): 5-pt 64^2 over 2 ranks, every one of the 768
    derived schedules, 1 and 2 streams: y bitwise identical across schedules
    (R-Q9 ticket combine) and equal to the oracle (exact mode bitwise)."""
    for exact in (True, False):
        n, (rp, col, val) = gen.config_matrix("c1")
        x = gen.x_values((0, n), exact=exact)
        plans = O2.plan_all(rp, col, n, 2)
        yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
        run = LocalRun(n, rp, col, val, 2)
        try:
            first = None
            for ops in S.enumerate_derived(2, S.EDGES):
                ss = run.schedule(oracle_ops_to_lib(ops))
                y = run.apply(ss, x)
                for s in ss:
                    D.dspmv_schedule_destroy(s)
                run.scheds.pop()
                if first is None:
                    first = y
                    if exact:
                        assert np.array_equal(y, yref)
                    else:
                        assert within_tol(y, yref, O1.o1_absdot(rp, col, val, x), 1e-12)
                assert np.array_equal(y.view(np.uint64), first.view(np.uint64))
        finally:
            run.close()


@pytest.mark.parametrize("P", [2, 4, 8])
def test_rank_count_invariance_27pt(P):
    n, (rp, col, val) = _mat("27pt20", exact=True)
    for exact in (True, False):
        x = gen.x_values((0, n), exact=exact)
        y1 = O1.o1_spmv(rp, col, val, x)
        run = LocalRun(n, rp, col, val, P)
        try:
            y = run.apply(run.schedule(derive_ops()), x, reps=3)   # ticket epochs
        finally:
            run.close()
        if exact:
            assert np.array_equal(y, y1)
        else:
            assert within_tol(y, y1, O1.o1_absdot(rp, col, val, x), 1e-12)


def test_fp32_tolerance():
    n, (rp, col, val) = _mat("pl20k")
    x = gen.x_values((0, n))
    v32, x32 = val.astype(np.float32), x.astype(np.float32)
    yref = O1.o1_spmv(rp, col, v32.astype(np.float64), x32.astype(np.float64))
    s = O1.o1_absdot(rp, col, v32.astype(np.float64), x32.astype(np.float64))
    for P in (1, 4):
        run = LocalRun(n, rp, col, v32, P, dtype=D.DSPMV_F32)
        try:
            y = run.apply(run.schedule(derive_ops()), x32)
        finally:
            run.close()
        assert within_tol(y, yref, s, 1e-5)
    # exact mode: fp32 bitwise (partial sums < 2^24)
    n, (rp, col, val) = _mat("pl20k", exact=True)
    x = gen.x_values((0, n), exact=True)
    run = LocalRun(n, rp, col, val.astype(np.float32), 4, dtype=D.DSPMV_F32)
    try:
        y = run.apply(run.schedule(derive_ops()), x.astype(np.float32))
    finally:
        run.close()
    assert np.array_equal(y, O1.o1_spmv(rp, col, val, x))


def test_more_ranks_than_rows_and_empty_matrix():
    n, (rp, col, val) = 5, gen.random_csr(5, 0.6, seed=9)
    x = gen.x_values((0, n))
    run = LocalRun(n, rp, col, val, 8)
    try:
        y = run.apply(run.schedule(derive_ops()), x)
    finally:
        run.close()
    assert within_tol(y, O1.o1_spmv(rp, col, val, x), O1.o1_absdot(rp, col, val, x), 1e-12)
    n = 1000
    rp = np.zeros(n + 1, np.int64)
    run = LocalRun(n, rp, np.zeros(0, np.int32), np.zeros(0), 2)
    try:
        y = run.apply(run.schedule(derive_ops()), gen.x_values((0, n)))
    finally:
        run.close()
    assert np.all(y == 0.0) and not np.any(np.signbit(y))


def test_nccl_single_rank_apply_and_apply_host():
    n, (rp, col, val) = _mat("7pt32")
    x = gen.x_values((0, n))
    uid = D.dspmv_comm_unique_id()
    comm = D.dspmv_comm_create(uid, 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val, keep_host=True)
    ops = derive_ops()
    s = D.dspmv_schedule_create(plan, ops, 2)
    try:
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        D.dspmv_schedule_set_timing(s, True)
        D.dspmv_apply(s, xd, yd)
        t = D.dspmv_schedule_op_times(s)
        yL = [i for i, o in enumerate(ops) if o[0] == D.DSPMV_OP_SPMV_LOCAL][0]
        assert t[yL] > 0
        yref = O1.o1_spmv(rp, col, val, x)
        assert np.array_equal(yd.cpu().numpy(), yref)
        yh = np.empty(n)
        D.dspmv_apply_host(s, x, yh)
        assert np.array_equal(yh, yref)
        assert np.array_equal(D.dspmv_plan_export(plan, D.DSPMV_AL_COL), col)
        info = D.dspmv_plan_info_get(plan)
        assert info["ready"] == 1 and info["nnz_remote"] == 0 and info["n_blocks_local"] > 0
    finally:
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)


def test_lifetime_errors():
    n, (rp, col, val) = _mat("5pt64")
    comms = D.dspmv_comm_create_local(2, 0)
    p0 = D.dspmv_plan_create(comms[0], n, rp[:2049], col[:rp[2048]], val[:rp[2048]])
    s0 = D.dspmv_schedule_create(p0, derive_ops(), 2)
    with pytest.raises(D.DspmvError) as e:     # group incomplete -> not ready
        D.dspmv_apply_group([s0], [0], [0])
    with pytest.raises(D.DspmvError) as e:
        D.dspmv_plan_destroy(p0)               # live schedule
    assert e.value.status == D.DSPMV_ERR_STATE
    with pytest.raises(D.DspmvError) as e:
        D.dspmv_comm_destroy(comms[0])         # live plan
    assert e.value.status == D.DSPMV_ERR_STATE
    bad = [tuple(o) for o in derive_ops() if o[0] < 10]
    with pytest.raises(D.DspmvError) as e:
        D.dspmv_schedule_create(p0, bad, 2)
    assert e.value.status == D.DSPMV_ERR_SCHEDULE
    D.dspmv_schedule_destroy(s0)
    D.dspmv_plan_destroy(p0)
    for c in comms:
        D.dspmv_comm_destroy(c)


def test_launch_count_increases():
    n, (rp, col, val) = _mat("7pt32")
    before = D.dspmv_launch_count()
    run = LocalRun(n, rp, col, val, 2)
    try:
        run.apply(run.schedule(derive_ops()), gen.x_values((0, n)))
    finally:
        run.close()
    assert D.dspmv_launch_count() - before >= 5   # pack, y_L, unpack, y_R (+ per rank)


def test_full_size_c2_bench_config():
    """BASELINE configs[1] (7-pt 128^3, 1 B200) in the launch configuration
    bench.py times: the whole y against O1, bitwise."""
    n, (rp, col, val) = gen.config_matrix("c2")
    x = gen.x_values((0, n))
    uid = D.dspmv_comm_unique_id()
    comm = D.dspmv_comm_create(uid, 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val)
    s = D.dspmv_schedule_create(plan, derive_ops(), 2)
    try:
        xd = torch.from_numpy(x).cuda()
        yd = torch.empty_like(xd)
        for _ in range(3):
            D.dspmv_l2_flush(0)
            D.dspmv_apply(s, xd, yd)
        assert np.array_equal(yd.cpu().numpy(), O1.o1_spmv(rp, col, val, x))
    finally:
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)


@pytest.mark.parametrize("cfg", list(range(8)))
def test_every_block_cfg(cfg):
    """Every row-block kernel configuration (tile / consumer warps / stages)
    on an irregular multi-rank case and a stencil (bitwise vs O1)."""
    n, (rp, col, val) = _mat("pl20k")
    x = gen.x_values((0, n))
    plans = O2.plan_all(rp, col, n, 3)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    run = LocalRun(n, rp, col, val, 3, block_cfg=cfg)
    try:
        y = run.apply(run.schedule(derive_ops()), x, reps=2)
    finally:
        run.close()
    assert within_tol(y, yref, O1.o1_absdot(rp, col, val, x), 1e-12)
    for name in ("27pt20", "7pt32"):
        n, (rp, col, val) = _mat(name)
        xs = gen.x_values((0, n))
        run = LocalRun(n, rp, col, val, 1, block_cfg=cfg)
        try:
            y = run.apply(run.schedule(derive_ops()), xs)
        finally:
            run.close()
        y1 = O1.o1_spmv(rp, col, val, xs)
        if name == "7pt32":
            assert np.array_equal(y, y1)
        else:
            assert within_tol(y, y1, O1.o1_absdot(rp, col, val, xs), 1e-12)


def _sampled_check(n, rp, col, val, P, n_sample=20000, seed=5, bitwise=False):
    """Full-size matrix over P ranks (LOCAL if P > 1, else the bench's NCCL
    comm of one rank): y on sampled rows vs O1 computed row by row."""
    x = gen.x_values((0, n))
    if P == 1:
        comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
        plan = D.dspmv_plan_create(comm, n, rp, col, val)
        s = D.dspmv_schedule_create(plan, derive_ops(), 2)
        try:
            xd = torch.from_numpy(x).cuda()
            yd = torch.empty_like(xd)
            D.dspmv_l2_flush(0)
            D.dspmv_apply(s, xd, yd)
            y = yd.cpu().numpy()
        finally:
            D.dspmv_schedule_destroy(s)
            D.dspmv_plan_destroy(plan)
            D.dspmv_comm_destroy(comm)
    else:
        run = LocalRun(n, rp, col, val, P)
        try:
            y = run.apply(run.schedule(derive_ops()), x)
        finally:
            run.close()
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([rng.integers(0, n, n_sample), [0, n - 1],
                                     D.dspmv_partition(n, P)[1:-1]]))
    rows = rows[rows < n]
    yref = O1.o1_spmv_rows(rows, rp, col, val, x)
    rr = np.concatenate([[0], np.cumsum(np.diff(rp)[rows])])
    sub_rp = rr.astype(np.int64)
    sub_col = np.concatenate([col[rp[i]:rp[i + 1]] for i in rows])
    sub_val = np.concatenate([val[rp[i]:rp[i + 1]] for i in rows])
    scale = O1.o1_absdot(sub_rp, sub_col, sub_val, x)
    assert within_tol(y[rows], yref, scale, 1e-12)
    if bitwise:
        assert np.array_equal(y[rows], yref)
    assert np.isfinite(y).all()


def test_full_size_c3_27pt_256_sampled():
    """BASELINE configs[2] at full size (449M nnz, 1 B200), sampled rows; the
    fp64 long-row configuration sums each row in one lane in stored order, so
    the sampled rows are bitwise those of O1."""
    n, (rp, col, val) = gen.config_matrix("c3")
    _sampled_check(n, rp, col, val, 1, bitwise=True)


def test_full_size_c4_powerlaw_sampled():
    """BASELINE configs[3] at full size (8M rows, 134M nnz) on 1 rank and on 8
    in-process ranks (irregular halo, up to 7 peers), sampled rows."""
    n, (rp, col, val) = gen.config_matrix("c4")
    _sampled_check(n, rp, col, val, 1)
    _sampled_check(n, rp, col, val, 8, n_sample=5000)


def test_full_size_c5_7pt_192_four_ranks_sampled():
    """BASELINE configs[4] matrix (7-pt 192^3) over 4 in-process ranks."""
    n, (rp, col, val) = gen.config_matrix("c5")
    _sampled_check(n, rp, col, val, 4)


@pytest.mark.parametrize("name,P", [("pl20k", 2), ("pl20k", 8), ("27pt20", 4), ("rand300", 3), ("5pt64", 2)])
def test_fused_pack_put_exchange(name, P):
    """DSPMV_EXCHANGE_PUT: Pack stores straight into the peers' receive
    buffers (parity double-buffered, epoch flags, stream wait-value) -- same
    bits as the copy exchange, over several applies (both parities)."""
    for exact in (True, False):
        n, (rp, col, val) = _mat(name, exact)
        x = gen.x_values((0, n), exact=exact)
        out = {}
        for mode in (D.DSPMV_EXCHANGE_COPY, D.DSPMV_EXCHANGE_PUT):
            run = LocalRun(n, rp, col, val, P, exchange=mode)
            try:
                out[mode] = run.apply(run.schedule(derive_ops()), x, reps=3)
            finally:
                run.close()
        assert np.array_equal(out[0].view(np.uint64), out[1].view(np.uint64))
        plans = O2.plan_all(rp, col, n, P)
        yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
        if exact:
            assert np.array_equal(out[1], yref)
        else:
            assert within_tol(out[1], yref, O1.o1_absdot(rp, col, val, x), 1e-12)


def test_fused_pack_put_every_schedule_c1():
    """All 768 schedules with the fused exchange: identical bits (C1)."""
    n, (rp, col, val) = gen.config_matrix("c1")
    x = gen.x_values((0, n))
    run = LocalRun(n, rp, col, val, 2, exchange=D.DSPMV_EXCHANGE_PUT)
    try:
        first = None
        for ops in S.enumerate_derived(2, S.EDGES):
            ss = run.schedule(oracle_ops_to_lib(ops))
            y = run.apply(ss, x)
            for s_ in ss:
                D.dspmv_schedule_destroy(s_)
            run.scheds.pop()
            if first is None:
                first = y
            assert np.array_equal(y.view(np.uint64), first.view(np.uint64))
    finally:
        run.close()
    assert within_tol(first, O1.o1_spmv(rp, col, val, x), O1.o1_absdot(rp, col, val, x), 1e-12)


@pytest.mark.parametrize("name", ["7pt32", "pl20k", "27pt20"])
def test_apply_graph_equals_host_mode(name):
    """GPU-resident (CUDA-graph) execution of a schedule gives the same bits as
    the host-synchronised apply; recaptures when x changes; op timing works."""
    n, (rp, col, val) = _mat(name)
    uid = D.dspmv_comm_unique_id()
    comm = D.dspmv_comm_create(uid, 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val)
    stream = torch.cuda.Stream()
    scheds = []
    try:
        for order_streams in [None, ("paper1",)]:
            ops = derive_ops() if order_streams is None else D.dspmv_schedule_derive(list(range(10)), [0] * 10, 2)
            s = D.dspmv_schedule_create(plan, ops, 2)
            scheds.append(s)
            for seed in (1, 2):
                x = torch.from_numpy(gen.x_values((0, n), seed=seed)).cuda()
                yh = torch.empty_like(x)
                yg = torch.full_like(x, float("nan"))
                D.dspmv_apply(s, x, yh)
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        D.dspmv_apply_graph(s, x, yg, stream)
                stream.synchronize()
                assert torch.equal(yh, yg)
            D.dspmv_schedule_set_timing(s, (1 << D.DSPMV_OP_SPMV_LOCAL) | 1)
            D.dspmv_apply_graph(s, x, yg, stream)
            stream.synchronize()
            t = D.dspmv_schedule_op_times(s)
            iyl = [i for i, o in enumerate(ops) if o[0] == D.DSPMV_OP_SPMV_LOCAL][0]
            assert t[iyl] > 0 and t[0] >= t[iyl]
        yref = O1.o1_spmv(rp, col, val, gen.x_values((0, n), seed=2))
        assert within_tol(yg.cpu().numpy(), yref, O1.o1_absdot(rp, col, val, gen.x_values((0, n), seed=2)), 1e-12)
    finally:
        for s in scheds:
            D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)


def test_timestamp_aliasing_keeps_times_consistent():
    """An op-begin event at START's stream position reuses START's event, and
    in a graph END reuses y_L's end event when nothing follows it (runtime.h,
    timestamp aliasing): timings stay ordered and y stays bitwise = O1."""
    n, (rp, col, val) = gen.config_matrix("c2", mz=32)
    x = gen.x_values((0, n))
    yref = O1.o1_spmv(rp, col, val, x)
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val, caller_stream0=True)
    stream = torch.cuda.Stream()
    order = ["start", "y_L", "Pack", "PostSend", "PostRecv", "WaitRecv", "Unpack", "WaitSend", "y_R", "end"]
    kinds = [D.VERTEX_NAMES.index(v) for v in order]
    cases = {"y_L first on the caller stream": [0] * 10,
             "y_L first on the caller stream, Pack on stream 1": [1 if v == "Pack" else 0 for v in order],
             "y_L on stream 1": [1 if v == "y_L" else 0 for v in order]}
    scheds = []
    try:
        xd = torch.from_numpy(x).cuda()
        for name, streams in cases.items():
            ops = D.dspmv_schedule_derive(kinds, streams, 2)
            iyl = [i for i, o in enumerate(ops) if o[0] == D.DSPMV_OP_SPMV_LOCAL][0]
            s = D.dspmv_schedule_create(plan, ops, 2)
            scheds.append(s)
            D.dspmv_schedule_set_timing(s, (1 << D.DSPMV_OP_SPMV_LOCAL) | (1 << D.DSPMV_OP_START))
            for mode, fn in (("host", D.dspmv_apply), ("graph", D.dspmv_apply_graph)):
                yd = torch.full_like(xd, float("nan"))
                for _ in range(3):
                    fn(s, xd, yd, stream)
                stream.synchronize()
                assert np.array_equal(yd.cpu().numpy(), yref), (name, mode)
                t = D.dspmv_schedule_op_times(s)
                b, e = D.dspmv_schedule_op_timeline(s)
                assert t[iyl] > 0 and t[0] >= t[iyl] - 1e-6, (name, mode, t[0], t[iyl])
                assert 0.0 <= b[iyl] <= e[iyl] <= e[0] + 1e-6, (name, mode, b[iyl], e[iyl], e[0])
                if streams[1] == 0:
                    assert b[iyl] == 0.0, (name, mode)          # begin aliased to START
                    if mode == "graph":
                        assert e[iyl] == e[0], (name, mode)     # END aliased to y_L's end
    finally:
        for s in scheds:
            D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)


@pytest.mark.parametrize("skern", [D.DSPMV_SKERNEL_STREAM, D.DSPMV_SKERNEL_STREAM_TMA, D.DSPMV_SKERNEL_SELL])
@pytest.mark.parametrize("name", ["pl20k", "rand300", "7pt32", "27pt20"])
@pytest.mark.parametrize("P", [1, 3])
def test_stream_kernel_bitwise_vs_oracle(name, P, skern):
    """CSR-stream S group (DSPMV_SKERNEL_STREAM): every row of <= 256 nnz is
    summed in stored order by one lane from rounded products, so y equals the
    oracle's O2 loops bit for bit on every row whose A_L and A_R parts both go
    to the stream kernel (whole row <= 256 nnz); longer rows (warp-per-row
    kernel) within the R-Q11 tolerance."""
    n, (rp, col, val) = _mat(name)
    x = gen.x_values((0, n))
    run = LocalRun(n, rp, col, val, P, s_kernel=skern)
    try:
        y = run.apply(run.schedule(derive_ops()), x, reps=2)
        assert all(D.dspmv_plan_info_get(p)["s_kernel_local"] == skern for p in run.plans)
    finally:
        run.close()
    plans = O2.plan_all(rp, col, n, P)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    short = np.diff(rp) <= 256
    assert np.array_equal(y[short], yref[short])
    assert within_tol(y, yref, O1.o1_absdot(rp, col, val, x), 1e-12)


def test_stream_kernel_auto_choice_and_fp32():
    """Auto choice: the power-law matrix (irregular rows) runs the CSR-stream
    kernel, the 7-pt stencil the row-block kernel; a forced block_cfg keeps
    the row-block kernel.  fp32 CSR-stream within the R-Q12 tolerance."""
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    try:
        for name, want in (("pl20k", D.DSPMV_SKERNEL_STREAM), ("7pt32", D.DSPMV_SKERNEL_BLOCK)):
            n, (rp, col, val) = _mat(name)
            plan = D.dspmv_plan_create(comm, n, rp, col, val)
            assert D.dspmv_plan_info_get(plan)["s_kernel_local"] == want, name
            D.dspmv_plan_destroy(plan)
        n, (rp, col, val) = _mat("pl20k")
        plan = D.dspmv_plan_create(comm, n, rp, col, val, block_cfg=3)
        assert D.dspmv_plan_info_get(plan)["s_kernel_local"] == D.DSPMV_SKERNEL_BLOCK
        D.dspmv_plan_destroy(plan)
    finally:
        D.dspmv_comm_destroy(comm)
    n, (rp, col, val) = _mat("pl20k")
    v32 = val.astype(np.float32)
    x32 = gen.x_values((0, n)).astype(np.float32)
    run = LocalRun(n, rp, col, v32, 2, dtype=D.DSPMV_F32, s_kernel=D.DSPMV_SKERNEL_STREAM)
    try:
        y = run.apply(run.schedule(derive_ops()), x32)
    finally:
        run.close()
    xr, vr = x32.astype(np.float64), v32.astype(np.float64)
    assert within_tol(y, O1.o1_spmv(rp, col, vr, xr), O1.o1_absdot(rp, col, vr, xr), 1e-5)


@pytest.mark.parametrize("skern", [D.DSPMV_SKERNEL_STREAM, D.DSPMV_SKERNEL_STREAM_TMA, D.DSPMV_SKERNEL_SELL])
def test_stream_kernel_edge_cases(skern):
    """CSR-stream with no S rows at all (every row > 256 nnz: the long-row
    kernel alone), with runs of empty rows (tiles whose rows sum to +0), and
    a 1-row matrix."""
    rng = np.random.default_rng(3)
    cases = []
    n = 600                                            # every row 300 nnz
    cols = np.stack([np.sort(rng.choice(n, 300, replace=False)) for _ in range(n)]).ravel().astype(np.int32)
    cases.append((n, np.arange(n + 1, dtype=np.int64) * 300, cols, rng.uniform(-1, 1, cols.size)))
    n = 5000                                           # 4000 empty rows in a row, then short rows
    lens = np.r_[np.zeros(4000, np.int64), rng.integers(1, 12, 1000)]
    rp = np.r_[0, np.cumsum(lens)].astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int32)
    cases.append((n, rp, cols, rng.uniform(-1, 1, cols.size)))
    cases.append((1, np.array([0, 1], np.int64), np.array([0], np.int32), np.array([2.5])))
    for n, rp, col, val in cases:
        x = gen.x_values((0, n))
        run = LocalRun(n, rp, col, val, 1, s_kernel=skern)
        try:
            y = run.apply(run.schedule(derive_ops()), x)
        finally:
            run.close()
        yref = O1.o1_spmv(rp, col, val, x)
        short = np.diff(rp) <= 256
        assert np.array_equal(y[short], yref[short]) and not np.any(np.signbit(y[np.diff(rp) == 0]))
        assert within_tol(y, yref, O1.o1_absdot(rp, col, val, x), 1e-12)


@pytest.mark.parametrize("cfg", ["c3", "c2", "c4"])
def test_full_size_bench_launch_configuration(cfg):
    """The launch configuration bench.py times at N = 1: the full BASELINE
    matrix, a GPU-resident graph with schedule stream 0 bound to the caller's
    stream, L2 flushed before each apply, two applies -- every row against
    O1 (C2/C3: bitwise, each row is summed in stored order in one lane; C4:
    rows <= 256 nnz bitwise, the rest within the R-Q11 tolerance)."""
    n, (rp, col, val) = gen.config_matrix(cfg)
    x = gen.x_values((0, n))
    yref = O1.o1_spmv(rp, col, val, x)
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val)
    order = ["start", "y_L", "Pack", "PostSend", "PostRecv", "WaitRecv", "Unpack", "y_R", "WaitSend", "end"]
    s = D.dspmv_schedule_create(plan, derive_ops(order, {"y_L": 0, "Pack": 1, "Unpack": 1, "y_R": 0}), 2)
    D.dspmv_schedule_set_timing(s, True)
    D.dspmv_schedule_set_caller_stream0(s, 1)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    st = torch.cuda.Stream()
    try:
        for _ in range(2):
            yd.fill_(float("nan"))
            D.dspmv_l2_flush(0, st)
            D.dspmv_apply_graph(s, xd, yd, st)
            torch.cuda.synchronize()
            y = yd.cpu().numpy()
            if cfg in ("c2", "c3"):
                assert np.array_equal(y, yref)
            else:
                short = np.diff(rp) <= 256
                assert np.array_equal(y[short], yref[short])
                assert within_tol(y, yref, O1.o1_absdot(rp, col, val, x), 1e-12)
    finally:
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)


@pytest.mark.parametrize("skern", [D.DSPMV_SKERNEL_STREAM, D.DSPMV_SKERNEL_SELL, D.DSPMV_SKERNEL_BLOCK])
@pytest.mark.parametrize("name,vthr", [("pl20k", -1), ("pl20k", 64), ("rand300", 8)])
@pytest.mark.parametrize("P", [1, 3])
def test_long_row_sum_stored_bitwise_every_row(name, vthr, P, skern):
    """long_row_sum = DSPMV_LONG_ROW_STORED: the warp-per-row rows (more than
    vector_threshold nnz, up to 4,096 on the power-law matrix) add their
    rounded products in stored order, so y equals the oracle's O2 loops bit
    for bit on EVERY row when the S-group kernel sums its rows in one lane
    (CSR-stream, sliced; the row-block kernel with rows of <= 8 nnz)."""
    n, (rp, col, val) = _mat(name)
    if skern == D.DSPMV_SKERNEL_BLOCK and name == "pl20k":
        pytest.skip("the row-block kernel sums rows of 9..256 nnz with several lanes (tolerance)")
    x = gen.x_values((0, n))
    run = LocalRun(n, rp, col, val, P, s_kernel=skern, vector_threshold=vthr,
                   long_row_sum=D.DSPMV_LONG_ROW_STORED)
    try:
        y = run.apply(run.schedule(derive_ops()), x, reps=2)
    finally:
        run.close()
    plans = O2.plan_all(rp, col, n, P)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    long_rows = np.diff(rp) > (256 if vthr < 0 else vthr)
    assert long_rows.any()
    assert np.array_equal(y.view(np.int64), yref.view(np.int64))
