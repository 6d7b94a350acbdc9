"""GPU-resident exchange (NEXT-3 (ii)+(iii), P:244 host-blocking MPI_Wait /
cudaDeviceSynchronize): schedules captured into CUDA graphs with
the exchange inside -- LOCAL groups of several ranks as one graph (COPY:
device copies ordered after the senders' Pack; PUT: fused Pack+put with a
device-resident epoch and flag-wait kernels), and separate processes with
the fused put -- each bitwise equal to the host-synchronised executor and to
the oracle."""
import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import gen
from oracle import plan as O2
from oracle import schedules as S
from oracle import spmv as O1
from paper_2203_02530_b200 import dspmv as D
from tests.gpu_helpers import LocalRun, derive_ops, oracle_ops_to_lib

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _case(name):
    if name == "c1":
        n, (rp, col, val) = gen.config_matrix("c1")
        return n, rp, col, val, 2
    if name == "pl":
        n = 20000
        rp, col, val = gen.powerlaw(n, exact=True)
        return n, rp, col, val, 3
    rp, col, val = gen.stencil("27pt", (16, 16, 16))
    return 16 ** 3, rp, col, val, 4


@pytest.mark.parametrize("pack_mode", [D.DSPMV_PACK_GATHER, D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS], ids=["gather", "alias"])
@pytest.mark.parametrize("exchange", [D.DSPMV_EXCHANGE_COPY, D.DSPMV_EXCHANGE_PUT], ids=["copy", "put"])
@pytest.mark.parametrize("name", ["c1", "pl", "27pt"])
def test_group_graph_equals_host_and_oracle(name, exchange, pack_mode):
    """A stride of the 768 derived and the 4,780 orderable schedules: the
    group graph (3 launches: both PUT parities, then host mode again) gives
    the bits of the host-synchronised group apply and of O2 (exact mode)."""
    n, rp, col, val, P = _case(name)
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, P)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    run = LocalRun(n, rp, col, val, P, exchange=exchange, pack_mode=pack_mode)
    xs, ys = run.xy(x)
    stream = torch.cuda.Stream()
    space = S.enumerate_derived(2, S.EDGES)[::89] + S.enumerate_orderable(2, S.EDGES)[::601]
    try:
        for k, ops in enumerate(space):
            ss = run.schedule(oracle_ops_to_lib(ops))
            if k % 2:
                for s in ss:
                    D.dspmv_schedule_set_timing(s, True)
            for rep in range(3):
                for y in ys:
                    y.fill_(float("nan"))
                if rep < 2:
                    D.dspmv_apply_graph_group(ss, xs, ys, stream)
                else:
                    D.dspmv_apply_group(ss, xs, ys)
                torch.cuda.synchronize()
                y = np.concatenate([t.cpu().numpy() for t in ys])
                assert np.array_equal(y, yref), (k, rep)
            if k % 2:
                t = D.dspmv_schedule_op_times(ss[0])
                assert t[0] > 0
    finally:
        run.close()


def _rand_topo(V, E, rng):
    pred = {v: {u for u, w in E if w == v} for v in V}
    done, out = set(), []
    while len(out) < len(V):
        v = rng.choice([v for v in V if v not in done and pred[v] <= done])
        out.append(v)
        done.add(v)
    return out


def test_group_graph_fine_schedules():
    """Per-destination vertices (offsets -1, +1) in a group graph, PUT and COPY."""
    n, rp, col, val, P = _case("c1")
    P = 3
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, P)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    V, E, _ = S.fine_dag([-1, 1])
    rng = random.Random(7)
    orders = [_rand_topo(V, E, rng) for _ in range(12)]
    stream = torch.cuda.Stream()
    for exchange in (D.DSPMV_EXCHANGE_COPY, D.DSPMV_EXCHANGE_PUT):
        run = LocalRun(n, rp, col, val, P, exchange=exchange)
        xs, ys = run.xy(x)
        try:
            for i in range(len(orders)):
                streams = {v: (j % 2) for j, v in enumerate(orders[i]) if S.base(v) in S.GPU_VERTICES}
                ss = run.schedule(oracle_ops_to_lib(S.derive(orders[i], streams, E)))
                for _ in range(2):
                    for y in ys:
                        y.fill_(float("nan"))
                    D.dspmv_apply_graph_group(ss, xs, ys, stream)
                    torch.cuda.synchronize()
                    assert np.array_equal(np.concatenate([t.cpu().numpy() for t in ys]), yref), i
        finally:
            run.close()


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        from paper_2203_02530_b200 import dspmv as D
        from tests.gpu_helpers import derive_ops
        torch.cuda.set_device(0)

        def allgather(b: bytes) -> bytes:
            out = [None] * world
            dist.all_gather_object(out, b)
            return b"".join(out)
        n = 30000
        rb = D.dspmv_partition(n, world)
        lo, hi = int(rb[rank]), int(rb[rank + 1])
        rp, col, val = gen.powerlaw(n, (lo, hi), exact=True)
        comm = D.dspmv_comm_create_host(world, rank, 0, allgather)
        plan = D.dspmv_plan_create(comm, n, rp, col, val, exchange=D.DSPMV_EXCHANGE_PUT)
        stream = torch.cuda.Stream()
        x = torch.from_numpy(gen.x_values((lo, hi), exact=True)).cuda()
        y = torch.empty_like(x)
        out = []
        for order, streams in ((None, None),
                               (["start", "y_L", "Pack", "PostSend", "PostRecv", "WaitRecv", "Unpack", "y_R",
                                 "WaitSend", "end"], {"y_L": 1})):
            s = D.dspmv_schedule_create(plan, derive_ops() if order is None else derive_ops(order, streams), 2)
            # graph, graph, host, graph: the device epoch stays in step with the host's
            for mode in ("graph", "graph", "host", "graph", "graph"):
                y.fill_(float("nan"))
                dist.barrier()
                if mode == "graph":
                    D.dspmv_apply_graph(s, x, y, stream)
                else:
                    D.dspmv_apply(s, x, y, stream)
                torch.cuda.synchronize()
                out.append(y.cpu().numpy().tolist())
            D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
        q.put((rank, lo, out))
    except Exception as e:  # noqa: BLE001
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_put_graph(world):
    """Separate processes on cuda:0 (HOST comm, CUDA IPC): the fused put
    exchange captured in each rank's graph; mixed with host-mode applies."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, lo, ys = q.get(timeout=600)
        assert lo >= 0, ys
        res[r] = ys
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 30000
    rp, col, val = gen.powerlaw(n, exact=True)
    yref = O1.o1_spmv(rp, col, val, gen.x_values((0, n), exact=True))
    for k in range(len(res[0])):
        y = np.concatenate([np.array(res[r][k]) for r in range(world)])
        assert np.array_equal(y, yref), k


@pytest.mark.parametrize("cfg,P,exchange,pack_mode", [
    ("c5", 4, D.DSPMV_EXCHANGE_PUT, D.DSPMV_PACK_GATHER),
    ("c5", 4, D.DSPMV_EXCHANGE_COPY, D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS),
    ("c4", 8, D.DSPMV_EXCHANGE_PUT, D.DSPMV_PACK_GATHER),
    ("c3", 8, D.DSPMV_EXCHANGE_COPY, D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS),
], ids=["c5-put", "c5-alias", "c4-put-8", "c3-alias-8"])
def test_full_size_group_graph_vs_o1(cfg, P, exchange, pack_mode):
    """BASELINE configs[4] (7-pt 192^3 over 4 ranks), configs[3] (power-law
    8M over 8 ranks, up to 7 peers) and configs[2] (27-pt 256^3 over 8 ranks,
    the N = 8 strong-scaling split) at full size, as ONE GPU-resident graph
    per apply with the fused put or aliased sends: every row against the O1
    oracle (the C loop runs the whole matrix in well under a second), over
    both PUT receive-buffer parities."""
    n, (rp, col, val) = gen.config_matrix(cfg)
    x = gen.x_values((0, n))
    yref = O1.o1_spmv(rp, col, val, x)
    scale = O1.o1_absdot(rp, col, val, x)
    run = LocalRun(n, rp, col, val, P, exchange=exchange, pack_mode=pack_mode)
    xs, ys = run.xy(x)
    stream = torch.cuda.Stream()
    try:
        ss = run.schedule(oracle_ops_to_lib(S.enumerate_derived(2, S.EDGES)[5]))
        for _ in range(2):
            for y in ys:
                y.fill_(float("nan"))
            D.dspmv_apply_graph_group(ss, xs, ys, stream)
            torch.cuda.synchronize()
            y = np.concatenate([t.cpu().numpy() for t in ys])
            assert np.all(np.abs(y - yref) <= 1e-12 * scale) and np.isfinite(y).all()
    finally:
        run.close()


def test_group_graph_survives_member_replacement():
    """Destroying one rank's schedule drops the group graph its leader holds
    (it references that schedule's events); the next group apply with a new
    schedule re-captures and is still exact."""
    n, rp, col, val, P = _case("c1")
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, P)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    run = LocalRun(n, rp, col, val, P)
    xs, ys = run.xy(x)
    stream = torch.cuda.Stream()
    try:
        ops = derive_ops()
        ss = run.schedule(ops)
        D.dspmv_apply_graph_group(ss, xs, ys, stream)
        torch.cuda.synchronize()
        D.dspmv_schedule_destroy(ss[1])
        ss[1] = D.dspmv_schedule_create(run.plans[1], ops, 2)
        for y in ys:
            y.fill_(float("nan"))
        D.dspmv_apply_graph_group(ss, xs, ys, stream)
        torch.cuda.synchronize()
        assert np.array_equal(np.concatenate([t.cpu().numpy() for t in ys]), yref)
    finally:
        run.close()
