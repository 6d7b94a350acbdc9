"""The §8(b) plan options through the C ABI (include/dspmv.h dspmv_plan_opts):
pack_mode ALIAS_IF_CONTIGUOUS (stencil send sets are planes,
sent straight from x), accumulate_mode EXPLICIT_IN_END (y = y_L + y_R
added at END), the alloc/free callbacks (torch's caching allocator),
debug_checks (COLLECTIVE arguments agree across ranks) and the
binding's argument checks -- each against the oracle."""
import os
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
from tests.gpu_helpers import LocalRun, derive_ops, oracle_ops_to_lib, within_tol

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stencil(name, exact=True):
    if name == "c1":
        n, (rp, col, val) = gen.config_matrix("c1")
        return n, rp, col, val
    if name == "7pt24":     # C5-shaped: 7-pt, slabs of whole planes per rank
        rp, col, val = gen.stencil("7pt", (24, 24, 24))
        return 24 ** 3, rp, col, val
    if name == "27pt16":
        rp, col, val = gen.stencil("27pt", (16, 16, 16))
        return 16 ** 3, rp, col, val
    n = 20000
    rp, col, val = gen.powerlaw(n, exact=exact)
    return n, rp, col, val


@pytest.mark.parametrize("name,P", [("c1", 2), ("7pt24", 2), ("7pt24", 4), ("27pt16", 4)])
def test_pack_alias_stencils_bitwise_oracle(name, P):
    """Stencil send lists are runs of consecutive rows (whole planes): the
    alias is taken (plan info pack_alias = 1, no send buffer, Pack launches
    nothing) and y equals O2 bitwise in exact mode for several schedules."""
    n, rp, col, val = _stencil(name)
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, P)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    run = LocalRun(n, rp, col, val, P, pack_mode=D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS)
    try:
        assert all(D.dspmv_plan_info_get(p)["pack_alias"] == 1 for p in run.plans)
        for k, ops in enumerate(S.enumerate_derived(2, S.EDGES)[::97]):
            ss = run.schedule(oracle_ops_to_lib(ops))
            l0 = D.dspmv_launch_count()
            y = run.apply(ss, x)
            launched = D.dspmv_launch_count() - l0
            assert np.array_equal(y, yref), k
            # P ranks x (y_L, Unpack, y_R) at most: no Pack kernel
            assert launched <= 3 * P, launched
    finally:
        run.close()


def test_pack_alias_declined_for_scattered_send_lists():
    """Power-law send lists are scattered: the option falls back to the
    gather (pack_alias = 0) and y still equals O2."""
    n, rp, col, val = _stencil("pl", exact=True)
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, 3)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    run = LocalRun(n, rp, col, val, 3, pack_mode=D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS)
    try:
        assert all(D.dspmv_plan_info_get(p)["pack_alias"] == 0 for p in run.plans)
        assert np.array_equal(run.apply(run.schedule(derive_ops()), x), yref)
    finally:
        run.close()


@pytest.mark.parametrize("name,P", [("c1", 2), ("pl", 3), ("27pt16", 4)])
def test_explicit_accumulate_same_bits_as_ticket(name, P):
    """EXPLICIT_IN_END deposits both partials and adds them at END: bitwise the
    ticket combine (two-operand addition is commutative) and = O2 in exact
    mode, over a stride of the 768 derived schedules, float and exact inputs."""
    for exact in (True, False):
        n, rp, col, val = _stencil(name, exact)
        x = gen.x_values((0, n), exact=exact)
        plans = O2.plan_all(rp, col, n, P)
        yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
        runs = [LocalRun(n, rp, col, val, P, accumulate_mode=m)
                for m in (D.DSPMV_ACC_TICKET, D.DSPMV_ACC_EXPLICIT_IN_END)]
        try:
            assert D.dspmv_plan_info_get(runs[1].plans[0])["accumulate_mode"] == D.DSPMV_ACC_EXPLICIT_IN_END
            for ops in S.enumerate_derived(2, S.EDGES)[::61]:
                lib_ops = oracle_ops_to_lib(ops)
                y0 = runs[0].apply(runs[0].schedule(lib_ops), x)
                y1 = runs[1].apply(runs[1].schedule(lib_ops), x)
                assert np.array_equal(y0.view(np.uint64), y1.view(np.uint64))
                if exact:
                    assert np.array_equal(y1, yref)
                else:
                    assert within_tol(y1, yref, O1.o1_absdot(rp, col, val, x), 1e-12)
        finally:
            for r in runs:
                r.close()


def test_plan_memory_from_torch_caching_allocator():
    """alloc/free callbacks: with torch_alloc the plan's device bytes show up
    in torch.cuda.memory_allocated and are returned at plan_destroy; with
    torch_alloc=False (cudaMalloc) torch's count does not move.  Results agree."""
    n = 64 ** 3
    rp, col, val = gen.stencil("7pt", (64, 64, 64))
    x = torch.from_numpy(gen.x_values((0, n))).cuda()
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    try:
        ys = []
        for ta in (True, False):
            torch.cuda.synchronize()
            m0 = torch.cuda.memory_allocated()
            plan = D.dspmv_plan_create(comm, n, rp, col, val, torch_alloc=ta)
            dev_bytes = D.dspmv_plan_info_get(plan)["device_bytes"]
            grew = torch.cuda.memory_allocated() - m0
            if ta:
                assert grew >= dev_bytes > 12 * len(col)
            else:
                assert grew == 0
            s = D.dspmv_schedule_create(plan, derive_ops(), 2)
            y = torch.empty_like(x)
            D.dspmv_apply(s, x, y)
            ys.append(y.cpu().numpy())
            del y
            D.dspmv_schedule_destroy(s)
            D.dspmv_plan_destroy(plan)
            torch.cuda.synchronize()
            assert torch.cuda.memory_allocated() == m0
        assert np.array_equal(ys[0], ys[1])
        assert np.array_equal(ys[0], O1.o1_spmv(rp, col, val, x.cpu().numpy()))
    finally:
        D.dspmv_comm_destroy(comm)


def test_binding_rejects_mismatched_tensors():
    """ADVICE: the binding checks x/y against the plan before the C call."""
    n = 4096
    rp, col, val = gen.stencil("7pt", (16, 16, 16))
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val)
    s = D.dspmv_schedule_create(plan, derive_ops(), 2)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    bad = [(x.float(), y), (x[:-1], y), (x, y[::2].contiguous()), (torch.zeros(2 * n, dtype=torch.float64,
                                                                               device="cuda")[::2], y),
           (x.cpu(), y)]
    try:
        for bx, by in bad:
            with pytest.raises(D.DspmvError) as e:
                D.dspmv_apply(s, bx, by)
            assert e.value.status == D.DSPMV_ERR_ARG
        with pytest.raises(D.DspmvError):
            D.dspmv_apply_host(s, x, y.cpu())
        D.dspmv_apply(s, x, y)   # the well-formed call still works
    finally:
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)


def _free_port():
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    p = so.getsockname()[1]
    so.close()
    return p


def _hash_worker(rank, world, port, q):
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
        n = 24 ** 3
        rb = D.dspmv_partition(n, world)
        lo, hi = int(rb[rank]), int(rb[rank + 1])
        rp, col, val = gen.stencil("7pt", (24, 24, 24), (lo, hi))
        comm = D.dspmv_comm_create_host(world, rank, 0, allgather)
        plan = D.dspmv_plan_create(comm, n, rp, col, val, exchange=D.DSPMV_EXCHANGE_PUT, debug_checks=True)
        x = torch.from_numpy(gen.x_values((lo, hi))).cuda()
        y = torch.empty_like(x)
        same = D.dspmv_schedule_create(plan, derive_ops(), 2)
        D.dspmv_apply(same, x, y)                 # identical schedules: passes the check
        order = ["start", "Pack", "y_L", "PostSend", "PostRecv", "WaitSend", "WaitRecv", "Unpack", "y_R", "end"]
        streams = {"Pack": 0, "y_L": rank % 2, "Unpack": 0, "y_R": 0}   # differs across ranks
        diff = D.dspmv_schedule_create(plan, derive_ops(order, streams), 2)
        status = 0
        try:
            D.dspmv_apply(diff, x, y)
        except D.DspmvError as e:
            status = e.status
        q.put((rank, status))
        D.dspmv_schedule_destroy(same)
        D.dspmv_schedule_destroy(diff)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_debug_checks_catch_schedules_that_differ_across_ranks():
    """debug_checks over a HOST communicator (2 processes on cuda:0): the
    first apply of a schedule whose ops differ between the ranks fails with
    ERR_SCHEDULE on every rank instead of exchanging mismatched data."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hash_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: D.DSPMV_ERR_SCHEDULE, 1: D.DSPMV_ERR_SCHEDULE}, res


def test_nvtx_ranges_do_not_change_results():
    """DSPMV_NVTX=1 wraps every executed op and apply in an NVTX range
    (SURVEY §5 tracing); the run under it gives the bits of a plain run."""
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, torch, gen\n"
        "from paper_2203_02530_b200 import dspmv as D\n"
        "from tests.gpu_helpers import LocalRun, derive_ops\n"
        "n, (rp, col, val) = gen.config_matrix('c1')\n"
        "run = LocalRun(n, rp, col, val, 2)\n"
        "y = run.apply(run.schedule(derive_ops()), gen.x_values((0, n), exact=True))\n"
        "run.close()\n"
        "np.save(sys.argv[1], y)\n" % ROOT)
    outs = []
    for env_on in ("0", "1"):
        path = os.path.join("/tmp", f"nvtx_y_{os.getpid()}_{env_on}.npy")
        r = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True, timeout=300,
                           env={**os.environ, "DSPMV_NVTX": env_on}, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
        os.unlink(path)
    assert np.array_equal(outs[0], outs[1])


def test_schedule_caller_stream0_override():
    """dspmv_schedule_set_caller_stream0: stream 0 bound to the caller's
    stream or to a library stream, per schedule, in host and graph mode (the
    cached graph is re-captured on a change): identical bits, = O1."""
    n = 32 ** 3
    rp, col, val = gen.stencil("7pt", (32, 32, 32))
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val)
    order = ["start", "y_L", "Pack", "PostSend", "PostRecv", "WaitRecv", "Unpack", "y_R", "WaitSend", "end"]
    s = D.dspmv_schedule_create(plan, derive_ops(order, {"y_L": 0, "Pack": 1, "Unpack": 1, "y_R": 0}), 2)
    D.dspmv_schedule_set_timing(s, True)
    x = torch.from_numpy(gen.x_values((0, n))).cuda()
    st = torch.cuda.Stream()
    ref = O1.o1_spmv(rp, col, val, x.cpu().numpy())
    try:
        for mode in (0, 1, -1, 1, 0):
            D.dspmv_schedule_set_caller_stream0(s, mode)
            for fn in (D.dspmv_apply, D.dspmv_apply_graph):
                y = torch.full_like(x, float("nan"))
                fn(s, x, y, st)
                torch.cuda.synchronize()
                assert np.array_equal(y.cpu().numpy(), ref), (mode, fn.__name__)
                assert D.dspmv_schedule_op_times(s)[0] > 0
        with pytest.raises(D.DspmvError):
            D.dspmv_schedule_set_caller_stream0(s, 2)
    finally:
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)


@pytest.mark.parametrize("exchange", [D.DSPMV_EXCHANGE_COPY, D.DSPMV_EXCHANGE_PUT], ids=["copy", "put"])
@pytest.mark.parametrize("name,P", [("c1", 2), ("pl", 3), ("27pt16", 4)])
def test_fused_unpack_bitwise_oracle(name, P, exchange):
    """unpack_mode FUSED: Unpack launches nothing and y_R gathers the halo
    from the receive buffer (PUT: the half of this apply's parity, from the
    device epoch).  Host lock-step and group graphs, several applies (both
    parities), a stride of the derived schedules: = O2 bitwise (exact mode)."""
    n, rp, col, val = _stencil(name, exact=True)
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, P)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    run = LocalRun(n, rp, col, val, P, exchange=exchange, unpack_mode=D.DSPMV_UNPACK_FUSED)
    xs, ys = run.xy(x)
    stream = torch.cuda.Stream()
    try:
        assert all(D.dspmv_plan_info_get(p)["unpack_fused"] == 1 for p in run.plans)
        for k, ops in enumerate(S.enumerate_derived(2, S.EDGES)[::128]):
            ss = run.schedule(oracle_ops_to_lib(ops))
            for rep in range(3):
                for y in ys:
                    y.fill_(float("nan"))
                if rep == 1:
                    D.dspmv_apply_group(ss, xs, ys)
                else:
                    D.dspmv_apply_graph_group(ss, xs, ys, stream)
                torch.cuda.synchronize()
                assert np.array_equal(np.concatenate([t.cpu().numpy() for t in ys]), yref), (k, rep)
    finally:
        run.close()
