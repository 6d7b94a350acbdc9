"""Real multi-process distributed SpMV on one B200: 2 and 3 processes, each its
own CUDA context, bootstrapped over a gloo group through the HOST-transport
communicator; the fused Pack+put exchange maps the peers' receive buffers and
flags with CUDA IPC and synchronises through epoch flags in peer memory."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mat, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        import numpy as np
        from paper_2203_02530_b200 import dspmv as D
        from tests.gpu_helpers import derive_ops
        torch.cuda.set_device(0)

        def allgather(b: bytes) -> bytes:
            out = [None] * world
            dist.all_gather_object(out, b)
            return b"".join(out)

        if mat == "pl":
            n = 30000
            rb = D.dspmv_partition(n, world)
            rp, col, val = gen.powerlaw(n, (int(rb[rank]), int(rb[rank + 1])))
        elif mat == "7pt":                       # >= 2 MB of x per rank: pipelined apply_host
            n = 64 * 64 * 128
            rb = D.dspmv_partition(n, world)
            rp, col, val = gen.stencil("7pt", (64, 64, 128), (int(rb[rank]), int(rb[rank + 1])))
        else:
            n = 24 ** 3
            rb = D.dspmv_partition(n, world)
            rp, col, val = gen.stencil("27pt", (24, 24, 24), (int(rb[rank]), int(rb[rank + 1])))
        lo, hi = int(rb[rank]), int(rb[rank + 1])
        comm = D.dspmv_comm_create_host(world, rank, 0, allgather)
        plan = D.dspmv_plan_create(comm, n, rp, col, val, exchange=D.DSPMV_EXCHANGE_PUT)
        s = D.dspmv_schedule_create(plan, derive_ops(), 2)
        x = torch.from_numpy(gen.x_values((lo, hi))).cuda()
        y = torch.empty_like(x)
        ys = []
        for _ in range(4):                       # both receive-buffer parities
            y.fill_(float("nan"))
            dist.barrier()
            D.dspmv_apply(s, x, y)
            ys.append(y.cpu().numpy().copy())
        # the end-to-end path (pinned host x/y) gives the same bits
        xh = x.cpu().pin_memory()
        yh = torch.empty(hi - lo, dtype=torch.float64).pin_memory()
        for _ in range(2):
            yh.fill_(float("nan"))
            dist.barrier()
            D.dspmv_apply_host(s, xh, yh)
            if not np.array_equal(yh.numpy(), ys[0]):
                raise AssertionError("apply_host differs from apply")
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
        q.put((rank, lo, [a.tolist() for a in ys]))
    except Exception as e:  # noqa: BLE001
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mat", [(2, "pl"), (3, "27pt"), (2, "7pt")])
def test_multiprocess_fused_put_on_one_gpu(world, mat):
    import gen
    from oracle import spmv as O1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mat, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, lo, ys = q.get(timeout=600)
        assert lo >= 0, ys
        res[r] = (lo, ys)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    if mat == "pl":
        n = 30000
        rp, col, val = gen.powerlaw(n)
    elif mat == "7pt":
        n = 64 * 64 * 128
        rp, col, val = gen.stencil("7pt", (64, 64, 128))
    else:
        n = 24 ** 3
        rp, col, val = gen.stencil("27pt", (24, 24, 24))
    x = gen.x_values((0, n))
    yref = O1.o1_spmv(rp, col, val, x)
    s = O1.o1_absdot(rp, col, val, x)
    for k in range(4):
        y = np.concatenate([np.array(res[r][1][k]) for r in range(world)])
        assert np.all(np.abs(y - yref) <= 1e-12 * s), k


def _lower_band(n, w=8):
    """Row i: columns i-w+1..i (clipped), integer values: a one-directional
    exchange (rank r only receives from r-1)."""
    import gen
    cols = [np.arange(max(0, i - w + 1), i + 1) for i in range(n)]
    rp = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    col = np.concatenate(cols).astype(np.int32)
    bits = gen.counter_u64(17, 3, np.arange(len(col), dtype=np.uint64))
    val = np.floor(gen.u01(bits) * 16.0) - 8.0
    val[val == 0] = 1.0
    return rp, col, val


def _race_worker(rank, world, port, fine, q):
    import sys
    import time
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        from oracle import schedules as S
        from oracle import spmv as O1
        from paper_2203_02530_b200 import dspmv as D
        from tests.gpu_helpers import derive_ops, oracle_ops_to_lib
        torch.cuda.set_device(0)

        def allgather(b: bytes) -> bytes:
            out = [None] * world
            dist.all_gather_object(out, b)
            return b"".join(out)

        n = 20000
        rp, col, val = _lower_band(n)
        rb = D.dspmv_partition(n, world)
        lo, hi = int(rb[rank]), int(rb[rank + 1])
        a, b = int(rp[lo]), int(rp[hi])
        comm = D.dspmv_comm_create_host(world, rank, 0, allgather)
        plan = D.dspmv_plan_create(comm, n, rp[lo:hi + 1], col[a:b], val[a:b], exchange=D.DSPMV_EXCHANGE_PUT)
        if fine:
            V, E, _ = S.fine_dag([-1, 1])
            ops = oracle_ops_to_lib(S.derive(S.topological_orders(E, V)[0], {v: 0 for v in V}))
        else:
            ops = derive_ops()
        s = D.dspmv_schedule_create(plan, ops, 2)
        x0 = gen.x_values((0, n), exact=True)
        y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        bad = []
        dist.barrier()
        for k in range(60):
            # the last rank (receives, never sends) is slow to start each
            # apply; the others (send only) would run ahead without the
            # receivers' acknowledgement flags
            if rank == world - 1:
                time.sleep(0.004)
            xk = x0 + k
            x = torch.from_numpy(np.ascontiguousarray(xk[lo:hi])).cuda()
            D.dspmv_apply(s, x, y)
            if rank == world - 1:
                want = O1.o1_spmv(rp, col, val, xk)[lo:hi]
                if not np.array_equal(y.cpu().numpy(), want):
                    bad.append(k)
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
        q.put((rank, 0, bad))
    except Exception as e:  # noqa: BLE001
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fine", [False, True], ids=["coarse", "per-destination"])
def test_put_sender_cannot_overrun_slow_receiver(fine):
    """One-directional pattern over 2 processes: rank 0 only sends.  Its epoch
    flags to rank 1 are paired with rank 1's acknowledgement flags, so rank 0
    stays at most one apply ahead and never overwrites the receive buffer rank
    1 has not unpacked: every apply of the slow rank 1 is exact."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_race_worker, args=(r, world, port, fine, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, st, bad = q.get(timeout=600)
        assert st == 0, bad
        res[r] = bad
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert res[world - 1] == []
