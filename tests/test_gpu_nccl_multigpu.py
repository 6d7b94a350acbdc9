"""The NCCL path with real peers (the halo exchanged between ranks on
different GPUs): 2 processes, one GPU each, the library's own NCCL
communicator (unique id broadcast over a gloo group).  Plan-time request
exchange over NCCL, the NCCL send/recv group (COPY), the fused Pack+put over
peer memory across GPUs (PUT), host-synchronised and graph execution -- every
y checked against the oracle.  Skipped unless the box has >= 2 GPUs (the
driver's 8-GPU node runs it; single-GPU leases skip it)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mat(name, lo=None, hi=None):
    import gen
    rr = None if lo is None else (lo, hi)
    if name == "27pt":
        return 24 ** 3, gen.stencil("27pt", (24, 24, 24), rr, )
    n = 30000
    return n, gen.powerlaw(n, rr, exact=True)


def _worker(rank, world, port, mat, q):
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
        torch.cuda.set_device(rank)
        uid = [D.dspmv_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = D.dspmv_comm_create(uid[0], world, rank, rank)
        n = _mat(mat)[0]
        rb = D.dspmv_partition(n, world)
        lo, hi = int(rb[rank]), int(rb[rank + 1])
        _, (rp, col, val) = _mat(mat, lo, hi)
        x = torch.from_numpy(gen.x_values((lo, hi), exact=(mat != "27pt"))).cuda()
        y = torch.empty_like(x)
        stream = torch.cuda.Stream()
        out = {}
        for ex_name, ex in (("copy", D.DSPMV_EXCHANGE_COPY), ("put", D.DSPMV_EXCHANGE_PUT)):
            plan = D.dspmv_plan_create(comm, n, rp, col, val, exchange=ex)
            s = D.dspmv_schedule_create(plan, derive_ops(), 2)
            for mode, fn in (("host", D.dspmv_apply), ("graph", D.dspmv_apply_graph)):
                ys = []
                for _ in range(3):           # both PUT receive-buffer parities
                    y.fill_(float("nan"))
                    dist.barrier()
                    fn(s, x, y, stream)
                    torch.cuda.synchronize()
                    ys.append(y.cpu().numpy().copy())
                out[(ex_name, mode)] = ys
            D.dspmv_schedule_destroy(s)
            D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
        q.put((rank, lo, {f"{k[0]}/{k[1]}": [a.tolist() for a in v] for k, v in out.items()}))
    except Exception as e:  # noqa: BLE001
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mat", ["27pt", "powerlaw"])
def test_two_gpus_nccl_and_put_vs_oracle(mat):
    from oracle import plan as O2
    from oracle import schedules as S
    from oracle import spmv as O1
    import gen
    world = 2
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
        res[r] = ys
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n, (rp, col, val) = _mat(mat)
    x = gen.x_values((0, n), exact=(mat != "27pt"))
    plans = O2.plan_all(rp, col, n, world)
    yref = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(S.EDGES)[0]])
    s = O1.o1_absdot(rp, col, val, x)
    for key in res[0]:
        for k in range(3):
            y = np.concatenate([np.array(res[r][key][k]) for r in range(world)])
            if mat == "27pt":
                assert np.all(np.abs(y - yref) <= 1e-12 * s), (key, k)
            else:
                assert np.array_equal(y, yref), (key, k)
