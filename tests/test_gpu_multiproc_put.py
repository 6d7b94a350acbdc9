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
        D.dspmv_schedule_destroy(s)
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
        q.put((rank, lo, [a.tolist() for a in ys]))
    except Exception as e:  # noqa: BLE001
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mat", [(2, "pl"), (3, "27pt")])
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
    else:
        n = 24 ** 3
        rp, col, val = gen.stencil("27pt", (24, 24, 24))
    x = gen.x_values((0, n))
    yref = O1.o1_spmv(rp, col, val, x)
    s = O1.o1_absdot(rp, col, val, x)
    for k in range(4):
        y = np.concatenate([np.array(res[r][1][k]) for r in range(world)])
        assert np.all(np.abs(y - yref) <= 1e-12 * s), k
