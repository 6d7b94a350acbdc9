"""World-size-2 (and 3) gloo tests of the N>1 host path: NCCL-id bootstrap
through torch.distributed, and the distributed planning protocol (each rank
plans only its own rows, exchanges request lists with the owners, builds its
pack map) -- compared bit-exactly with the oracle's global planner."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mat, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        from paper_2203_02530_b200 import dspmv as D
        # 1. NCCL unique-id bootstrap as bench.py does it
        uid = D.dspmv_comm_unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert all(i == ids[0] for i in ids) and len(ids[0]) == 128
        # 2. distributed planning protocol on this rank's rows only
        if mat == "7pt":
            dims = (8, 8, 4 * world)
            n = dims[0] * dims[1] * dims[2]
            rb = D.dspmv_partition(n, world)
            rp, col, val = gen.stencil("7pt", dims, (int(rb[rank]), int(rb[rank + 1])))
        else:
            n = 3000
            rb = D.dspmv_partition(n, world)
            rp, col, val = gen.powerlaw(n, (int(rb[rank]), int(rb[rank + 1])))
        hp = D.dspmv_rank_plan_build_host(world, rank, n, rp, col, val)
        mine = [D.dspmv_host_plan_requests(hp, o) for o in range(world)]
        allreq = [None] * world
        dist.all_gather_object(allreq, mine)
        D.dspmv_host_plan_set_requests(hp, [allreq[r][rank] for r in range(world)])
        out = {w: D.dspmv_host_plan_export(hp, 0, getattr(D, "DSPMV_" + w))
               for w in ("HALO_GID", "RECV_COUNTS", "RECV_DISPL", "SEND_COUNTS", "SEND_DISPL",
                         "PACK_MAP", "AL_ROWPTR", "AL_COL", "AR_ROWS", "AR_ROWPTR", "AR_COL")}
        D.dspmv_host_plan_destroy(hp)
        # 3. max-over-ranks timing reduction as bench.py does it
        import torch
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
        q.put((rank, {k: v.tolist() for k, v in out.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mat", [(2, "7pt"), (2, "powerlaw"), (3, "powerlaw")])
def test_distributed_planning_protocol_gloo(world, mat):
    import gen
    from oracle import plan as O2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mat, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if mat == "7pt":
        dims = (8, 8, 4 * world)
        n = dims[0] * dims[1] * dims[2]
        rp, col, val = gen.stencil("7pt", dims)
    else:
        n = 3000
        rp, col, val = gen.powerlaw(n)
    ref = O2.plan_all(rp, col, n, world)
    key = {"HALO_GID": "halo_gid", "RECV_COUNTS": "recv_count", "RECV_DISPL": "recv_displ",
           "SEND_COUNTS": "send_count", "SEND_DISPL": "send_displ", "PACK_MAP": "pack_map",
           "AL_ROWPTR": "al_rowptr", "AL_COL": "al_col", "AR_ROWS": "ar_rows",
           "AR_ROWPTR": "ar_rowptr", "AR_COL": "ar_col"}
    for r in range(world):
        for w, k in key.items():
            assert res[r][w] == list(np.asarray(ref[r][k]).tolist()), (r, w)


def test_set_requests_rejects_foreign_ids():
    import gen
    from paper_2203_02530_b200 import dspmv as D
    rp, col, val = gen.stencil("7pt", (4, 4, 4), (0, 32))
    hp = D.dspmv_rank_plan_build_host(2, 0, 64, rp, col, val)
    with pytest.raises(D.DspmvError):
        D.dspmv_host_plan_set_requests(hp, [np.zeros(0, np.int32), np.array([40], np.int32)])
    D.dspmv_host_plan_destroy(hp)
