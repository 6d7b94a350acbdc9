"""dspmv_apply_host (the end-to-end path): with pinned x/y the transfers are
pipelined with y_L (x in chunks, finished y rows streamed back while later row
blocks compute); results must be bitwise those of dspmv_apply on device
buffers, for pinned and pageable host memory, fp64 and fp32, with long rows
(V group) and for several schedules."""
import numpy as np
import pytest
import torch

import gen
from oracle import spmv as O1
from paper_2203_02530_b200 import dspmv as D
from tests.gpu_helpers import derive_ops

pytestmark = pytest.mark.gpu

ORDERS = [
    (["start", "y_L", "Pack", "PostSend", "PostRecv", "WaitRecv", "Unpack", "y_R", "WaitSend", "end"], {}),
    (["start", "PostRecv", "Pack", "y_L", "PostSend", "WaitRecv", "Unpack", "y_R", "WaitSend", "end"],
     {"Pack": 0, "y_L": 1, "Unpack": 0, "y_R": 1}),
    (["start", "Pack", "PostSend", "PostRecv", "WaitSend", "WaitRecv", "Unpack", "y_R", "y_L", "end"],
     {"y_R": 1}),
]


def _case(name):
    if name == "7pt96":
        return 96 ** 3, gen.stencil("7pt", (96, 96, 96))
    if name == "7pt97":  # odd n: x bytes not a multiple of 16
        return 97 ** 3, gen.stencil("7pt", (97, 97, 97))
    if name == "pl400k":
        n = 400000
        return n, gen.powerlaw(n)
    raise KeyError(name)


@pytest.mark.parametrize("dtype", [D.DSPMV_F64, D.DSPMV_F32], ids=["f64", "f32"])
@pytest.mark.parametrize("name", ["7pt96", "7pt97", "pl400k", "pl400k-sell"])
def test_apply_host_pipelined_equals_device_apply(name, dtype):
    skern = D.DSPMV_SKERNEL_SELL if name.endswith("-sell") else D.DSPMV_SKERNEL_AUTO
    n, (rp, col, val) = _case(name.replace("-sell", ""))
    tdt = torch.float32 if dtype == D.DSPMV_F32 else torch.float64
    npdt = np.float32 if dtype == D.DSPMV_F32 else np.float64
    v = val.astype(npdt)
    comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, v, dtype=dtype, vector_threshold=64, s_kernel=skern)
    x = gen.x_values((0, n)).astype(npdt)
    xd = torch.from_numpy(x).cuda()
    try:
        for order, streams in ORDERS:
            ops = derive_ops(order, streams)
            s = D.dspmv_schedule_create(plan, ops, 2)
            yd = torch.empty_like(xd)
            D.dspmv_apply(s, xd, yd)
            want = yd.cpu().numpy()
            xp = torch.from_numpy(x).pin_memory()
            for pinned in (True, False):
                xh = xp if pinned else torch.from_numpy(x.copy())
                yh = torch.full((n,), float("nan"), dtype=tdt)
                if pinned:
                    yh = yh.pin_memory()
                for _ in range(2):
                    yh.fill_(float("nan"))
                    D.dspmv_apply_host(s, xh, yh)
                    assert np.array_equal(yh.numpy().view(np.uint8), want.view(np.uint8)), (order, pinned)
            D.dspmv_schedule_destroy(s)
        if dtype == D.DSPMV_F64:
            y1 = O1.o1_spmv(rp, col, val, x)
            assert np.all(np.abs(want - y1) <= 1e-12 * O1.o1_absdot(rp, col, val, x))
    finally:
        D.dspmv_plan_destroy(plan)
        D.dspmv_comm_destroy(comm)
