"""Helpers for the GPU parity tests: run the CUDA path through the C ABI on an
in-process LOCAL group (P simulated ranks sharing cuda:0) or a 1-rank NCCL
communicator, and fetch the global y."""
import numpy as np
import torch

import gen
from oracle import schedules as S
from paper_2203_02530_b200 import dspmv as D

KIND = {v: i for i, v in enumerate(S.VERTICES)}
GPUS = ["Pack", "y_L", "Unpack", "y_R"]

# A class-1-shaped schedule: Pack before y_L on different streams,
# y_L launched before CES-b4-PostSend.
BEST_ORDER = ["start", "PostRecv", "Pack", "y_L", "PostSend", "WaitRecv", "Unpack", "y_R",
              "WaitSend", "end"]
BEST_STREAMS = {"Pack": 0, "y_L": 1, "Unpack": 0, "y_R": 0}


def derive_ops(order=BEST_ORDER, streams=BEST_STREAMS, n_streams=2):
    return D.dspmv_schedule_derive([KIND[v] for v in order],
                                   [streams.get(v, 0) for v in order], n_streams)


def oracle_ops_to_lib(ops):
    out = []
    for op in ops:
        n = op[0]
        b, d = S.split_name(n)
        if b in KIND:
            out.append((KIND[b], op[1] if b in S.GPU_VERTICES else 0, 0, d))
        elif n == "CER":
            out.append((D.DSPMV_OP_EVENT_RECORD, op[1], op[2], 0))
        elif n == "CES":
            out.append((D.DSPMV_OP_EVENT_SYNC, 0, op[1], 0))
        else:
            out.append((D.DSPMV_OP_STREAM_WAIT_EVENT, op[1], op[2], 0))
    return out


class LocalRun:
    """P LOCAL ranks on cuda:0 holding the row blocks of one global matrix."""

    def __init__(self, n, rp, col, val, P, dtype=D.DSPMV_F64, vector_threshold=-1,
                 keep_host=False, block_cfg=-1, exchange=D.DSPMV_EXCHANGE_COPY, s_kernel=D.DSPMV_SKERNEL_AUTO,
                 **opts):
        self.n, self.P, self.dtype = n, P, dtype
        self.tdt = torch.float32 if dtype == D.DSPMV_F32 else torch.float64
        self.rb = D.dspmv_partition(n, P)
        self.comms = D.dspmv_comm_create_local(P, 0)
        self.plans = []
        for r in range(P):
            b, e = int(self.rb[r]), int(self.rb[r + 1])
            rpr = rp[b:e + 1]
            lo, hi = int(rpr[0]), int(rpr[-1])
            self.plans.append(D.dspmv_plan_create(self.comms[r], n, rpr, col[lo:hi], val[lo:hi],
                                                  dtype=dtype, vector_threshold=vector_threshold,
                                                  keep_host=keep_host, block_cfg=block_cfg, s_kernel=s_kernel,
                                                  exchange=exchange, **opts))
        self.scheds = []

    def schedule(self, ops, n_streams=2):
        ss = [D.dspmv_schedule_create(p, ops, n_streams) for p in self.plans]
        self.scheds.append(ss)
        return ss

    def xy(self, x_global):
        xs, ys = [], []
        for r in range(self.P):
            b, e = int(self.rb[r]), int(self.rb[r + 1])
            xs.append(torch.from_numpy(np.ascontiguousarray(x_global[b:e])).to("cuda", self.tdt))
            ys.append(torch.full((e - b,), float("nan"), dtype=self.tdt, device="cuda"))
        return xs, ys

    def apply(self, scheds, x_global, reps=1):
        xs, ys = self.xy(x_global)
        for _ in range(reps):
            for y in ys:
                y.fill_(float("nan"))
            D.dspmv_apply_group(scheds, xs, ys)
        torch.cuda.synchronize()
        return np.concatenate([y.cpu().numpy() for y in ys]).astype(np.float64)

    def close(self):
        for ss in self.scheds:
            for s in ss:
                D.dspmv_schedule_destroy(s)
        for p in self.plans:
            D.dspmv_plan_destroy(p)
        for c in self.comms:
            D.dspmv_comm_destroy(c)


def within_tol(y, yref, scale, rel):
    return np.all(np.abs(y - yref) <= rel * scale) and np.array_equal(np.isnan(y), np.isnan(yref))
