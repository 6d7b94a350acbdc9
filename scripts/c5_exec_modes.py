"""C5 (7-pt 192^3 over 4 ranks) on one B200: step time of the class-1
schedule under each execution model -- host-synchronised lock-step group
(dspmv_apply_group) vs one GPU-resident graph (dspmv_apply_graph_group), each
with the NCCL-analogue device copy exchange and the fused Pack+put exchange,
gather Pack vs aliased sends.  The verdict's NEXT-3 measurement (P:244 host
blocking).  Prints one JSON object; L2 flushed before each step,
CUDA events on the caller stream, median of 100 steps.

    python scripts/c5_exec_modes.py [--out profiles/r2_c5_exec_modes.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
from paper_2203_02530_b200 import dspmv as D  # noqa: E402

ORDER = ["start", "PostRecv", "Pack", "y_L", "PostSend", "WaitRecv", "Unpack", "y_R", "WaitSend", "end"]
STREAMS = {"Pack": 0, "y_L": 1, "Unpack": 0, "y_R": 0}
VERTS = ["start", "Pack", "y_L", "PostSend", "PostRecv", "WaitSend", "WaitRecv", "Unpack", "y_R", "end"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--ranks", type=int, default=4)
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    n, (rp, col, val) = gen.config_matrix("c5")
    x = gen.x_values((0, n))
    P = a.ranks
    rb = D.dspmv_partition(n, P)
    ops = D.dspmv_schedule_derive([VERTS.index(v) for v in ORDER], [STREAMS.get(v, 0) for v in ORDER], 2)
    stream = torch.cuda.Stream()
    out = {"workload": "c5: 7-pt 192^3 fp64 over %d in-process ranks on one B200" % P,
           "schedule": " ".join(ORDER) + f" streams={STREAMS}", "steps": a.steps, "results": {}}
    ref = None
    for ex_name, ex in (("copy", D.DSPMV_EXCHANGE_COPY), ("put", D.DSPMV_EXCHANGE_PUT)):
        for pm_name, pm, um in (("gather", D.DSPMV_PACK_GATHER, D.DSPMV_UNPACK_COPY),
                                ("alias", D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS, D.DSPMV_UNPACK_COPY),
                                ("alias+fused-unpack", D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS, D.DSPMV_UNPACK_FUSED),
                                ("gather+fused-unpack", D.DSPMV_PACK_GATHER, D.DSPMV_UNPACK_FUSED)):
            if ex_name == "put" and pm_name.startswith("alias"):
                continue   # the put already fuses the gather with the store
            comms = D.dspmv_comm_create_local(P, 0)
            plans, xs, ys = [], [], []
            for r in range(P):
                b, e = int(rb[r]), int(rb[r + 1])
                lo, hi = int(rp[b]), int(rp[e])
                plans.append(D.dspmv_plan_create(comms[r], n, rp[b:e + 1], col[lo:hi], val[lo:hi], exchange=ex,
                                                 pack_mode=pm, unpack_mode=um))
                xs.append(torch.from_numpy(x[b:e].copy()).cuda())
                ys.append(torch.empty(e - b, dtype=torch.float64, device="cuda"))
            ss = [D.dspmv_schedule_create(p, ops, 2) for p in plans]
            for mode, fn in (("host", lambda: D.dspmv_apply_group(ss, xs, ys, stream)),
                             ("graph", lambda: D.dspmv_apply_graph_group(ss, xs, ys, stream))):
                for _ in range(10):
                    fn()
                torch.cuda.synchronize()
                ts = []
                for _ in range(a.steps):
                    D.dspmv_l2_flush(0, stream)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    fn()
                    e1.record(stream)
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e3)
                y = torch.cat(ys).cpu().numpy()
                if ref is None:
                    ref = y
                key = f"{mode}/{ex_name}/{pm_name}"
                out["results"][key] = {"step_us_median": round(float(np.median(ts)), 2),
                                       "step_us_min": round(float(np.min(ts)), 2),
                                       "bitwise_equal_to_first": bool(np.array_equal(y, ref)),
                                       "pack_alias": D.dspmv_plan_info_get(plans[0])["pack_alias"]}
            for s in ss:
                D.dspmv_schedule_destroy(s)
            for p in plans:
                D.dspmv_plan_destroy(p)
            for c in comms:
                D.dspmv_comm_destroy(c)
    print(json.dumps(out, indent=1))
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
