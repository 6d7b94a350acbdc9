"""Column-panel experiment on C4: A = sum_b A[:, panel b].  Each panel is its
own 1-rank plan (same rows, only the columns of that x block), applied back
to back on one stream after one L2 flush; the sum of the panel times is set
against the single-plan time.  Tests whether keeping the gathered x block
L2-resident (x is 64 MB; ncu shows ~35 % of C4's gathers missing L2) beats
the extra passes over the rows.

    python scripts/c4_panels.py [--ks 1,2,4,8] [--kernels 2,4]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_2203_02530_b200 import dspmv as D  # noqa: E402
from tests.gpu_helpers import derive_ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--ks", default="1,2,4,8")
ap.add_argument("--kernels", default="2,4")
ap.add_argument("--vthr", type=int, default=64)
a = ap.parse_args()

t0 = time.time()
n, (rp, col, val) = gen.config_matrix("c4")
x = torch.from_numpy(gen.x_values((0, n))).cuda()
print(f"# c4: n={n} nnz={rp[-1]} generated in {time.time() - t0:.1f} s", flush=True)
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
stream = torch.cuda.Stream()
rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
ref = None
for sk in [int(k) for k in a.kernels.split(",")]:
    for K in [int(k) for k in a.ks.split(",")]:
        bounds = [n * b // K for b in range(K + 1)]
        plans, scheds, ys = [], [], []
        for b in range(K):
            m = (col >= bounds[b]) & (col < bounds[b + 1])
            rpb = np.zeros(n + 1, np.int64)
            np.cumsum(np.bincount(rows[m], minlength=n), out=rpb[1:])
            p = D.dspmv_plan_create(comm, n, rpb, col[m], val[m], s_kernel=sk, vector_threshold=a.vthr)
            s = D.dspmv_schedule_create(p, derive_ops(), 2)
            D.dspmv_schedule_set_caller_stream0(s, 1)
            plans.append(p)
            scheds.append(s)
            ys.append(torch.empty(n, dtype=torch.float64, device="cuda"))
        ts = []
        with torch.cuda.stream(stream):
            for i in range(a.reps + 3):
                D.dspmv_l2_flush(0, stream.cuda_stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for s, y in zip(scheds, ys):
                    D.dspmv_apply_graph(s, x, y, stream.cuda_stream)
                e1.record(stream)
                e1.synchronize()
                if i >= 3:
                    ts.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        ysum = sum(y.double() for y in ys).cpu().numpy()
        if ref is None:
            ref = ysum
        rel = float(np.max(np.abs(ysum - ref)) / np.max(np.abs(ref)))
        ms = float(np.median(ts))
        print(f"kernel {sk} K {K}: {ms:.4f} ms (min {min(ts):.4f})  {rp[-1] / ms / 1e6:.1f} G gathers/s  "
              f"max|y-y_K1|/max|y| {rel:.1e}", flush=True)
        for s in scheds:
            D.dspmv_schedule_destroy(s)
        for p in plans:
            D.dspmv_plan_destroy(p)
D.dspmv_comm_destroy(comm)
