"""C4 y_L by S-group kernel: the CSR-stream kernel (K1b) against the sliced
kernel (K1d, DSPMV_SKERNEL_SELL) over its window / unroll settings, on the
full BASELINE configs[3] matrix at 1 rank (a GPU-resident graph on one
stream, L2 flushed before every apply, CUDA events around each apply).
Every variant's y must equal K1b's bit for bit (both are the serial loop on
rows <= 256 nnz, and the same long-row kernel above).

    python scripts/sell_sweep.py [--reps 30] [--cfgs stream,sell:256:8,...]
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
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--workload", default="c4")
ap.add_argument("--long-row-sum", type=int, default=0, help="1: DSPMV_LONG_ROW_STORED")
ap.add_argument("--flush", type=int, default=1, help="flush L2 before each apply (0: back-to-back applies)")
ap.add_argument("--cfgs", default="stream,sell:256:8:256:4096,sell:1024:8:256:4096,sell:4096:8:256:4096,"
                "sell:256:8:64:4096,sell:1024:8:64:4096,sell:1024:8:128:4096,sell:1024:8:32:4096,"
                "sell:1024:4:64:4096,sell:1024:16:64:4096,sell:1024:8:64:16384,sell:1024:8:64:1024,stream")
a = ap.parse_args()

t0 = time.time()
n, (rp, col, val) = gen.config_matrix(a.workload)
x = torch.from_numpy(gen.x_values((0, n))).cuda()
print(f"# {a.workload}: n={n} nnz={rp[-1]} generated in {time.time() - t0:.1f} s", flush=True)
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
stream = torch.cuda.Stream()
ref = None
for c in a.cfgs.split(","):
    parts = c.split(":")   # sell:window:unroll[:vector_threshold[:chunk_cost[:ctas_per_sm[:x_in_L1]]]]
    vthr = -1
    bcfg = -1
    if parts[0] == "sell":
        os.environ["DSPMV_SELL_WINDOW"] = parts[1]
        os.environ["DSPMV_SELL_UNROLL"] = parts[2]
        if len(parts) > 3:
            vthr = int(parts[3])
        if len(parts) > 4:
            os.environ["DSPMV_SELL_CHUNK"] = parts[4]
        if len(parts) > 5:
            os.environ["DSPMV_SELL_CTAS"] = parts[5]
        if len(parts) > 6:
            os.environ["DSPMV_SELL_L1"] = parts[6]
        sk = D.DSPMV_SKERNEL_SELL
    elif parts[0] in ("auto", "cfg"):   # auto[:l2_prefetch_distance] / cfg:block_cfg[:l2_prefetch_distance]
        sk = D.DSPMV_SKERNEL_AUTO
        if parts[0] == "cfg":
            bcfg = int(parts[1])
            parts = parts[1:]
        os.environ["DSPMV_L2PF"] = parts[1] if len(parts) > 1 else "1"
    else:
        sk = D.DSPMV_SKERNEL_STREAM
    t1 = time.time()
    plan = D.dspmv_plan_create(comm, n, rp, col, val, s_kernel=sk, vector_threshold=vthr, block_cfg=bcfg,
                                 long_row_sum=a.long_row_sum)
    tp = time.time() - t1
    info = D.dspmv_plan_info_get(plan)
    sched = D.dspmv_schedule_create(plan, derive_ops(), 2)
    D.dspmv_schedule_set_caller_stream0(sched, 1)
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    gbytes = (12 * int(rp[-1]) + 4 * (n + 1) + 16 * n) / 1e9   # SURVEY 8(d) algorithmic bytes
    ts = []
    with torch.cuda.stream(stream):
        for i in range(a.reps + 3):
            if a.flush:
                D.dspmv_l2_flush(0, stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            D.dspmv_apply_graph(sched, x, y, stream.cuda_stream)
            e1.record(stream)
            e1.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    yh = y.cpu().numpy()
    if ref is None:
        ref = yh
    same = bool(np.array_equal(yh.view(np.int64), ref.view(np.int64)))
    rel = float(np.max(np.abs(yh - ref)) / max(1e-300, np.max(np.abs(ref))))
    ms = float(np.median(ts))
    nnz = int(rp[-1])
    print(f"{c:16s} kernel={info['s_kernel_local']} yL_ms {ms:.4f} min {min(ts):.4f} "
          f"G_gathers/s {nnz / ms / 1e6:.1f} TB/s {gbytes / ms:.3f} plan_s {tp:.1f} bitwise_eq_first {same} maxrel {rel:.1e}", flush=True)
    D.dspmv_schedule_destroy(sched)
    D.dspmv_plan_destroy(plan)
D.dspmv_comm_destroy(comm)
