"""Sustained y_L on one workload: R back-to-back graph applies (no host sync,
no flush in between) timed with one event pair, after a warm-up, printing
the mean step.  B200 draws ~1 kW on C3 at full HBM bandwidth, so a long run
meets the power cap (sw_power_cap, lower SM clock) where the short bursts of
sell_sweep.py do not; this measures the capped steady state.

    python scripts/sustained.py [c3|c2|c4] [R]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
from paper_2203_02530_b200 import dspmv as D  # noqa: E402
from tests.gpu_helpers import derive_ops  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
n, (rp, col, val) = gen.config_matrix(w)
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val)
sched = D.dspmv_schedule_create(plan, derive_ops(), 2)
D.dspmv_schedule_set_caller_stream0(sched, 1)
x = torch.from_numpy(gen.x_values((0, n))).cuda()
y = torch.empty_like(x)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(20):
        D.dspmv_apply_graph(sched, x, y, s.cuda_stream)
    s.synchronize()
    for chunk in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.time()
        e0.record(s)
        for _ in range(R):
            D.dspmv_apply_graph(sched, x, y, s.cuda_stream)
        e1.record(s)
        e1.synchronize()
        print(f"{w} env={os.environ.get('DSPMV_L2PF', '-')} chunk {chunk}: {R} back-to-back applies, "
              f"{e0.elapsed_time(e1) / R * 1e3:.1f} us/step, {time.time() - t0:.1f} s", flush=True)
