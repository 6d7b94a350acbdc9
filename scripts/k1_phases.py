"""Phase split of the row-block kernel K1 (instrumented build, `make PROFILE=1`,
DSPMV_LIB=prof): clock64 totals summed over warps -- producer waiting for an
empty slot, producer issuing, consumers waiting for a full slot, consumer row
passes -- for one workload on one rank.  Tells whether K1 waits on the TMA
stream (consumers starve) or on its consumers (producer starves).

    DSPMV_LIB=prof python scripts/k1_phases.py [c3|c2]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
from paper_2203_02530_b200 import dspmv as D  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c3"
n, (rp, col, val) = gen.config_matrix(w)
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val)
info = D.dspmv_plan_info_get(plan)
ops = D.dspmv_schedule_derive(list(range(10)), [0] * 10, 1)
s = D.dspmv_schedule_create(plan, ops, 1)
x = torch.from_numpy(gen.x_values((0, n))).cuda()
y = torch.empty_like(x)
for _ in range(3):
    D.dspmv_apply(s, x, y)
torch.cuda.synchronize()
D.dspmv_profile_counters(reset=True)
reps = 20
for _ in range(reps):
    D.dspmv_l2_flush(0)
    D.dspmv_apply(s, x, y)
torch.cuda.synchronize()
c = D.dspmv_profile_counters(reset=True)
grid = info["grid_local"]
names = ["producer wait empty", "producer issue", "consumer wait full", "consumer rows", "blocks", "consumer passes"]
print(w, "grid", grid, "blocks/launch", c[4] // reps)
for i, nm in enumerate(names[:4]):
    per = c[i] / reps
    who = grid if i < 2 else grid * 8
    print(f"{nm:22s} total cycles/launch {per:.3e}  per CTA-or-warp {per / who:.3e}")
