"""Per-phase clock64 breakdown of the row-block kernel (instrumented build).
DSPMV_LIB=prof python scripts/prof_phases.py c4 [cfg]"""
import os, sys
os.environ["DSPMV_LIB"] = "prof"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2203_02530_b200 import dspmv as D
from paper_2203_02530_b200 import schedules as PS
w = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else -1
n, (rp, col, val) = gen.config_matrix(w)
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val, block_cfg=cfg)
info = D.dspmv_plan_info_get(plan)
ops = D.dspmv_schedule_derive(list(range(10)), [0] * 10, 2)
s = D.dspmv_schedule_create(plan, ops, 2)
x = torch.from_numpy(gen.x_values((0, n))).cuda(); y = torch.empty_like(x)
for _ in range(3): D.dspmv_apply(s, x, y)
D.dspmv_profile_counters(reset=True)
D.dspmv_schedule_set_timing(s, 1 << 2)
reps = 5
tt = 0
for _ in range(reps):
    D.dspmv_l2_flush(0); D.dspmv_apply(s, x, y); tt += D.dspmv_schedule_op_times(s)[2]
c = D.dspmv_profile_counters(reset=True)
blocks, passes = c[4] / reps, c[5] / reps
print(w, "cfg", cfg, "grid", info["grid_local"], "blocks", info["n_blocks_local"], "vrows", info["n_vrows_local"])
print(f"y_L {tt/reps*1e3:.1f} us; per block: producer wait-empty {c[0]/max(c[4],1):.0f} cyc, issue {c[1]/max(c[4],1):.0f} cyc; "
      f"per warp-pass: wait-full {c[2]/max(c[5],1):.0f} cyc, compute {c[3]/max(c[5],1):.0f} cyc")
