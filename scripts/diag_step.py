"""Where the C2 step's overhead around y_L comes from: y_L start offset and
step time after (a) the library's L2 flush, (b) a torch read of 2x L2, (c) no
flush, in host and graph execution, timing every GPU op or START/END + y_L
(the bench's mask)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2203_02530_b200 import dspmv as D

n, (rp, col, val) = gen.config_matrix("c2")
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val)
x = torch.from_numpy(gen.x_values((0, n))).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream()
V = D.VERTEX_NAMES
order = ["start", "y_L", "PostRecv", "Pack", "PostSend", "WaitRecv", "Unpack", "WaitSend", "y_R", "end"]
idx = [V.index(o) for o in order]
ops = D.dspmv_schedule_derive(idx, [1 if o == "Pack" else 0 for o in order], 2)
iyl = [i for i, o in enumerate(ops) if o[0] == D.DSPMV_OP_SPMV_LOCAL][0]
big = torch.empty(2 * 128 * 2**20 // 8, dtype=torch.float64, device="cuda")
sink = torch.empty(1, dtype=torch.float64, device="cuda")
flushes = {"dspmv": lambda: D.dspmv_l2_flush(0, st),
           "torch": lambda: sink.copy_(big.sum().reshape(1)),
           "none": lambda: None}
tag = os.environ.get("DSPMV_FLUSH_CARVEOUT", "default")
for mname, fn in (("host", D.dspmv_apply), ("graph", D.dspmv_apply_graph)):
    for mask_name, mask in (("every-op", 1), ("START+yL", 1 | (1 << D.DSPMV_OP_SPMV_LOCAL))):  # 1 = time every GPU op
        s = D.dspmv_schedule_create(plan, ops, 2)
        D.dspmv_schedule_set_timing(s, mask)
        for fl_name, fl in flushes.items():
            with torch.cuda.stream(st):
                for _ in range(10):
                    fl(); fn(s, x, y, st)
                steps, yl, b0, e0 = [], [], [], []
                for _ in range(200):
                    fl()
                    fn(s, x, y, st)
                    t = D.dspmv_schedule_op_times(s)
                    steps.append(t[0] * 1e3)
                    if mask != 1:
                        b, e = D.dspmv_schedule_op_timeline(s)
                        yl.append(t[iyl] * 1e3); b0.append(b[iyl] * 1e3); e0.append(e[iyl] * 1e3)
            extra = (f" yL {np.median(yl):6.2f} window [{np.median(b0):5.2f}, {np.median(e0):6.2f}]"
                     if yl else "")
            print(f"carveout={tag:7s} {mname:5s} {mask_name:9s} flush={fl_name:5s} step median "
                  f"{np.median(steps):6.2f} min {np.min(steps):6.2f}{extra}", flush=True)
        D.dspmv_schedule_destroy(s)
