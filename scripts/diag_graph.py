"""Step overhead of the executor around the y_L kernel (C2, P=1): host vs
graph execution, timing masks, y_L on the caller stream vs a forked stream."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2203_02530_b200 import dspmv as D
from paper_2203_02530_b200 import schedules as PS

n, (rp, col, val) = gen.config_matrix(sys.argv[1] if len(sys.argv) > 1 else "c2")
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val)
x = torch.from_numpy(gen.x_values((0, n))).cuda(); y = torch.empty_like(x)
st = torch.cuda.Stream()
V = D.VERTEX_NAMES
order = ["start", "y_L", "Pack", "PostSend", "PostRecv", "WaitRecv", "Unpack", "y_R", "WaitSend", "end"]
idx = [V.index(o) for o in order]
variants = {"yL@s0 all s0": [0] * 10,
            "yL@s1 rest s0": [1 if o == "y_L" else 0 for o in order],
            "yL@s0 rest s1": [1 if o in ("Pack", "Unpack", "y_R") else 0 for o in order]}
for vname, streams in variants.items():
    ops = D.dspmv_schedule_derive(idx, streams, 2)
    iyl = [i for i, o in enumerate(ops) if o[0] == D.DSPMV_OP_SPMV_LOCAL][0]
    for mname, fn in (("host", D.dspmv_apply), ("graph", D.dspmv_apply_graph)):
        for tname, mask in (("START", 1), ("START+yL", 1 | (1 << D.DSPMV_OP_SPMV_LOCAL))):
            s = D.dspmv_schedule_create(plan, ops, 2)
            D.dspmv_schedule_set_timing(s, mask)
            for _ in range(10):
                fn(s, x, y, st)
            steps, yl, b0 = [], [], []
            for _ in range(200):
                D.dspmv_l2_flush(0, st)
                fn(s, x, y, st)
                t = D.dspmv_schedule_op_times(s)
                steps.append(t[0] * 1e3)
                if mask != 1:
                    b, e = D.dspmv_schedule_op_timeline(s)
                    yl.append(t[iyl] * 1e3); b0.append(b[iyl] * 1e3)
            extra = f" yL {np.median(yl):6.2f} us starts at {np.median(b0):5.2f}" if yl else ""
            print(f"{vname:16s} {mname:5s} {tname:9s} step median {np.median(steps):6.2f} mean {np.mean(steps):6.2f}{extra}",
                  flush=True)
            D.dspmv_schedule_destroy(s)
