"""Per-op device timeline of one apply (C2, P=1) for a few schedules, and the
pure executor overhead on an empty matrix."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, time
import gen
from paper_2203_02530_b200 import dspmv as D
from paper_2203_02530_b200 import schedules as PS

def run(n, rp, col, val, label, flush=True, reps=50):
    uid = D.dspmv_comm_unique_id(); comm = D.dspmv_comm_create(uid, 1, 0, 0)
    plan = D.dspmv_plan_create(comm, n, rp, col, val)
    x = torch.from_numpy(gen.x_values((0, n))).cuda(); y = torch.empty_like(x)
    st = torch.cuda.current_stream()
    all_ops = PS.enumerate_derived(2)
    picks = [all_ops[0], all_ops[len(all_ops)//2], all_ops[-1]]
    for ops in picks:
        s = D.dspmv_schedule_create(plan, ops, 2)
        D.dspmv_schedule_set_timing(s, 1 | (1 << 0) | 0x1FE)
        for _ in range(5): D.dspmv_apply(s, x, y, st)
        tot = []; tl = None
        for _ in range(reps):
            if flush: D.dspmv_l2_flush(0, st)
            D.dspmv_apply(s, x, y, st)
            b, e = D.dspmv_schedule_op_timeline(s)
            tot.append(e[0]); tl = (b, e)
        b, e = tl
        print(f"[{label}] step median {np.median(tot)*1e3:.1f} us  sched: {PS.describe(ops)}")
        for i, o in enumerate(ops):
            if b[i] >= 0 and i > 0:
                print(f"     op {i:2d} {D.VERTEX_NAMES[o[0]] if o[0] < 10 else o[0]:8s} s{o[1]}  {b[i]*1e3:8.2f} .. {e[i]*1e3:8.2f} us")
        # host wall
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(200): D.dspmv_apply(s, x, y, st)
        print(f"     host wall per apply (no flush, back-to-back): {(time.perf_counter()-t0)/200*1e6:.1f} us")
        D.dspmv_schedule_destroy(s)
    D.dspmv_plan_destroy(plan); D.dspmv_comm_destroy(comm)

n = 1 << 20
run(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0), "empty", flush=False)
n, (rp, col, val) = gen.config_matrix("c2")
run(n, rp, col, val, "c2")
