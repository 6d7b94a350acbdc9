"""PCIe bounds for the e2e path: pinned H2D and D2H of 16.7 MB alone and
concurrently (two streams), and dspmv_apply_host on C2 with the pipeline."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2203_02530_b200 import dspmv as D

nb = 16777216
h1 = torch.empty(nb, dtype=torch.uint8).pin_memory(); h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d1 = torch.empty(nb, dtype=torch.uint8, device="cuda"); d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def t(fn, reps=50):
    for _ in range(5): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3

def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
def chunked(k=8):
    c = nb // k
    for i in range(k):
        with torch.cuda.stream(s1): d1[i*c:(i+1)*c].copy_(h1[i*c:(i+1)*c], non_blocking=True)
print(f"H2D 16.7MB {t(h2d):.3f} ms  D2H {t(d2h):.3f} ms  both concurrent {t(both):.3f} ms  H2D in 8 chunks {t(chunked):.3f} ms")
n, (rp, col, val) = gen.config_matrix("c2")
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val)
ops = D.dspmv_schedule_derive([0, 2, 1, 3, 4, 6, 7, 8, 5, 9], [0] * 10, 2)
s = D.dspmv_schedule_create(plan, ops, 2)
xh = torch.from_numpy(gen.x_values((0, n))).pin_memory(); yh = torch.empty(n, dtype=torch.float64).pin_memory()
st = torch.cuda.Stream()
print(f"apply_host pipelined C2 {t(lambda: D.dspmv_apply_host(s, xh, yh, st), 100):.3f} ms")
xp = torch.from_numpy(gen.x_values((0, n))); yp = torch.empty(n, dtype=torch.float64)
print(f"apply_host pageable C2 {t(lambda: D.dspmv_apply_host(s, xp, yp, st), 30):.3f} ms")
D.dspmv_schedule_set_timing(s, 1 | (1 << D.DSPMV_OP_SPMV_LOCAL))
iyl = [i for i, o in enumerate(ops) if o[0] == D.DSPMV_OP_SPMV_LOCAL][0]
for _ in range(5):
    D.dspmv_apply_host(s, xh, yh, st)
b, e = D.dspmv_schedule_op_timeline(s)
print(f"timeline (ms from START): y_L {b[iyl]:.3f}..{e[iyl]:.3f}  END {e[0]:.3f}")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(100):
    D.dspmv_apply_host(s, xh, yh, st)
print(f"wall per apply_host {(time.perf_counter() - t0) * 10:.3f} ms")
