"""Zero-copy y: the C2 SpMV with y in mapped pinned host memory vs device."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_2203_02530_b200 import dspmv as D

n, (rp, col, val) = gen.config_matrix("c2")
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
plan = D.dspmv_plan_create(comm, n, rp, col, val)
ops = D.dspmv_schedule_derive([0, 2, 1, 3, 4, 6, 7, 8, 5, 9], [0] * 10, 2)
s = D.dspmv_schedule_create(plan, ops, 2)
xd = torch.from_numpy(gen.x_values((0, n))).cuda()
yd = torch.empty_like(xd)
yh = torch.empty(n, dtype=torch.float64).pin_memory()
st = torch.cuda.Stream()

def t(fn, reps=100):
    for _ in range(5): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3

print(f"apply, y on device       {t(lambda: D.dspmv_apply(s, xd, yd, st)):.3f} ms")
print(f"apply, y in pinned host  {t(lambda: D.dspmv_apply(s, xd, yh, st)):.3f} ms")
assert torch.equal(yh, yd.cpu())
print(f"D2H copy of y            {t(lambda: yh.copy_(yd)):.3f} ms")
