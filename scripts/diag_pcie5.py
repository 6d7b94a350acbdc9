"""A/B of the apply_host chunk count in one process (plans built with
DSPMV_HOST_CHUNKS = K), measurements interleaved."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen
from paper_2203_02530_b200 import dspmv as D

n, (rp, col, val) = gen.config_matrix("c2")
comm = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)
ops = D.dspmv_schedule_derive([0, 2, 1, 3, 4, 6, 7, 8, 5, 9], [0] * 10, 2)
runs = {}
for K in (1, 2, 4, 6, 8, 12):
    os.environ["DSPMV_HOST_CHUNKS"] = str(K)
    p = D.dspmv_plan_create(comm, n, rp, col, val)
    runs[K] = (p, D.dspmv_schedule_create(p, ops, 2))
xh = torch.from_numpy(gen.x_values((0, n))).pin_memory(); yh = torch.empty(n, dtype=torch.float64).pin_memory()
st = torch.cuda.Stream()
res = {K: [] for K in runs}
for rep in range(6):
    for K, (p, s) in runs.items():
        for _ in range(3): D.dspmv_apply_host(s, xh, yh, st)
        t0 = time.perf_counter()
        for _ in range(50): D.dspmv_apply_host(s, xh, yh, st)
        res[K].append((time.perf_counter() - t0) / 50 * 1e3)
for K, v in res.items():
    print(f"K={K:2d}: median {np.median(v):.3f} ms  min {min(v):.3f}")
