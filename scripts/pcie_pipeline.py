"""The copy-only bound of dspmv_apply_host's pipeline at C3 size: x goes H2D
in K chunks on one stream, y comes back D2H in K chunks on another, chunk k
of y released when x chunk k+lag has landed (the stencil halo needs the next
chunk) -- no kernel at all.  Compared with the two directions fully
concurrent (the pcie_frac floor) it shows how much of the e2e gap is the
pipeline's fill and drain rather than the SpMV.

    python scripts/pcie_pipeline.py [n_rows]
"""
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
xh = torch.empty(n, dtype=torch.float64).pin_memory()
yh = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.zeros_like(xd)
sx, sy = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    ts = []
    for _ in range(reps + 2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in (sx, sy):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts[2:])[len(ts[2:]) // 2]


def pipeline(K, lag):
    c = (n + K - 1) // K
    ev = [torch.cuda.Event() for _ in range(K)]
    start = torch.cuda.Event()
    start.record()
    sx.wait_event(start)
    sy.wait_event(start)
    for k in range(K):
        with torch.cuda.stream(sx):
            xd[k * c:(k + 1) * c].copy_(xh[k * c:(k + 1) * c], non_blocking=True)
            ev[k].record()
    for k in range(K):
        with torch.cuda.stream(sy):
            sy.wait_event(ev[min(K - 1, k + lag)])
            yh[k * c:(k + 1) * c].copy_(yd[k * c:(k + 1) * c], non_blocking=True)


def both():
    start = torch.cuda.Event()
    start.record()
    sx.wait_event(start)
    sy.wait_event(start)
    with torch.cuda.stream(sx):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(sy):
        yh.copy_(yd, non_blocking=True)


mb = n * 8 / 1e6
t = timed(lambda: xd.copy_(xh, non_blocking=True))
print(f"H2D alone {mb:.0f} MB: {t:.3f} ms ({mb / t:.1f} GB/s)")
t = timed(lambda: yh.copy_(yd, non_blocking=True))
print(f"D2H alone {mb:.0f} MB: {t:.3f} ms ({mb / t:.1f} GB/s)")
t = timed(both)
print(f"H2D + D2H concurrent: {t:.3f} ms ({2 * mb / t:.1f} GB/s both ways)")
for K in (8, 16, 32):
    for lag in (0, 1, 2):
        print(f"pipeline K={K:2d} lag={lag}: {timed(lambda: pipeline(K, lag)):.3f} ms")
