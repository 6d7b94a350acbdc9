"""Replica of the apply_host pipeline with torch ops: 8 H2D chunks on s1,
per-chunk compute on s0 after chunk k+1, D2H chunk k on s2 after compute k."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
n = 2097152
xh = torch.randn(n, dtype=torch.float64).pin_memory(); yh = torch.empty(n, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda"); yd = torch.empty_like(xd)
s0, s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
K = 8; c = n // K
evx = [torch.cuda.Event() for _ in range(K)]; evy = [torch.cuda.Event() for _ in range(K)]

def pipe(d2h_chunks=True, lag=1):
    for k in range(K):
        with torch.cuda.stream(s1):
            xd[k * c:(k + 1) * c].copy_(xh[k * c:(k + 1) * c], non_blocking=True); evx[k].record()
    for k in range(K):
        with torch.cuda.stream(s0):
            s0.wait_event(evx[min(K - 1, k + lag)])
            torch.mul(xd[k * c:(k + 1) * c], 2.0, out=yd[k * c:(k + 1) * c]); evy[k].record()
        if d2h_chunks:
            with torch.cuda.stream(s2):
                s2.wait_event(evy[k]); yh[k * c:(k + 1) * c].copy_(yd[k * c:(k + 1) * c], non_blocking=True)
    if not d2h_chunks:
        with torch.cuda.stream(s0):
            yh.copy_(yd, non_blocking=True)
    torch.cuda.synchronize()

for args in ((True, 1), (True, 0), (False, 1)):
    for _ in range(5): pipe(*args)
    t0 = time.perf_counter()
    for _ in range(50): pipe(*args)
    print(f"replica d2h_chunks={args[0]} lag={args[1]}: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms")

def both_chunked(kh, kd):
    ch, cd = n // kh, n // kd
    with torch.cuda.stream(s1):
        for k in range(kh):
            xd[k * ch:(k + 1) * ch].copy_(xh[k * ch:(k + 1) * ch], non_blocking=True)
    with torch.cuda.stream(s2):
        for k in range(kd):
            yh[k * cd:(k + 1) * cd].copy_(yd[k * cd:(k + 1) * cd], non_blocking=True)
    torch.cuda.synchronize()

for kh, kd in ((1, 1), (8, 1), (1, 8), (8, 8), (32, 32)):
    for _ in range(5): both_chunked(kh, kd)
    t0 = time.perf_counter()
    for _ in range(50): both_chunked(kh, kd)
    print(f"concurrent H2D x{kh} chunks + D2H x{kd} chunks, no deps: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms")
