"""Is chunked H2D slowed by a concurrent HBM-saturating kernel?  And the
pipelined apply_host with spin vs blocking host waits."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
nb = 16777216
h1 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d1 = torch.empty(nb, dtype=torch.uint8, device="cuda")
big_a = torch.empty(1 << 28, dtype=torch.uint8, device="cuda"); big_b = torch.empty_like(big_a)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

def h2d_time(with_kernel):
    torch.cuda.synchronize()
    if with_kernel:
        with torch.cuda.stream(s2):
            for _ in range(8):
                big_b.copy_(big_a, non_blocking=True)   # ~8 x 80 us of HBM streaming
    with torch.cuda.stream(s1):
        e0.record()
        c = nb // 8
        for i in range(8):
            d1[i * c:(i + 1) * c].copy_(h1[i * c:(i + 1) * c], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)

for wk in (False, True, False, True):
    ts = sorted(h2d_time(wk) for _ in range(20))
    print(f"chunked H2D 16.7 MB, concurrent HBM copy kernel={wk}: median {ts[10]:.3f} ms")
