"""Measured host<->device copy bandwidth (pinned memory) -- the ceiling of the
e2e leg of bench.py (x H2D + y D2H every step).  Writes profiles/pcie_peak.json.

    python scripts/pcie_peak.py [--mib 64] [--reps 20]

Each direction: torch copy_ of a pinned host tensor to / from a device tensor
(cudaMemcpyAsync), timed with CUDA events on the copy stream, best of `reps`.
Also both directions at once on two streams (the copy engines are separate).
"""
import argparse
import json
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def timed(fn, stream, reps):
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    nbytes = a.mib << 20
    h_src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        for _ in range(3):
            d_a.copy_(h_src, non_blocking=True)
            h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        h2d = timed(lambda: d_a.copy_(h_src, non_blocking=True), s1, a.reps)
        d2h = timed(lambda: h_dst.copy_(d_b, non_blocking=True), s1, a.reps)

    def both():
        ev = torch.cuda.Event()
        ev.record(s1)
        s2.wait_event(ev)
        d_a.copy_(h_src, non_blocking=True)
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s1.wait_event(ev2)
    with torch.cuda.stream(s1):
        bidir = timed(both, s1, a.reps)
    out = {"h2d_GB_s": round(nbytes / (h2d * 1e-3) / 1e9, 2),
           "d2h_GB_s": round(nbytes / (d2h * 1e-3) / 1e9, 2),
           "bidir_GB_s_total": round(2 * nbytes / (bidir * 1e-3) / 1e9, 2),
           "bytes": nbytes, "reps": a.reps, "method": "pinned host <-> device copy_, CUDA events, best of reps",
           "gpu": torch.cuda.get_device_name()}
    print(json.dumps(out))
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "pcie_peak.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
