"""bench.py's host-side pieces (no GPU): the workload table matches BASELINE
configs, both arms print the same workload string, the sampled-row parity
self-check accepts a correct y and rejects a wrong one, and the secondary
workload policy."""
import argparse
import json
import os

import numpy as np

import bench
import gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_workloads_are_the_baseline_configs():
    cfgs = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert bench.workload_n("c2") == 128 ** 3 and "128" in cfgs[1]
    assert bench.workload_n("c3") == 256 ** 3 and "256" in cfgs[2] and "27-point" in cfgs[2]
    assert bench.workload_n("c4") == 1 << 23 and "8M" in cfgs[3]
    assert bench.workload_n("c5") == 192 ** 3 and "192" in cfgs[4]
    # same string in both arms for the same N (the driver's same_config check)
    assert bench.workload_desc("c3", 8) == bench.workload_desc("c3", 8)
    assert "over 8 rank(s)" in bench.workload_desc("c3", 8)


def test_parity_sample_accepts_correct_and_rejects_wrong_y():
    n = 24 ** 3
    lo, hi = 4000, 9000
    rp, col, val = gen.stencil("27pt", (24, 24, 24), (lo, hi))
    sample = bench.parity_sample(rp, col, val, lo, hi, n, np.float64)
    rows, yref, scale = sample
    assert rows.min() == 0 and rows.max() == hi - lo - 1
    # the rows with remote entries (columns outside [lo, hi)) are sampled too
    has_remote = np.array([np.any((col[rp[i] - rp[0]:rp[i + 1] - rp[0]] < lo) |
                                  (col[rp[i] - rp[0]:rp[i + 1] - rp[0]] >= hi)) for i in rows])
    assert has_remote.any()
    x = gen.x_values((0, n))
    y = np.array([np.dot(val[rp[i] - rp[0]:rp[i + 1] - rp[0]], x[col[rp[i] - rp[0]:rp[i + 1] - rp[0]]])
                  for i in range(hi - lo)])
    ok, worst = bench.check_parity(sample, y, 1e-12)
    assert ok and worst < 1e-14
    bad = y.copy()
    bad[rows[len(rows) // 2]] += 1e-6
    assert not bench.check_parity(sample, bad, 1e-12)[0]
    bad = y.copy()
    bad[rows[-1]] = np.nan
    assert not bench.check_parity(sample, bad, 1e-12)[0]


def test_secondary_policy():
    a = argparse.Namespace(secondary="auto", workload="c3")
    assert bench.secondaries(a, 1) == ["c4", "c2"]
    assert bench.secondaries(a, 8) == ["c4"]
    a.workload = "c4"
    assert bench.secondaries(a, 1) == ["c2"]
    a.secondary = "none"
    assert bench.secondaries(a, 1) == []
    a.secondary = "c2,c4"
    assert bench.secondaries(a, 2) == ["c2"]
