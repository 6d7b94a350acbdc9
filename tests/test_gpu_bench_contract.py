"""bench.py keeps the driver's JSON-line contract (ours and --impl reference)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1 and lines[0].startswith("{"), r.stdout   # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_bench_line_ours():
    d = _run("--steps", "20", "--warmup", "3", "--no-cpu-baseline", "--rerank", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
              "clocks", "schedule_sweep", "parity_ok", "secondary"):
        assert k in d, k
    assert d["parity_ok"] is True and set(d["secondary"]) == {"c4", "c2"}
    assert "c3" in d["config"]["workload"] and d["scaling"] == "strong"
    assert d["secondary"]["c4"]["roofline"]["gather_roofline"]["frac"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 3 and d["value"] > 0
    assert d["unit"] == "GFLOP/s" and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 20
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    s = d["schedule_sweep"]
    assert s["n_schedules"] == 768 and s["fast_slow_ratio"] >= 1.0


def test_bench_line_reference():
    d = _run("--impl", "reference", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_multirank_path_on_one_gpu():
    """torchrun with 2 ranks sharing cuda:0 (--comm host: gloo + HOST
    communicator + fused put exchange): the N>1 code path of bench.py --
    schedule sweep across ranks, max-over-ranks timing, JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--comm", "host", "--steps", "10", "--warmup", "3", "--rerank", "2",
                        "--workload", "c2", "--secondary", "c4"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1 and lines[0].startswith("{"), r.stdout   # rank 0's line only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert "put" in d["config"]["parallelism"] and d["schedule_sweep"]["n_schedules"] == 768
    assert d["config"]["nnz_global"] == 14_581_760          # C2 strong-scaled over the 2 ranks
    assert d["parity_ok"] is True and d["secondary"]["c4"]["parity"]["ok"] is True
    assert d["exchange"]["bytes_in_per_rank_max"] == 128 * 128 * 8
    o = d["overlap"]
    assert o["T_noexch_ms"] > 0 and o["T_exch_alone_ms"] is not None
    assert d["scaling_efficiency"]["P"] == 2 and d["scaling_efficiency"]["T1_ms"] > 0
