#!/usr/bin/env python
"""Benchmark of the distributed SpMV hot path (arXiv 2203.02530).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c4|c2|c5] [--space derived|orderable] ...

One "step" = one dspmv_apply of the whole hot path (Pack, halo exchange,
Unpack, y_L, y_R + combine, all host syncs of the schedule) over the rank's
rows, inputs resident in HBM.  Every workload is strong-scaled: the BASELINE
matrix is row-partitioned over the N ranks, one process per GPU.

  c3 (default)  BASELINE configs[2]: 27-point stencil 256^3, fp64, 1/2/4/8 GPUs
  c4            BASELINE configs[3]: power-law 8M rows, avg 16 nnz, fp64, 1/2/4/8
  c2            BASELINE configs[1]: 7-point Laplacian 128^3, fp64, 1 GPU
  c5            BASELINE configs[4]: 7-point 192^3 over 4 ranks, the schedule sweep

The default run measures c3 (headline) and carries c4 (every N) and c2 (N=1)
as secondary records in the same JSON line, each with its own roofline and a
sampled-row parity check.  At N>1 it also reports the exchange bytes against
NVLink, the overlap efficiency 1 - (T_best - T_noexch)/T_exch_alone and the
scaling efficiency T_1/(P T_P).  Between timed steps the L2 is
flushed (flush kernel outside the per-step CUDA events) unless every rank's
step reads >= 8x the L2 capacity (C3, C4: inputs larger than L2; the flushed
time is recorded beside it); config.l2 says which.  Step time = sum of
per-step event intervals on the caller stream, max over ranks.

``--impl reference`` times the oracle (oracle/o1.c, serial CSR, 1 core) on a
bounded row sample of the same workload -- the tier's reference arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

_RED_DEV = "cuda"   # device of the small reduction tensors ("cpu" with gloo)
METRIC = "SpMV GFLOP/s, HBM GB/s vs peak at 1/2/4/8 B200; schedule fast/slow ratio"
BEST_ORDER = ["start", "PostRecv", "Pack", "y_L", "PostSend", "WaitRecv", "Unpack", "y_R",
              "WaitSend", "end"]
BEST_STREAMS = {"Pack": 0, "y_L": 1, "Unpack": 0, "y_R": 0}
PAPER1_ORDER = ["start", "Pack", "y_L", "PostSend", "PostRecv", "WaitSend", "WaitRecv",
                "Unpack", "y_R", "end"]
# the exchange with nothing beside it: both Waits before any SpMV (T_exch_alone)
SERIAL_ORDER = ["start", "Pack", "PostSend", "PostRecv", "WaitSend", "WaitRecv", "Unpack",
                "y_L", "y_R", "end"]
VERTS = ["start", "Pack", "y_L", "PostSend", "PostRecv", "WaitSend", "WaitRecv", "Unpack",
         "y_R", "end"]

# name: (generator kind, dims or n, BASELINE text) -- BASELINE.json configs[1..4]
WORKLOADS = {
    "c2": ("7pt", (128, 128, 128), "BASELINE configs[1]: 3D 7-point Laplacian 128^3 (2,097,152 rows) fp64"),
    "c3": ("27pt", (256, 256, 256), "BASELINE configs[2]: 3D 27-point stencil 256^3 (16,777,216 rows) fp64"),
    "c4": ("powerlaw", 1 << 23, "BASELINE configs[3]: power-law 8,388,608 rows, avg 16 nnz/row, long tail, fp64"),
    "c5": ("7pt", (192, 192, 192), "BASELINE configs[4]: 3D 7-point Laplacian 192^3 (7,077,888 rows) fp64"),
}
# input values (SURVEY §5 config flags): x seed, float or exact-integer values (R-Q23)
X_SEED = 2530
EXACT = False


def xvals(lo, hi):
    import gen
    return gen.x_values((lo, hi), seed=X_SEED, exact=EXACT)


# measured random-gather ceiling of the x operand: the best LSU rate measured
# for random fp64 gathers from a 64 MB x (ld.global.nc.L1::no_allocate + L2
# evict_last, 8 gathers in flight per thread, 148 SMs): 271.4 G/s
# (scripts/ubench_tma_gather4.cu, profiles/r2_ubench_tma_gather4.txt; round 1's
# scripts/ubench_gather_scope.cu gave 256.3 at 67 MB) -- the second roofline
# of irregular matrices
GATHER_CEILING_GPS = 271.4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--secondary", default="auto",
                    help="comma list of secondary workloads, 'none', or auto (c4 at every N, c2 at N=1)")
    ap.add_argument("--schedule", default="best", choices=["best", "paper1"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--space", default="auto", choices=["auto", "derived", "orderable"],
                    help="sweep space: derived syncs (768 schedules), orderable syncs (4,780, DESIGN.md "
                         "R-N5); auto = orderable for c5, derived otherwise")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the schedule sweep (use the class-1 'best' schedule)")
    ap.add_argument("--sweep-out", default=None,
                    help="write every swept schedule with its time (JSON) for the design-rule pipeline")
    ap.add_argument("--caller-stream0", type=int, default=0,
                    help="schedule stream 0 is the caller's stream (plan option; 0 keeps the two "
                         "schedule streams interchangeable, as the stream-bijection pruning assumes)")
    ap.add_argument("--rerank", type=int, default=16,
                    help="re-time the k fastest sweep schedules with the step method")
    ap.add_argument("--execution", default="auto", choices=["auto", "host", "graph"],
                    help="host: dspmv_apply (host-synchronised schedule, the paper's model); "
                         "graph: dspmv_apply_graph (GPU-resident CUDA graph of the same schedule); "
                         "auto: time both and report the faster as the headline")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "host"],
                    help="host: gloo process group + HOST-transport communicator with the fused "
                         "put exchange (lets N ranks share one GPU, for testing the N>1 path)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "copy", "put"],
                    help="halo exchange: NCCL group (copy), fused Pack+put over peer memory "
                         "(put), or auto = time both at N>1 and keep the faster")
    ap.add_argument("--value-mode", default="float", choices=["float", "exact"],
                    help="exact: small-integer matrix values and x (R-Q23), every result exact; the parity "
                         "self-check then requires bitwise equality")
    ap.add_argument("--seed", type=int, default=2530, help="seed of the x values (counter-based, gen/)")
    ap.add_argument("--plain-exchange", action="store_true",
                    help="Pack gathers into a send buffer and Unpack copies to x_halo (the DAG's literal "
                         "kernels) instead of aliased sends and the fused Unpack")
    ap.add_argument("--settle-s", type=float, default=2.0,
                    help="idle seconds before each workload's warm-up + timed region, so the board's power "
                         "controller does not carry the schedule sweep's draw into it (C3 runs at ~1 kW; "
                         "sustained, power-capped figures: DESIGN.md section 6)")
    ap.add_argument("--no-t1", action="store_true",
                    help="N>1: skip the 1-GPU run of the whole matrix on rank 0 (scaling efficiency)")
    return ap.parse_args()


# ----------------------------------------------------------------- workload
def workload_desc(name, world):
    """Identical in both arms (ours / reference) for the same N."""
    return f"{name}: {WORKLOADS[name][2]}, row-partitioned over {world} rank(s)"


def workload_rows(name, lo, hi):
    """(n_global, rowptr, col, val) of rows [lo, hi) of the BASELINE matrix."""
    import gen
    kind, dims, _ = WORKLOADS[name]
    if kind == "powerlaw":
        rp, col, val = gen.powerlaw(dims, (lo, hi), exact=EXACT)
        return dims, rp, col, val
    rp, col, val = gen.stencil(kind, dims, (lo, hi))
    return dims[0] * dims[1] * dims[2], rp, col, val


def workload_n(name):
    kind, dims, _ = WORKLOADS[name]
    return dims if kind == "powerlaw" else dims[0] * dims[1] * dims[2]


L2_INPUT_FACTOR = 8   # per-step inputs >= 8x L2: "inputs larger than L2", no flush between timed steps


def alg_bytes_local(n_r, nnz_L, v):
    """y_L bytes = (v+4)·nnz_L + 4(n_r+1) + v·n_r (x) + v·n_r (y)."""
    return (v + 4) * nnz_L + 4 * (n_r + 1) + 2 * v * n_r


def alg_bytes_rank(info, v):
    """Per-rank distributed bytes B_r."""
    n_r = info["row_end"] - info["row_begin"]
    R, h, s = info["n_remote_rows"], info["n_halo"], info["n_send"]
    nnz = info["nnz_local"] + info["nnz_remote"]
    return ((v + 4) * nnz + 4 * (n_r + 1) + 2 * v * n_r + 8 * R + v * h + 2 * v * R
            + (4 + 2 * v) * s + 2 * v * h)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload_key, world):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        e = d.get(f"{workload_key}_n{world}")
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def parity_sample(rp, col, val, lo, hi, n, npdt, seed=7, k=2048):
    """Rows of this rank to check after the timed region, with y_ref and the
    tolerance scale s_i = sum |a_ij x_j| computed here in numpy fp64 (the
    bench's own self-check, independent of the CUDA path): the first and last
    rows, rows with remote entries, and random rows."""
    import gen
    n_r = hi - lo
    if n_r == 0:
        return None
    rng = np.random.default_rng(seed + lo)
    rows = set(range(min(8, n_r))) | set(range(max(0, n_r - 8), n_r))
    rows |= set(rng.integers(0, n_r, size=min(k, n_r)).tolist())
    base = int(rp[0])
    # rows with an entry outside [lo, hi) (they take the y_R combine)
    if lo > 0 or hi < n:
        idx = np.flatnonzero((col < lo) | (col >= hi))
        if idx.size:
            pick = rng.choice(idx, size=min(256, idx.size), replace=False)
            rows |= set((np.searchsorted(rp - base, pick, side="right") - 1).tolist())
    rows = np.array(sorted(rows), np.int64)
    x = xvals(0, n).astype(npdt).astype(np.float64)
    yref = np.empty(rows.size)
    scale = np.empty(rows.size)
    for t, i in enumerate(rows):
        a, b = int(rp[i]) - base, int(rp[i + 1]) - base
        prod = val[a:b].astype(npdt).astype(np.float64) * x[col[a:b]]
        yref[t] = prod.sum()
        scale[t] = np.abs(prod).sum()
    return rows, yref, scale


def check_parity(sample, y, rel):
    if sample is None:
        return True, 0.0
    rows, yref, scale = sample
    if hasattr(y, "cpu"):
        import torch
        yy = y[torch.from_numpy(rows).to(y.device)].double().cpu().numpy()
    else:
        yy = np.asarray(y)[rows]
    err = np.abs(yy - yref)
    # both sides round differently (any order within a row, R-Q10/Q11): within
    # rel * s_i, plus an fp64 rounding term of the numpy reference itself
    ok = bool(np.all(err <= rel * scale) and np.all(np.isfinite(yy))) if rel > 0 else \
        bool(np.array_equal(yy, yref))
    worst = float(np.max(err / np.maximum(scale, 1e-300))) if rows.size else 0.0
    return ok, worst


_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
hs = [pynvml.nvmlDeviceGetHandleByIndex(int(i)) for i in sys.argv[2].split(",")]
get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
with open(sys.argv[1], "w", buffering=1) as f:
    for h in hs:
        f.write("max %d\n" % pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
    while True:
        for h in hs:
            f.write("%.6f %d %d\n" % (time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), get_r(h)))
        time.sleep(0.0005)
"""


class Clocks:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed
    region by a separate NVML polling process (no GIL contention), started
    before the warm-up; only samples inside [mark_start, mark_end] count."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpus):
        self.path = f"/tmp/bench_clocks_{os.getpid()}.txt"
        self.spans = []
        self.t0 = None
        try:
            self.p = subprocess.Popen([sys.executable, "-c", _SAMPLER, self.path,
                                       ",".join(map(str, gpus))], stderr=subprocess.DEVNULL)
            for _ in range(200):            # wait until sampling has started
                if os.path.exists(self.path) and os.path.getsize(self.path) > 40:
                    break
                time.sleep(0.01)
        except Exception:
            self.p = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.spans.append((self.t0, time.time()))

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": [],
                    "source": "unavailable"}
        time.sleep(0.005)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, smax, reasons = [], [], set()
        for line in open(self.path):
            f = line.split()
            if f[0] == "max":
                smax.append(float(f[1]))
                continue
            if len(f) != 3:
                continue
            t, c, r = float(f[0]), float(f[1]), int(f[2])
            if not any(a <= t <= b for a, b in self.spans):
                continue
            sm.append(c)
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons), "source": "nvml (separate process)"}


# ---------------------------------------------------------------- ours
def timing_mask(world):
    """Events of the timed region: START..END on the caller stream, the y_L op
    on its stream (roofline), and at N > 1 the exchange on the comm stream.
    The schedule re-ranking uses the same mask, so the event records it adds
    to each step are the same in the ranking and in the timed region."""
    from paper_2203_02530_b200 import dspmv as D
    m = (1 << D.DSPMV_OP_SPMV_LOCAL) | (1 << D.DSPMV_OP_START)
    if world > 1:
        m |= (1 << D.DSPMV_OP_POST_SEND) | (1 << D.DSPMV_OP_POST_RECV)
    return m


class Ctx:
    """One rank's process-level state: dist group, communicator, device."""

    def __init__(self, a):
        import torch
        import torch.distributed as dist
        from paper_2203_02530_b200 import dspmv as D
        self.a, self.D, self.torch, self.dist = a, D, torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != a.gpus:
            raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={self.world}")
        self.device = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(self.device)
        global _RED_DEV
        if self.world > 1:
            if a.comm == "host":
                dist.init_process_group("gloo")
                _RED_DEV = "cpu"
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.device))
        self.dt = D.DSPMV_F32 if a.dtype == "f32" else D.DSPMV_F64
        self.v = 4 if self.dt == D.DSPMV_F32 else 8
        self.npdt = np.float32 if self.dt == D.DSPMV_F32 else np.float64
        self.tdt = torch.float32 if self.dt == D.DSPMV_F32 else torch.float64
        self.rel = 1e-5 if self.dt == D.DSPMV_F32 else 1e-12   # north_star tolerances
        if a.comm == "host":
            world = self.world

            def allgather(b: bytes) -> bytes:
                out = [None] * world
                dist.all_gather_object(out, b) if world > 1 else out.__setitem__(0, b)
                return b"".join(out)
            self.comm = D.dspmv_comm_create_host(self.world, self.rank, self.device, allgather)
        else:
            uid = D.dspmv_comm_unique_id() if self.rank == 0 else None
            if self.world > 1:
                obj = [uid]
                dist.broadcast_object_list(obj, src=0)
                uid = obj[0]
            self.comm = D.dspmv_comm_create(uid, self.world, self.rank, self.device)
        self.stream = torch.cuda.Stream()   # a non-default stream (the graph mode captures on it)
        self.launches = 0

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def allmax(self, t):
        if self.world > 1:
            tt = self.torch.tensor([t], dtype=self.torch.float64, device=_RED_DEV)
            self.dist.all_reduce(tt, op=self.dist.ReduceOp.MAX)
            return float(tt.item())
        return t

    def allmin(self, t):
        return -self.allmax(-t)

    def allsum(self, t):
        if self.world > 1:
            tt = self.torch.tensor([t], dtype=self.torch.float64, device=_RED_DEV)
            self.dist.all_reduce(tt, op=self.dist.ReduceOp.SUM)
            return float(tt.item())
        return t

    def alland(self, ok):
        return self.allmin(1.0 if ok else 0.0) > 0.5

    def close(self):
        self.D.dspmv_comm_destroy(self.comm)
        if self.world > 1:
            self.dist.destroy_process_group()


def derive(D, order, streams):
    return D.dspmv_schedule_derive([VERTS.index(x) for x in order],
                                   [streams.get(x, 0) for x in order], 2)


def time_steps(ctx, sched, apply_fn, x, y, steps, iyl=None, iposts=(), clocks=None, flush=True):
    """K steps, the L2 flushed before each (outside the per-step events).
    Returns per-rank lists: step ms (START..END events), y_L ms, exchange us."""
    D = ctx.D
    step, yl, xus, tl = [], [], [], []
    ctx.barrier()
    if clocks:
        clocks.mark_start()
    l0 = D.dspmv_launch_count()
    for _ in range(steps):
        if flush:
            D.dspmv_l2_flush(ctx.device, ctx.stream)
        apply_fn(sched, x, y, ctx.stream)
        t = D.dspmv_schedule_op_times(sched)
        step.append(float(t[0]))
        if iyl is not None:
            yl.append(float(t[iyl]))
            b_, e_ = D.dspmv_schedule_op_timeline(sched)
            tl.append((float(b_[iyl]), float(e_[iyl])))
        if iposts:
            xus.append(max(float(t[i]) for i in iposts) * 1e3)
    ctx.barrier()
    if clocks:
        clocks.mark_end()
    launches = D.dspmv_launch_count() - l0
    return step, yl, xus, tl, launches


def pick_mode(ctx, sched, x, y, pref, exchange):
    """Execution mode: host-synchronised apply vs GPU-resident graph, chosen
    by 30 flushed steps each (max over ranks); falls back to host on failure."""
    D = ctx.D
    graph_ok = pref != "host"
    note = None
    if graph_ok:
        try:   # capture only: every rank agrees before any rank launches (PUT epochs)
            D.dspmv_apply_graph_prepare(sched, x, y, ctx.stream)
        except Exception as e:  # noqa: BLE001 -- falls back to the host mode, reported
            graph_ok, note = False, f"graph capture failed, host mode used: {e}"
            print(f"[bench rank {ctx.rank}] {note}", file=sys.stderr, flush=True)
    graph_ok = ctx.alland(graph_ok)
    if not graph_ok:
        return D.dspmv_apply, "host", note
    for _ in range(3):
        D.dspmv_apply_graph(sched, x, y, ctx.stream)
    ctx.torch.cuda.synchronize()
    if pref == "graph":
        return D.dspmv_apply_graph, "graph", note
    tms = {}
    for name, fn in (("host", D.dspmv_apply), ("graph", D.dspmv_apply_graph)):
        step = time_steps(ctx, sched, fn, x, y, 30)[0]
        tms[name] = ctx.allmax(sum(step) / 30)
    best = "graph" if tms["graph"] < tms["host"] else "host"
    note = {"ms_per_step_30": {k: round(v, 5) for k, v in tms.items()}}
    return (D.dspmv_apply_graph if best == "graph" else D.dspmv_apply), best, note


def exec_name(mode):
    return {"host": "host-synchronised (dspmv_apply)",
            "graph": "GPU-resident CUDA graph (dspmv_apply_graph)"}[mode]


def measure(ctx, wname, headline, clocks=None, sched_from=None):
    """Plan + schedule + K timed steps of one workload at this N.  The
    headline workload also gets the schedule sweep, the e2e leg, the warm-L2
    column and (N>1) the overlap efficiency."""
    import gen
    a, D, torch = ctx.a, ctx.D, ctx.torch
    world, rank = ctx.world, ctx.rank
    n = workload_n(wname)
    rb = D.dspmv_partition(n, world)
    lo, hi = int(rb[rank]), int(rb[rank + 1])
    _, rp, col, val = workload_rows(wname, lo, hi)
    nnz_rank = int(rp[-1] - rp[0])
    sample = parity_sample(rp, col, val, lo, hi, n, ctx.npdt)
    valn = val.astype(ctx.npdt)
    del val

    def mk(ex):
        # stencil send lists are planes: sent straight from x (no Pack kernel)
        # where possible, and y_R reads the halo where it was received
        # (profiles/r2_c5_exec_modes.json); --plain-exchange keeps Pack/Unpack
        extra = {} if a.plain_exchange else dict(pack_mode=D.DSPMV_PACK_ALIAS_IF_CONTIGUOUS,
                                                  unpack_mode=D.DSPMV_UNPACK_FUSED)
        return D.dspmv_plan_create(ctx.comm, n, rp, col, valn, dtype=ctx.dt,
                                   caller_stream0=bool(a.caller_stream0), exchange=ex, **extra)
    exchange_note = None
    if a.comm == "host":
        plan, exchange, ex_mode = mk(D.DSPMV_EXCHANGE_PUT), "put (fused Pack+put over peer memory)", "put"
    elif world == 1 or a.exchange == "copy":
        plan, exchange, ex_mode = mk(D.DSPMV_EXCHANGE_COPY), "copy (NCCL group)", "copy"
    elif a.exchange == "put":
        plan, exchange, ex_mode = mk(D.DSPMV_EXCHANGE_PUT), "put (fused Pack+put over peer memory)", "put"
    else:
        plan, exchange, ex_mode, exchange_note = choose_exchange(ctx, mk, lo, hi)
    info = D.dspmv_plan_info_get(plan)
    # N>1 overlap baseline: the same plan with a zero-byte exchange (T_noexch)
    plan_none = mk(D.DSPMV_EXCHANGE_NONE) if (headline and world > 1) else None
    del col, valn
    x = torch.from_numpy(xvals(lo, hi).astype(ctx.npdt)).cuda()
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    # L2 between timed steps (timing rules): flushed, unless every rank's step
    # reads at least L2_INPUT_FACTOR x the L2 capacity -- then the inputs are
    # far larger than L2 and a step cannot find its data there anyway (C3:
    # 45x, C4: 14x; C2 at 1.7x keeps the flush); the flushed time is recorded
    # beside it (it differs only by the flush kernel's power draw on leases
    # that hit sw_power_cap)
    l2_bytes = int(torch.cuda.get_device_properties(ctx.device).L2_cache_size)
    min_rank_bytes = ctx.allmin(float(alg_bytes_rank(info, ctx.v)))
    flush_steps = min_rank_bytes < L2_INPUT_FACTOR * l2_bytes
    l2_note = ("flushed between timed steps (flush kernel reads 2x L2, outside per-step CUDA events)"
               if flush_steps else
               f"not flushed: every rank's step reads >= {min_rank_bytes / 1e9:.2f} GB = "
               f"{min_rank_bytes / l2_bytes:.0f}x the {l2_bytes / 1e6:.0f} MB L2 (inputs larger than L2)")

    # ---- schedule: sweep over the design space (paper protocol) + re-ranking
    sweep = None
    mode_pref = a.execution
    if headline and not a.no_sweep:
        space = a.space if a.space != "auto" else ("orderable" if wname == "c5" else "derived")
        sweep = schedule_sweep(ctx, plan, x, y, space=space, out_path=a.sweep_out)
        ranked = sweep.pop("_ranked_ops")
        ranked_top = ranked[:16]
        ops, best_mode, cs0, rerank_log = rerank(ctx, plan, x, y, ranked, a.rerank, mode_pref, ex_mode)
        sweep["rerank_us"] = rerank_log
        from paper_2203_02530_b200 import schedules as PS
        sched_desc = (f"best of the {min(a.rerank, len(ranked))} sweep-fastest (+1) re-timed per step "
                      f"({best_mode} execution, stream 0 = {'caller' if cs0 else 'library'} stream): "
                      + PS.describe(ops))
        if mode_pref == "auto":
            mode_pref = best_mode
    elif sched_from is not None:
        # secondary workloads re-time the headline sweep's fastest schedules
        # on their own matrix (no second sweep) and keep the best
        from paper_2203_02530_b200 import schedules as PS
        head_ops, head_mode, head_ranked = sched_from
        cands = list(head_ranked[:8]) if head_ranked else []
        if not any(np.array_equal(head_ops, c) for c in cands):
            cands.append(head_ops)
        ops, best_mode, cs0, _ = rerank(ctx, plan, x, y, cands, len(cands), mode_pref, ex_mode)
        sched_desc = (f"best of the headline sweep's {len(cands)} fastest, re-timed on this matrix "
                      f"({best_mode} execution, stream 0 = {'caller' if cs0 else 'library'} stream): "
                      + PS.describe(ops))
        if mode_pref == "auto":
            mode_pref = best_mode
    else:
        order = BEST_ORDER if a.schedule == "best" else PAPER1_ORDER
        streams = BEST_STREAMS if a.schedule == "best" else dict.fromkeys(BEST_STREAMS, 0)
        ops = derive(D, order, streams)
        cs0 = 0
        sched_desc = a.schedule + ": " + " ".join(order) + f" streams={streams}"
    sched = D.dspmv_schedule_create(plan, ops, 2)
    D.dspmv_schedule_set_timing(sched, timing_mask(world))
    D.dspmv_schedule_set_caller_stream0(sched, cs0)
    iyl = [i for i, o in enumerate(ops) if o[0] == D.DSPMV_OP_SPMV_LOCAL][0]
    iposts = [i for i, o in enumerate(ops) if o[0] in (D.DSPMV_OP_POST_SEND, D.DSPMV_OP_POST_RECV)] \
        if world > 1 else []
    apply_fn, mode, exec_note = pick_mode(ctx, sched, x, y, mode_pref, ex_mode)

    # ---- warmup + timed region
    if a.settle_s > 0:
        torch.cuda.synchronize()
        time.sleep(a.settle_s)
        ctx.barrier()
    for _ in range(a.warmup):
        if flush_steps:
            D.dspmv_l2_flush(ctx.device, ctx.stream)
        apply_fn(sched, x, y, ctx.stream)
    steps = a.steps if headline else max(3, min(a.steps, 100))
    t_wall0 = time.perf_counter()
    step, yl, xus, tl, launches = time_steps(ctx, sched, apply_fn, x, y, steps, iyl, iposts, clocks,
                                             flush=flush_steps)
    t_wall = time.perf_counter() - t_wall0
    ms_per_step = ctx.allmax(sum(step)) / steps
    stats = [round(ctx.allmax(float(np.percentile(step, q))) * 1e3, 2) for q in (50, 0, 90)]
    yl_ms = sum(yl) / steps
    yl_ms_max = ctx.allmax(yl_ms)
    nnz_total = ctx.allsum(float(nnz_rank))
    gflops = 2.0 * nnz_total / (ms_per_step * 1e-3) / 1e9
    launches_total = int(ctx.allsum(float(launches)))

    # ---- parity self-check (outside the timed region): one more apply
    y.fill_(float("nan"))
    apply_fn(sched, x, y, ctx.stream)
    torch.cuda.synchronize()
    ok, worst = check_parity(sample, y, 0.0 if EXACT else ctx.rel)
    parity = {"ok": ctx.alland(ok), "rows_checked": int(ctx.allsum(float(0 if sample is None else len(sample[0])))),
              "max_err_over_scale": ctx.allmax(worst), "tolerance": 0.0 if EXACT else ctx.rel,
              "reference": "numpy fp64 row products of sampled rows (first/last, remote, random) vs the "
                           "north_star bound |y - y_ref| <= tol * sum|a_ij x_j|"}

    # ---- roofline of the dominant kernel (y_L)
    n_r = hi - lo
    yl_bytes = alg_bytes_local(n_r, info["nnz_local"], ctx.v)
    achieved = yl_bytes / (yl_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    sk = info.get("s_kernel_local")
    kname = {D.DSPMV_SKERNEL_STREAM: "spmv_stream_kernel",
             D.DSPMV_SKERNEL_STREAM_TMA: "spmv_stream_tma_kernel",
             D.DSPMV_SKERNEL_SELL: "spmv_sell_kernel"}.get(sk, "spmv_block_kernel")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": ncu_traffic(wname, world),
            "kernel": kname + " (y_L, SPMV_LOCAL op)", "alg_bytes_per_launch": int(yl_bytes),
            "avg_launch_ms": round(yl_ms, 6), "max_rank_launch_ms": round(yl_ms_max, 6),
            "peak_source": peak_src}
    if sk in (D.DSPMV_SKERNEL_STREAM, D.DSPMV_SKERNEL_STREAM_TMA, D.DSPMV_SKERNEL_SELL):
        gps = info["nnz_local"] / (yl_ms * 1e-3) / 1e9
        roof["gather_roofline"] = {
            "gathers_per_launch": int(info["nnz_local"]), "achieved_G_per_s": round(gps, 1),
            "ceiling_G_per_s": GATHER_CEILING_GPS, "frac": round(gps / GATHER_CEILING_GPS, 4),
            "ceiling_source": "best measured random fp64 LSU gather rate from a 64 MB x, 148 SMs "
                              "(profiles/r2_ubench_tma_gather4.txt)"}
    step_bytes = ctx.allsum(float(alg_bytes_rank(info, ctx.v)))
    rec = {
        "workload": workload_desc(wname, world), "value": round(gflops, 3), "unit": "GFLOP/s",
        "ms_per_step": round(ms_per_step, 6), "steps": steps,
        "n_global": n, "nnz_global": int(nnz_total),
        "parallelism": (f"row-partition x{world}, halo exchange: {exchange}"
                        + ("" if a.plain_exchange else
                           f", pack: {'aliased sends' if info.get('pack_alias') else 'gather'}, unpack: fused into y_R")),
        "exchange_selection": exchange_note,
        "execution": exec_name(mode), "execution_selection": exec_note, "schedule": sched_desc,
        "step_us_median_min_p90": stats,
        "step_hbm_gbs_algorithmic": round(step_bytes / (ms_per_step * 1e-3) / 1e9, 1),
        "yL_window_in_step_us_median": [round(float(np.median([t[0] for t in tl])) * 1e3, 2),
                                        round(float(np.median([t[1] for t in tl])) * 1e3, 2)],
        "wall_s_timed_region": round(t_wall, 3),
        "roofline": roof, "parity": parity,
        "gpu_launches": launches_total,
    }
    if sweep is not None:
        rec["schedule_sweep"] = sweep

    # ---- halo exchange vs NVLink (N > 1)
    if world > 1:
        xmed = float(np.median(xus)) if xus else 0.0
        bmax = ctx.allmax(float(info["n_halo"] * ctx.v))
        xmax = ctx.allmax(xmed)
        rec["exchange"] = {
            "bytes_in_per_rank_max": int(bmax), "bytes_out_rank0": int(info["n_send"] * ctx.v),
            "bytes_total_per_step": int(ctx.allsum(float(info["n_halo"] * ctx.v))),
            "peers_max": int(ctx.allmax(float(max(info["n_recv_peers"], info["n_send_peers"])))),
            "exchange_us_median_max_rank": round(xmax, 2),
            "GB_s": round(bmax / (xmax * 1e-6) / 1e9, 1) if xmax > 0 else None,
            "nvlink_ref_GB_s": 770.0,
            "note": "comm-stream time of the exchange issued at the later Post (NCCL group, or the "
                    "wait on peers' put flags) inside the timed steps; 770 GB/s = measured peer copy "
                    "per direction (B200_PROFILING.md), 900 GB/s spec"}
    # ---- overlap efficiency (N > 1): 1 - (T_best - T_noexch) / T_exch_alone
    if plan_none is not None:
        rec["overlap"] = overlap_efficiency(ctx, plan, plan_none, ops, mode, x, y, ms_per_step, cs0)
    if plan_none is not None:
        D.dspmv_plan_destroy(plan_none)

    rec["l2"] = l2_note
    rec["_flushed"] = flush_steps
    if headline:
        # secondary column: the same steps with the other L2 treatment
        other = time_steps(ctx, sched, apply_fn, x, y, min(steps, 50), flush=not flush_steps)[0]
        key = "step_us_median_warm_l2" if flush_steps else "step_us_median_flushed_l2"
        rec[key] = round(ctx.allmax(float(np.median(other))) * 1e3, 2)
        rec["e2e"] = e2e_leg(ctx, sched, lo, hi, nnz_total, steps)
        rec["_sched_ops"] = ops
        rec["_mode"] = mode
        rec["_cs0"] = cs0
        rec["_ranked"] = ranked_top if sweep is not None else None
    D.dspmv_schedule_destroy(sched)
    D.dspmv_plan_destroy(plan)
    del x, y
    torch.cuda.empty_cache()
    return rec


def e2e_leg(ctx, sched, lo, hi, nnz_total, steps):
    """The same apply through the C ABI with HOST buffers (pinned): the H2D of
    x, the schedule, and the D2H of y inside every timed step."""
    import gen
    D, torch = ctx.D, ctx.torch
    xh = torch.from_numpy(xvals(lo, hi).astype(ctx.npdt)).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    k = max(3, min(steps, 100))
    for _ in range(3):
        D.dspmv_apply_host(sched, xh, yh, ctx.stream)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
    ctx.barrier()
    for i in range(k):
        D.dspmv_l2_flush(ctx.device, ctx.stream)
        evs[i][0].record(ctx.stream)
        D.dspmv_apply_host(sched, xh, yh, ctx.stream)
        evs[i][1].record(ctx.stream)
    ctx.barrier()
    ms = ctx.allmax(sum(e0.elapsed_time(e1) for e0, e1 in evs)) / k
    n_total = ctx.allsum(float(hi - lo))
    bytes_io = n_total * ctx.v
    out = {"value": round(2.0 * nnz_total / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
           "h2d_bytes_per_step": int(bytes_io), "d2h_bytes_per_step": int(bytes_io),
           "ms_per_step": round(ms, 6), "api": "dspmv_apply_host (pinned host x/y)"}
    pc = pcie_peak()
    if pc:
        # the copies alone at the measured PCIe rates, per rank, the two
        # directions overlapped (x in while y goes out): the e2e floor
        b = bytes_io / ctx.world
        floor_ms = max(b / (pc["h2d_GB_s"] * 1e9), b / (pc["d2h_GB_s"] * 1e9),
                       2 * b / (pc["bidir_GB_s"] * 1e9)) * 1e3
        out["pcie"] = {"h2d_GB_s_measured": pc["h2d_GB_s"], "d2h_GB_s_measured": pc["d2h_GB_s"],
                       "bidir_GB_s_measured": pc["bidir_GB_s"],
                       "copy_floor_ms": round(floor_ms, 6),
                       "pcie_frac": round(floor_ms / ms, 4),
                       "note": "floor = max(x/H2D, y/D2H, (x+y)/bidirectional) at the measured pinned-copy "
                               "rates; pcie_frac = floor / e2e step time",
                       "source": pc["source"]}
    return out


def build_ids():
    """Content hashes of the library that ran and of its sources (the box has
    no .git): ties a JSON line to a build."""
    import hashlib

    def h(paths):
        d = hashlib.sha256()
        for q in paths:
            try:
                d.update(open(q, "rb").read())
            except OSError:
                pass
        return d.hexdigest()[:16]
    from paper_2203_02530_b200 import dspmv as D
    src = sorted(os.path.join(dp, f) for dp, _, fs in os.walk(os.path.join(ROOT, "paper_2203_02530_b200", "csrc"))
                 for f in fs) + [os.path.join(ROOT, "include", "dspmv.h")]
    return {"lib_sha16": h([D.LIB_PATH]), "src_sha16": h(src), "bench_sha16": h([os.path.abspath(__file__)])}


def pcie_peak():
    p = os.path.join(ROOT, "profiles", "pcie_peak.json")
    try:
        d = json.load(open(p))
        return {"h2d_GB_s": float(d["h2d_GB_s"]), "d2h_GB_s": float(d["d2h_GB_s"]),
                "bidir_GB_s": float(d["bidir_GB_s_total"]),
                "source": "profiles/pcie_peak.json (scripts/pcie_peak.py, pinned, 64 MiB, best of 20)"}
    except Exception:
        return None


def overlap_efficiency(ctx, plan, plan_none, ops, mode, x, y, t_best, cs0=0):
    """T_noexch = the headline schedule on a plan whose exchange
    moves no bytes (DSPMV_EXCHANGE_NONE, same syncs); T_exch_alone = the
    serial schedule (both Waits before any SpMV) minus the same serial
    schedule without bytes."""
    D = ctx.D
    fn = D.dspmv_apply_graph if mode == "graph" else D.dspmv_apply

    def t_of(p, o):
        s = D.dspmv_schedule_create(p, o, 2)
        D.dspmv_schedule_set_timing(s, timing_mask(ctx.world))
        D.dspmv_schedule_set_caller_stream0(s, cs0)
        f = fn
        if f is D.dspmv_apply_graph:   # agree on the graph before any rank launches one
            ok = True
            try:
                D.dspmv_apply_graph_prepare(s, x, y, ctx.stream)
            except Exception:  # noqa: BLE001 -- this measurement then runs host-synchronised
                ok = False
            if not ctx.alland(ok):
                f = D.dspmv_apply
        try:
            for _ in range(5):
                f(s, x, y, ctx.stream)
            st = time_steps(ctx, s, f, x, y, 50)[0]
            return ctx.allmax(sum(st) / len(st))
        finally:
            D.dspmv_schedule_destroy(s)
    serial = derive(D, SERIAL_ORDER, {})
    t_noexch = t_of(plan_none, ops)
    t_serial = t_of(plan, serial)
    t_serial_none = t_of(plan_none, serial)
    t_exch = t_serial - t_serial_none
    eff = 1.0 - (t_best - t_noexch) / t_exch if t_exch > 0 else None
    return {"T_best_ms": round(t_best, 6), "T_noexch_ms": round(t_noexch, 6),
            "T_exch_alone_ms": round(t_exch, 6), "T_serial_ms": round(t_serial, 6),
            "efficiency": None if eff is None else round(eff, 4),
            "note": "1 - (T_best - T_noexch)/T_exch_alone; T_noexch: same schedule, exchange moves 0 B "
                    "(DSPMV_EXCHANGE_NONE); T_exch_alone: serial schedule (Waits before y_L) minus its "
                    "0-byte twin; 50 flushed steps each, max over ranks"}


def rerank(ctx, plan, x, y, ranked, k, mode_pref, ex_mode):
    """The sweep ranks by back-to-back wall time (paper protocol); the headline
    is per-step device time with a flushed L2: re-time the k fastest (plus the
    fastest whose first GPU vertex is y_L) in both execution modes, keep the best."""
    D = ctx.D
    from paper_2203_02530_b200 import schedules as PS
    modes = [("host", D.dspmv_apply)]
    if mode_pref != "host":
        modes.append(("graph", D.dspmv_apply_graph))
    if mode_pref == "graph":
        modes = modes[1:]
    cands = list(ranked[:max(1, k)])
    first_yl = next((o for o in ranked if [int(v) for v in o[:, 0] if v in PS.GPU][0]
                     == D.DSPMV_OP_SPMV_LOCAL), None)
    if first_yl is not None and not any(np.array_equal(first_yl, c) for c in cands):
        cands.append(first_yl)
    best, log = None, []
    for ci, cand in enumerate(cands):
        sc = D.dspmv_schedule_create(plan, cand, 2)
        D.dspmv_schedule_set_timing(sc, timing_mask(ctx.world))
        # stream 0 bound to a library stream (the sweep's symmetric setting) or
        # to the caller's stream (no fork for its first op): a timing choice
        # made after the sweep, so the sweep's stream bijection still holds
        for (mname, fn), cs0 in [(m, b) for m in modes for b in (0, 1)]:
            D.dspmv_schedule_set_caller_stream0(sc, cs0)
            # every rank must run the same applies (PUT epochs): capture first,
            # agree, then run
            ok = True
            if mname == "graph":
                try:
                    D.dspmv_apply_graph_prepare(sc, x, y, ctx.stream)
                except Exception as e:  # noqa: BLE001 -- mode unavailable for this schedule
                    ok = False
                    print(f"[bench rank {ctx.rank}] rerank candidate {ci} graph: {e}", file=sys.stderr, flush=True)
            if not ctx.alland(ok):
                continue
            for _ in range(3):
                fn(sc, x, y, ctx.stream)
            ctx.torch.cuda.synchronize()
            st = time_steps(ctx, sc, fn, x, y, 30)[0]
            tot = ctx.allmax(sum(st) / 30)
            log.append([ci, mname, cs0, round(tot * 1e3, 2)])
            if best is None or tot < best[0]:
                best = (tot, cand, mname, cs0)
        D.dspmv_schedule_destroy(sc)
    return best[1], best[2], best[3], log


def choose_exchange(ctx, mk, lo, hi):
    """N > 1: build both exchange variants, time each with the class-1
    schedule (same inputs, max over ranks) and keep the faster.  A PUT setup
    or run failure falls back to the NCCL copy exchange (reported)."""
    import gen
    D, torch, dist = ctx.D, ctx.torch, ctx.dist
    ops = derive(D, BEST_ORDER, BEST_STREAMS)
    x = torch.from_numpy(xvals(lo, hi).astype(ctx.npdt)).cuda()
    y = torch.empty_like(x)
    times, plans, errs = {}, {}, {}
    for name, ex in (("copy", D.DSPMV_EXCHANGE_COPY), ("put", D.DSPMV_EXCHANGE_PUT)):
        ok = 1.0
        try:
            p = mk(ex)
            plans[name] = p
            s = D.dspmv_schedule_create(p, ops, 2)
            for _ in range(10):
                D.dspmv_apply(s, x, y)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(50):
                D.dspmv_apply(s, x, y)
            torch.cuda.synchronize()
            t = (time.perf_counter() - t0) / 50
            D.dspmv_schedule_destroy(s)
        except Exception as e:  # noqa: BLE001 -- the alternative is reported, not fatal
            ok, t = 0.0, float("inf")
            errs[name] = str(e)[:200]
        tt = torch.tensor([t if ok else 1e9, ok], dtype=torch.float64, device=_RED_DEV)
        dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.MIN)
        times[name] = float(tt[0].item()) if tt[1].item() > 0 else None
    if times.get("copy") is None and times.get("put") is None:
        raise RuntimeError(f"neither halo exchange variant could be set up: {errs}")
    best = "put" if times.get("put") is not None and (times.get("copy") is None or times["put"] < times["copy"]) \
        else "copy"
    for name, p in plans.items():
        if name != best:
            D.dspmv_plan_destroy(p)
    label = {"copy": "copy (NCCL group)", "put": "put (fused Pack+put over peer memory)"}[best]
    note = {"us_per_apply_class1_schedule": {k: (round(v * 1e6, 2) if v is not None else "failed")
                                             for k, v in times.items()}, "chosen": best}
    if errs:
        note["errors"] = errs
    return plans[best], label, best, note


def schedule_sweep(ctx, plan, x, y, t_measure=0.01, space="derived", out_path=None):
    """Every schedule of the DAG (768 with derived syncs under DESIGN.md R-Q13,
    4,780 with orderable syncs, R-N5), measured with the paper's protocol
    (P:461-464): repeat samples until t_measure = 0.01 s, time = max over
    ranks of t_measure / n_samples.  Rank 0 calibrates n_samples and
    broadcasts it so every rank runs the same number of exchanges (R-Q19)."""
    D, torch = ctx.D, ctx.torch
    dist = ctx.dist if ctx.world > 1 else None
    from paper_2203_02530_b200 import schedules as PS
    all_ops = PS.enumerate_orderable(2) if space == "orderable" else PS.enumerate_derived(2)
    times = []
    t_start = time.perf_counter()
    for ops in all_ops:
        s = D.dspmv_schedule_create(plan, ops, 2)
        for _ in range(2):
            D.dspmv_apply(s, x, y, ctx.stream)
        ctx.barrier()
        t0 = time.perf_counter()
        D.dspmv_apply(s, x, y, ctx.stream)
        n = max(1, math.ceil(t_measure / max(time.perf_counter() - t0, 1e-7)))
        if dist is not None:
            nt = torch.tensor([n], dtype=torch.int64, device=_RED_DEV)
            dist.broadcast(nt, src=0)
            n = int(nt.item())
        ctx.barrier()
        t0 = time.perf_counter()
        for _ in range(n):
            D.dspmv_apply(s, x, y, ctx.stream)
        t = ctx.allmax((time.perf_counter() - t0) / n)
        times.append(t)
        D.dspmv_schedule_destroy(s)
    times = np.array(times)
    ib, iw = int(times.argmin()), int(times.argmax())
    q = np.percentile(times, [10, 50, 90])
    if out_path and ctx.rank == 0:
        with open(out_path, "w") as f:
            json.dump({"space": space, "n_ranks": ctx.world, "comm": ctx.a.comm,
                       "protocol": "P:461-464, t_measure 0.01 s, max over ranks (SPMD processes)",
                       "schedules": [[[int(v) for v in row] for row in o] for o in all_ops],
                       "times_s": [float(t) for t in times]}, f)
    return {
        "n_schedules": len(all_ops), "space": space,
        "protocol": "P:461-464, t_measure 0.01 s, max over ranks",
        "fastest_ms": round(times[ib] * 1e3, 5), "slowest_ms": round(times[iw] * 1e3, 5),
        "p10_p50_p90_ms": [round(v * 1e3, 5) for v in q],
        "fast_slow_ratio": round(times[iw] / times[ib], 4),
        "fastest": PS.describe(all_ops[ib]), "slowest": PS.describe(all_ops[iw]),
        "sweep_wall_s": round(time.perf_counter() - t_start, 2),
        "paper_context": "1.47x over 2036 implementations, 4x A100 Perlmutter, 150K banded (P:52-60)",
        "_ranked_ops": [all_ops[i] for i in np.argsort(times, kind="stable")],
    }


def t1_run(ctx, wname, ops, mode, cs0=0):
    """N>1 scaling efficiency: rank 0 alone runs the whole matrix on its GPU
    through a 1-rank communicator (same schedule and execution mode, 30
    flushed steps); the other ranks wait."""
    import gen
    D, torch = ctx.D, ctx.torch
    out = None
    if ctx.rank == 0:
        comm1 = D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, ctx.device)
        try:
            n, rp, col, val = workload_rows(wname, 0, workload_n(wname))
            plan = D.dspmv_plan_create(comm1, n, rp, col, val.astype(ctx.npdt), dtype=ctx.dt,
                                       caller_stream0=bool(ctx.a.caller_stream0))
            del rp, col, val
            x = torch.from_numpy(xvals(0, n).astype(ctx.npdt)).cuda()
            y = torch.empty_like(x)
            s = D.dspmv_schedule_create(plan, ops, 2)
            D.dspmv_schedule_set_timing(s, timing_mask(1))
            D.dspmv_schedule_set_caller_stream0(s, cs0)
            fn = D.dspmv_apply_graph if mode == "graph" else D.dspmv_apply
            for _ in range(5):
                D.dspmv_l2_flush(ctx.device, ctx.stream)
                fn(s, x, y, ctx.stream)
            tot = 0.0
            for _ in range(30):
                D.dspmv_l2_flush(ctx.device, ctx.stream)
                fn(s, x, y, ctx.stream)
                tot += float(D.dspmv_schedule_op_times(s)[0])
            out = tot / 30
            D.dspmv_schedule_destroy(s)
            D.dspmv_plan_destroy(plan)
            del x, y
            torch.cuda.empty_cache()
        finally:
            D.dspmv_comm_destroy(comm1)
    if ctx.world > 1:
        ctx.dist.barrier()
    return out


def secondaries(a, world):
    if a.secondary == "none":
        return []
    if a.secondary != "auto":
        return [w for w in a.secondary.split(",") if w and w != a.workload]
    out = [] if a.workload == "c4" else ["c4"]
    if world == 1 and a.workload != "c2":
        out.append("c2")
    return out


def run_ours(a):
    ctx = Ctx(a)
    world, rank = ctx.world, ctx.rank
    clocks = Clocks(list(range(min(world, ctx.torch.cuda.device_count())))) if rank == 0 else None
    head = measure(ctx, a.workload, True, clocks)
    ops, mode, ranked, cs0 = head.pop("_sched_ops"), head.pop("_mode"), head.pop("_ranked"), head.pop("_cs0")
    secs = {}
    for w in secondaries(a, world):
        secs[w] = measure(ctx, w, False, clocks, sched_from=(ops, mode, ranked))
        secs[w].pop("_flushed", None)
    scaling = None
    if world > 1 and not a.no_t1:
        t1 = t1_run(ctx, a.workload, ops, mode, cs0)
        if rank == 0 and t1:
            scaling = {"T1_ms": round(t1, 6), "TP_ms": head["ms_per_step"], "P": world,
                       "efficiency": round(t1 / (world * head["ms_per_step"]), 4),
                       "note": "T_1 / (P T_P) (SURVEY 8(d)); T_1 = the whole matrix on rank 0's GPU "
                               "through a 1-rank communicator, same schedule and execution mode, "
                               "30 flushed steps"}
    clk = clocks.stop() if clocks else None
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a.workload, budget_s=10.0)
    if rank == 0:
        steps = head.pop("steps")
        launches = head.pop("gpu_launches")
        out = {
            "metric": METRIC, "value": head.pop("value"), "unit": head.pop("unit"), "n_gpus": world,
            "steps": steps, "warmup": a.warmup, "ms_per_step": head.pop("ms_per_step"),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": a.dtype,
            "data": "synthetic",
            "config": {
                "workload": head.pop("workload"), "n_global": head.pop("n_global"),
                "nnz_global": head.pop("nnz_global"), "ranks": world,
                "parallelism": head.pop("parallelism"),
                "exchange_selection": head.pop("exchange_selection"),
                "execution": head.pop("execution"), "execution_selection": head.pop("execution_selection"),
                "schedule": head.pop("schedule"),
                "l2": head.pop("l2"),
                "step_timing": ("CUDA events recorded by dspmv_apply on the caller stream at START "
                                "and END (the whole schedule incl. host syncs); max over ranks; "
                                f"{a.settle_s:g} s idle before the warm-up (power controller)"),
                "step_us_median_min_p90": head.pop("step_us_median_min_p90"),
                **{k: head.pop(k) for k in ("step_us_median_warm_l2", "step_us_median_flushed_l2") if k in head},
                "step_hbm_gbs_algorithmic": head.pop("step_hbm_gbs_algorithmic"),
                "yL_window_in_step_us_median": head.pop("yL_window_in_step_us_median"),
                "wall_s_timed_region": head.pop("wall_s_timed_region"),
                "values": {"mode": "exact" if EXACT else "float", "x_seed": X_SEED, "matrix_seed": 2203},
                "build": build_ids(),
            },
            "roofline": head.pop("roofline"),
            "parity_ok": head["parity"]["ok"], "parity": head.pop("parity"),
            "e2e": head.pop("e2e"),
            "gpu_launches": launches + sum(s["gpu_launches"] for s in secs.values()),
            "gpu_launches_detail": {"headline_timed_region": launches,
                                    "l2_flush_per_step": int(head.pop("_flushed")),
                                    "secondary_timed_regions": {w: s["gpu_launches"] for w, s in secs.items()}},
            "clocks": clk,
        }
        for k in ("schedule_sweep", "exchange", "overlap"):
            if k in head:
                out[k] = head.pop(k)
        if scaling:
            out["scaling_efficiency"] = scaling
        if secs:
            out["secondary"] = secs
            out["parity_ok"] = out["parity_ok"] and all(s["parity"]["ok"] for s in secs.values())
        if cpu is not None:
            out["cpu_baseline"] = cpu
        emit(json.dumps(out))
    ctx.close()


# ----------------------------------------------------------- oracle legs
def cpu_baseline(workload_name, budget_s=10.0):
    """The oracle O1 (oracle/o1.c, serial, unmodified) on the same matrix and x
    as the GPU run (N=1); repeats the full SpMV until `budget_s` of CPU work."""
    import gen
    from oracle import spmv as O1
    n, rp, col, val = workload_rows(workload_name, 0, workload_n(workload_name))
    desc = workload_desc(workload_name, 1)
    x = xvals(0, n)
    O1.o1_spmv(rp, col, val, x)  # warm
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        O1.o1_spmv(rp, col, val, x)
        reps += 1
    dt = time.perf_counter() - t0
    nnz = int(rp[-1])
    # the same loop over rows on all host cores (OpenMP, static)
    O1.o1_spmv_omp(rp, col, val, x)  # warm
    reps_m, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s / 2:
        O1.o1_spmv_omp(rp, col, val, x)
        reps_m += 1
    dt_m = time.perf_counter() - t0
    threads = O1.o1_threads()
    return {"value": round(2.0 * nnz * reps / dt / 1e9, 4), "unit": "GFLOP/s", "cores": 1,
            "kind": "oracle",
            "sample": f"full {desc}: {reps} O1 SpMVs ({nnz} nnz each) in {dt:.2f} s, 1 thread",
            "all_cores": {"value": round(2.0 * nnz * reps_m / dt_m / 1e9, 4), "unit": "GFLOP/s",
                          "cores": threads,
                          "sample": f"full {desc}: {reps_m} O1 SpMVs, rows over {threads} OpenMP threads "
                                    f"(static schedule) in {dt_m:.2f} s"},
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(a, budget_s=90.0):
    """The oracle as the reference arm: rank 0 only; others exit 0.  Each
    step is O1 over a bounded prefix of the workload's rows, sized so all
    W + K steps take about `budget_s`."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import gen
    from oracle import spmv as O1
    n = workload_n(a.workload)
    probe = min(n, 1 << 18)
    _, rp, col, val = workload_rows(a.workload, 0, probe)
    x = xvals(0, n)
    t0 = time.perf_counter()
    O1.o1_spmv(rp, col, val, x)
    t_probe = max(time.perf_counter() - t0, 1e-6)
    per_row = t_probe / probe
    rows = int(min(n, max(probe, budget_s / max(1, a.steps + a.warmup) / per_row)))
    if rows > probe:
        _, rp, col, val = workload_rows(a.workload, 0, rows)
    for _ in range(a.warmup):
        O1.o1_spmv(rp, col, val, x)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        O1.o1_spmv(rp, col, val, x)
    dt = time.perf_counter() - t0
    nnz = int(rp[-1])
    gflops = 2.0 * nnz * a.steps / dt / 1e9
    desc = workload_desc(a.workload, world)
    sample = (f"rows [0,{rows}) of {n} ({nnz} nnz) per step, O1 serial, 1 thread"
              + (" (the whole matrix)" if rows == n else " (bounded sample)"))
    emit(json.dumps({
        "metric": METRIC, "value": round(gflops, 4), "unit": "GFLOP/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(dt / a.steps * 1e3, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": a.dtype,
        "data": "synthetic", "impl": "reference",
        "config": {"workload": desc, "sample": sample},
        "cpu_baseline": {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": 1,
                         "kind": "oracle", "sample": sample, "cpu": _cpu_model()},
        "e2e": {"value": round(gflops, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }))


_JSON_OUT = None   # the process's real stdout while fd 1 points at stderr


def emit(line: str):
    """The one JSON line on stdout (libraries' own prints, e.g. NCCL's version
    banner under NCCL_DEBUG, go to stderr while the bench runs)."""
    if _JSON_OUT is not None:
        _JSON_OUT.write(line + "\n")
        _JSON_OUT.flush()
    else:
        print(line, flush=True)


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)   # everything else written to fd 1 (C libraries included) -> stderr
    a = parse()
    global X_SEED, EXACT
    X_SEED, EXACT = a.seed, a.value_mode == "exact"
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
