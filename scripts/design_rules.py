#!/usr/bin/env python
"""The paper's end-to-end experiment on B200 (NEXT-1 + NEXT-2; §III-C,
§IV, §V): measure every schedule of the DAG with the paper's protocol, label
performance classes, train the CART tree (Algorithm 1), print the rulesets,
then run MCTS for 50/100/200/400 iterations and report the Table V class
accuracy against the exhaustive space.

    python scripts/design_rules.py --workload g3 --ranks 4 --out profiles/r1_rules_g3.json

g3 = the paper's banded 150K matrix on `ranks` in-process LOCAL
ranks of one B200 (only one GPU is reachable this round); c2 = 7-pt 128^3 on
one rank (NCCL comm of size 1).

--granularity fine: the per-destination DAG (DESIGN.md R-N4) of the
peer offsets the partition uses.  Its space cannot be enumerated, so MCTS and
the random-rollout baseline sample it with equal budgets; rules
are learned from the MCTS samples and checked on the random samples, and the
best schedules are compared with the coarse sweep's.
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
from paper_2203_02530_b200 import dspmv as D  # noqa: E402
from paper_2203_02530_b200 import mcts as M  # noqa: E402
from paper_2203_02530_b200 import rules as R  # noqa: E402
from paper_2203_02530_b200 import schedules as PS  # noqa: E402


def peer_offsets(workload, ranks):
    """Rank offsets d with some rank r sending to r+d (plus their negatives)."""
    if workload == "g3":
        n = 150000
        rp, col, _ = gen.banded(n)
    elif workload in ("c5", "c5b"):
        n, (rp, col, _) = gen.config_matrix(workload)
    else:
        n, (rp, col, _) = gen.config_matrix("c2")
    rb = np.asarray(D.dspmv_partition(n, ranks))
    row_owner = np.repeat(np.arange(ranks), np.diff(rb))
    nnz_owner = np.repeat(row_owner, np.diff(rp))
    col_owner = np.searchsorted(rb, col, side="right") - 1
    d = np.unique(col_owner - nnz_owner)
    d = set(int(v) for v in d if v != 0)
    return sorted(d | {-v for v in d})


def setup(workload, ranks):
    if workload == "g3":
        n = 150000
        rp, col, val = gen.banded(n)
    elif workload in ("c5", "c5b"):
        n, (rp, col, val) = gen.config_matrix(workload)
    else:
        n, (rp, col, val) = gen.config_matrix("c2")
    x = gen.x_values((0, n))
    rb = D.dspmv_partition(n, ranks)
    if ranks == 1:
        comms = [D.dspmv_comm_create(D.dspmv_comm_unique_id(), 1, 0, 0)]
    else:
        comms = D.dspmv_comm_create_local(ranks, 0)
    plans, xs, ys = [], [], []
    for r in range(ranks):
        b, e = int(rb[r]), int(rb[r + 1])
        lo, hi = int(rp[b]), int(rp[e])
        plans.append(D.dspmv_plan_create(comms[r], n, rp[b:e + 1], col[lo:hi], val[lo:hi]))
        xs.append(torch.from_numpy(x[b:e].copy()).cuda())
        ys.append(torch.empty(e - b, dtype=torch.float64, device="cuda"))
    return comms, plans, xs, ys


def make_measure(plans, xs, ys, t_measure=0.01):
    stream = torch.cuda.current_stream()
    ranks = len(plans)

    def apply(ss):
        if ranks == 1:
            D.dspmv_apply(ss[0], xs[0], ys[0], stream)
        else:
            D.dspmv_apply_group(ss, xs, ys, stream)

    def measure(ops, n_meas=3):
        """a measurement repeats samples until t_measure has
        elapsed, time = t_measure / n_samples (one process drives every rank
        here); f = mean of n_meas measurements (R-Q19)."""
        ss = [D.dspmv_schedule_create(p, ops, 2) for p in plans]
        for _ in range(2):
            apply(ss)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        apply(ss)
        n = max(1, math.ceil(t_measure / max(time.perf_counter() - t0, 1e-7)))
        ts = []
        for _ in range(n_meas):
            t0 = time.perf_counter()
            for _ in range(n):
                apply(ss)
            ts.append((time.perf_counter() - t0) / n)
        for s in ss:
            D.dspmv_schedule_destroy(s)
        return float(np.mean(ts))
    return measure


def setup_distributed(workload, comm_kind):
    """One process per rank (torchrun): this rank's rows, NCCL comm (or the
    HOST-transport comm with the fused put exchange for ranks sharing a GPU)."""
    import torch.distributed as dist
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dev = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    if comm_kind == "host":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    if workload == "g3":
        n = 150000
        rp, col, val = gen.banded(n)
    elif workload in ("c5", "c5b"):
        n, (rp, col, val) = gen.config_matrix(workload)
    else:
        n, (rp, col, val) = gen.config_matrix("c2")
    rb = D.dspmv_partition(n, world)
    b, e = int(rb[rank]), int(rb[rank + 1])
    lo, hi = int(rp[b]), int(rp[e])
    if comm_kind == "host":
        def allgather(bb):
            out = [None] * world
            dist.all_gather_object(out, bb)
            return b"".join(out)
        comm = D.dspmv_comm_create_host(world, rank, dev, allgather)
        ex = D.DSPMV_EXCHANGE_PUT
    else:
        uid = [D.dspmv_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = D.dspmv_comm_create(uid[0], world, rank, dev)
        ex = D.DSPMV_EXCHANGE_COPY
    plan = D.dspmv_plan_create(comm, n, rp[b:e + 1], col[lo:hi], val[lo:hi], exchange=ex)
    x = torch.from_numpy(gen.x_values((b, e))).cuda()
    y = torch.empty_like(x)
    return dist, world, rank, comm, plan, x, y


def make_measure_distributed(dist, rank, plan, x, y, t_measure=0.01, n_meas=3):
    """P:460-464 across processes: rank 0 proposes ops, every rank builds the
    schedule, rank 0 calibrates n_samples (broadcast, R-Q19), every rank times
    the same number of samples, time = max over ranks, f = mean of n_meas."""
    red = "cpu" if dist.get_backend() == "gloo" else "cuda"

    def measure(ops):
        box = [ops]
        dist.broadcast_object_list(box, src=0)         # P:460 "broadcast to all ranks"
        ops = box[0]
        if ops is None:
            return None
        s = D.dspmv_schedule_create(plan, ops, 2)
        for _ in range(2):
            D.dspmv_apply(s, x, y)
        dist.barrier()
        t0 = time.perf_counter()
        D.dspmv_apply(s, x, y)
        n = torch.tensor([max(1, math.ceil(t_measure / max(time.perf_counter() - t0, 1e-7)))], device=red)
        dist.broadcast(n, src=0)
        ts = []
        for _ in range(n_meas):
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(int(n.item())):
                D.dspmv_apply(s, x, y)
            tt = torch.tensor([(time.perf_counter() - t0) / int(n.item())], dtype=torch.float64, device=red)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ts.append(float(tt.item()))
        D.dspmv_schedule_destroy(s)
        return float(np.mean(ts))
    return measure


def sweep_with_resume(space, measure, path):
    """Measure every schedule of `space` in order; with `path` (JSONL), each
    measured schedule is appended as {"i", "schedule", "t"} and flushed, and a
    restarted sweep reuses the lines whose index and schedule text match, so a
    sweep of the 4,780-schedule space survives a lost lease."""
    done = {}
    if path and os.path.exists(path):
        for line in open(path):
            try:
                r = json.loads(line)
            except ValueError:
                continue                                  # a torn last line
            done[int(r["i"])] = r
    f = open(path, "a") if path else None
    if f and os.path.getsize(path) > 0:
        with open(path, "rb") as g:
            g.seek(-1, os.SEEK_END)
            if g.read(1) != b"\n":
                f.write("\n")                          # end a torn last line
    times = []
    reused = 0
    for i, ops in enumerate(space):
        text = PS.describe(ops)
        r = done.get(i)
        if r is not None and r.get("schedule") == text:
            times.append(float(r["t"]))
            reused += 1
            continue
        t = measure(ops)
        times.append(t)
        if f:
            f.write(json.dumps({"i": i, "schedule": text, "t": t}) + "\n")
            f.flush()
    if f:
        f.close()
    return np.array(times), reused


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="g3", choices=["g3", "c2", "c5", "c5b"])
    ap.add_argument("--ranks", type=int, default=4, help="in-process ranks (single process mode)")
    ap.add_argument("--comm", default=None, choices=[None, "nccl", "host"],
                    help="torchrun mode: one process per rank over NCCL (or host + fused put)")
    ap.add_argument("--out", default="gpurun_out/rules.json")
    ap.add_argument("--granularity", default="coarse", choices=["coarse", "fine"])
    ap.add_argument("--budget", type=int, default=800, help="fine: MCTS / random-rollout samples")
    ap.add_argument("--syncs", default="derived", choices=["derived", "orderable"],
                    help="orderable: syncs are moves of their own (R-N5; 4,780 coarse schedules)")
    ap.add_argument("--resume", default=None,
                    help="JSONL checkpoint of the sweep: measured schedules are appended, a rerun skips them")
    a = ap.parse_args()
    if a.comm is not None:
        return main_distributed(a)
    if a.granularity == "fine":
        return main_fine(a)
    comms, plans, xs, ys = setup(a.workload, a.ranks)
    measure = make_measure(plans, xs, ys)
    space = PS.enumerate_orderable(2) if a.syncs == "orderable" else PS.enumerate_derived(2)
    t0 = time.perf_counter()
    times, reused = sweep_with_resume(space, measure, a.resume)
    sweep_s = time.perf_counter() - t0
    labels, ranges, bounds = R.class_labels(times)
    X, cols = R.features(space)
    clf, mln, hist = R.train_tree(X, labels)
    rs = R.rulesets(clf, cols)
    out = {
        "workload": a.workload, "ranks": a.ranks, "syncs": a.syncs, "n_schedules": len(space),
        "sweep_wall_s": round(sweep_s, 2),
        "fastest_us": float(times.min() * 1e6), "slowest_us": float(times.max() * 1e6),
        "fast_slow_ratio": float(times.max() / times.min()),
        "sorted_times_us": [round(float(t) * 1e6, 3) for t in np.sort(times)],
        "classes": {str(k): {"range_us": [v[0] * 1e6, v[1] * 1e6], "count": int((labels == k).sum())}
                    for k, v in ranges.items()},
        "tree": {"max_leaf_nodes": int(mln), "depth": int(clf.get_depth()),
                 "train_error": float(1 - (clf.predict(X) == labels).mean()),
                 "alg1_history": [[int(m), float(e), int(d)] for m, e, d in hist]},
        "rulesets": {str(k): [{"samples": n, "rules": r} for n, r in v[:3]] for k, v in rs.items()},
        "fastest": PS.describe(space[int(times.argmin())]),
        "slowest": PS.describe(space[int(times.argmax())]),
    }
    # Table V protocol: MCTS subsets vs the exhaustive space
    acc = {}
    for iters in (50, 100, 200, 400):
        m = M.MCTS(measure, n_streams=2, seed=2203, syncs=a.syncs).run(iters)
        recs = m.records()
        sub_ops = [o for o, _ in recs]
        sub_t = np.array([t for _, t in recs])
        acc[str(iters)] = {"distinct": len(recs),
                           "accuracy": R.class_accuracy(sub_ops, sub_t, space, times),
                           "best_found_us": float(sub_t.min() * 1e6)}
    out["mcts_table_v"] = acc
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "sorted_times_us"}, indent=1))
    for p in plans:
        D.dspmv_plan_destroy(p)
    for c in comms:
        D.dspmv_comm_destroy(c)


def main_fine(a):
    import random
    offs = peer_offsets(a.workload, a.ranks)
    sp = PS.Space(offs)
    comms, plans, xs, ys = setup(a.workload, a.ranks)
    measure = make_measure(plans, xs, ys)
    t0 = time.perf_counter()
    coarse = PS.enumerate_derived(2)
    ct = np.array([measure(o) for o in coarse])
    coarse_s = time.perf_counter() - t0
    # MCTS over the per-destination space
    t0 = time.perf_counter()
    m = M.MCTS(measure, n_streams=2, seed=2203, space=sp).run(a.budget)
    mcts_s = time.perf_counter() - t0
    recs = m.records()
    mo = [o for o, _ in recs]
    mt = np.array([t for _, t in recs])
    # random-rollout baseline with the same budget
    rng = random.Random(2530)
    ro, rt = [], []
    seen = set()
    while len(ro) < a.budget:
        prefix = []
        while True:
            mv = M.legal_moves(prefix, 2, sp)
            if not mv:
                break
            prefix.append(rng.choice(mv))
        ops = M.ops_of(prefix, 2, sp)
        k = PS.canonical_key(ops)
        if k in seen:
            continue
        seen.add(k)
        ro.append(ops)
        rt.append(measure(ops))
    rt = np.array(rt)
    labels, ranges, _ = R.class_labels(mt)
    X, cols = R.features(mo)
    clf, mln, hist = R.train_tree(X, labels)
    rs = R.rulesets(clf, cols)
    out = {
        "workload": a.workload, "ranks": a.ranks, "granularity": "per-destination (P:281-284)",
        "offsets": offs, "n_vertices": len(sp.vertices), "budget": a.budget,
        "coarse": {"n_schedules": len(coarse), "fastest_us": float(ct.min() * 1e6),
                   "slowest_us": float(ct.max() * 1e6), "fast_slow_ratio": float(ct.max() / ct.min()),
                   "fastest": PS.describe(coarse[int(ct.argmin())]), "sweep_wall_s": round(coarse_s, 1)},
        "mcts": {"distinct": len(recs), "fastest_us": float(mt.min() * 1e6), "slowest_us": float(mt.max() * 1e6),
                 "fast_slow_ratio": float(mt.max() / mt.min()), "median_us": float(np.median(mt) * 1e6),
                 "fastest": PS.describe(mo[int(mt.argmin())]), "wall_s": round(mcts_s, 1),
                 "best_after": {str(k): float(min(mt[:k]) * 1e6) for k in (50, 100, 200, 400, a.budget)
                                if k <= len(mt)}},
        "random": {"distinct": len(ro), "fastest_us": float(rt.min() * 1e6), "slowest_us": float(rt.max() * 1e6),
                   "median_us": float(np.median(rt) * 1e6),
                   "best_after": {str(k): float(min(rt[:k]) * 1e6) for k in (50, 100, 200, 400, a.budget)
                                  if k <= len(rt)}},
        "fine_vs_coarse_best": float(ct.min() / mt.min()),
        "classes": {str(k): {"range_us": [v[0] * 1e6, v[1] * 1e6], "count": int((labels == k).sum())}
                    for k, v in ranges.items()},
        "tree": {"max_leaf_nodes": int(mln), "depth": int(clf.get_depth()),
                 "train_error": float(1 - (clf.predict(X) == labels).mean())},
        "rulesets": {str(k): [{"samples": n, "rules": r} for n, r in v[:3]] for k, v in rs.items()},
        # Table V protocol with the random samples standing in for the
        # (unenumerable) full space
        "accuracy_on_random_samples": {str(k): R.class_accuracy(mo[:k], mt[:k], ro, rt)
                                       for k in (100, 200, 400, a.budget) if k <= len(mo)},
    }
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out, indent=1))
    for p in plans:
        D.dspmv_plan_destroy(p)
    for c in comms:
        D.dspmv_comm_destroy(c)


def analyse(space, times, measure_sub, workload, ranks, sweep_s, syncs="derived", execution=None):
    labels, ranges, bounds = R.class_labels(times)
    X, cols = R.features(space)
    clf, mln, hist = R.train_tree(X, labels)
    rs = R.rulesets(clf, cols)
    out = {
        "workload": workload, "ranks": ranks, "syncs": syncs, "execution_model": execution,
        "n_schedules": len(space), "sweep_wall_s": round(sweep_s, 2),
        "fastest_us": float(times.min() * 1e6), "slowest_us": float(times.max() * 1e6),
        "fast_slow_ratio": float(times.max() / times.min()),
        "sorted_times_us": [round(float(t) * 1e6, 3) for t in np.sort(times)],
        "classes": {str(k): {"range_us": [v[0] * 1e6, v[1] * 1e6], "count": int((labels == k).sum())}
                    for k, v in ranges.items()},
        "tree": {"max_leaf_nodes": int(mln), "depth": int(clf.get_depth()),
                 "train_error": float(1 - (clf.predict(X) == labels).mean())},
        "rulesets": {str(k): [{"samples": n, "rules": r} for n, r in v[:3]] for k, v in rs.items()},
        "fastest": PS.describe(space[int(times.argmin())]),
        "slowest": PS.describe(space[int(times.argmax())]),
    }
    acc = {}
    for iters in (50, 100, 200, 400):
        m = M.MCTS(measure_sub, n_streams=2, seed=2203, syncs=syncs).run(iters)
        recs = m.records()
        sub_t = np.array([t for _, t in recs])
        acc[str(iters)] = {"distinct": len(recs),
                           "accuracy": R.class_accuracy([o for o, _ in recs], sub_t, space, times),
                           "best_found_us": float(sub_t.min() * 1e6)}
    out["mcts_table_v"] = acc
    # class counts under the three readings of P:508 (DESIGN.md R-N2)
    out["classes_by_threshold"] = {th: len(R.class_labels(times, threshold=th)[1])
                                   for th in ("signal", "peaks", "mad")}
    return out


def main_distributed(a):
    dist, world, rank, comm, plan, x, y = setup_distributed(a.workload, a.comm)
    measure = make_measure_distributed(dist, rank, plan, x, y)
    if rank == 0:
        space = PS.enumerate_orderable(2) if a.syncs == "orderable" else PS.enumerate_derived(2)
        t0 = time.perf_counter()
        times, reused = sweep_with_resume(space, measure, a.resume)
        model = (f"SPMD: {world} processes, one rank each, "
                 + ("NCCL communicator, NCCL send/recv exchange" if a.comm == "nccl" else
                    "HOST communicator (gloo bootstrap), fused Pack+put exchange over CUDA IPC")
                 + f", {torch.cuda.device_count()} GPU(s) visible")
        out = analyse(space, times, measure, a.workload, world, time.perf_counter() - t0, a.syncs, model)
        measure(None)                                     # release the other ranks
        json.dump(out, open(a.out, "w"), indent=1)
        print(json.dumps({k: v for k, v in out.items() if k != "sorted_times_us"}, indent=1))
    else:
        while measure(None) is not None:                  # follow rank 0's proposals
            pass
    D.dspmv_plan_destroy(plan)
    D.dspmv_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
