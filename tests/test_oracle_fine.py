"""Pins for the per-destination ("fine") schedule DAG of the oracle
(reading R-N4): structure, reduction to the coarse DAG,
and the deadlock rule checked against the lock-step MPI simulation."""
import random

import numpy as np
import pytest

import gen
from oracle import plan as O2
from oracle import schedules as S


def random_topo(V, E, rng):
    pred = {v: set() for v in V}
    for u, v in E:
        pred[v].add(u)
    done, out = set(), []
    while len(out) < len(V):
        ready = [v for v in V if v not in done and pred[v] <= done]
        v = rng.choice(ready)
        out.append(v)
        done.add(v)
    return out


def used_offsets(plans):
    return sorted({q - r for r, pl in enumerate(plans) for q in range(len(plans)) if pl["send_count"][q] > 0})


@pytest.mark.parametrize("d", [1, -2])
def test_single_offset_dag_is_the_coarse_dag(d):
    V, E, Dl = S.fine_dag([d])
    strip = lambda v: S.base(v)  # noqa: E731
    assert sorted(map(strip, V)) == sorted(S.VERTICES)
    assert {(strip(u), strip(v)) for u, v in E} == set(S.EDGES)
    assert {(strip(u), strip(v)) for u, v in Dl} == set(S.DEADLOCK_EDGES)
    assert len(S.topological_orders(E, V)) == len(S.topological_orders(S.EDGES))


def test_fine_dag_structure():
    V, E, Dl = S.fine_dag([-1, 1])
    assert len(V) == 4 + 6 * 2 and len(set(V)) == len(V)
    assert len(E) == 3 + 4 * 2 + 4 * 2 + 2 * 2
    assert all(u in V and v in V for u, v in E)
    # acyclic, every vertex on a start -> end path
    succ = {v: [w for u, w in E if u == v] for v in V}
    pred = {v: [u for u, w in E if w == v] for v in V}
    assert len(random_topo(V, E, random.Random(0))) == len(V)

    def reach(a, nxt):
        seen, st = {a}, [a]
        while st:
            for w in nxt[st.pop()]:
                if w not in seen:
                    seen.add(w)
                    st.append(w)
        return seen
    assert reach("start", succ) == set(V) and reach("end", pred) == set(V)
    # the deadlock edges pair a rank's post with the peer's wait: PostSend[+1]
    # (to r+1) must precede WaitRecv[-1] (from r-1, whose matching send is its
    # own PostSend[+1] at the same position of the SPMD program)
    assert ("PostSend[+1]", "WaitRecv[-1]") in Dl and ("PostRecv[+1]", "WaitSend[-1]") in Dl


def _workloads():
    n1, (rp1, c1, v1) = gen.config_matrix("c1", exact=True)            # 5-pt, offsets +-1
    n2 = 600
    rp2, c2, v2 = gen.banded(n2, 6000, 150, exact=True)                 # offsets +-1, +-2 at P=6
    return [("c1-P3", n1, rp1, c1, v1, 3), ("banded-P6", n2, rp2, c2, v2, 6)]


@pytest.mark.parametrize("wl", _workloads(), ids=lambda w: w[0])
def test_fine_deadlock_rule_matches_simulation(wl):
    """Random traversals of the fine DAG without its deadlock edges: the static
    rule (a Wait before the peer's matching Post in the SPMD program) holds
    exactly when the lock-step MPI simulation deadlocks; every other
    traversal gives the serial product exactly (integer-valued inputs)."""
    _, n, rp, col, val, P = wl
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, P)
    offs = used_offsets(plans)
    assert len(offs) >= 2
    V, E, Dl = S.fine_dag(offs)
    base_edges = [e for e in E if e not in Dl]
    from oracle import spmv as O1
    yref = O1.o1_spmv(rp, col, val, x)
    rng = random.Random(2530)
    n_dead = n_ok = 0
    for _ in range(300):
        order = random_topo(V, base_edges, rng)
        pos = {v: i for i, v in enumerate(order)}
        static_dead = any(pos[u] > pos[v] for u, v in Dl)
        try:
            y = O2.simulate(plans, val, x, [(v,) for v in order])
            dyn_dead = False
        except O2.Deadlock:
            dyn_dead = True
        assert static_dead == dyn_dead, order
        if not dyn_dead:
            assert np.array_equal(y, yref)
            n_ok += 1
        n_dead += dyn_dead
    assert n_dead > 0 and n_ok > 0


def test_uncovered_offset_leaves_halo_unwritten():
    """A fine schedule must name every peer offset the plan uses: dropping the
    -1 direction leaves halo entries from rank r+1 unwritten (NaN in y)."""
    n, (rp, col, val) = gen.config_matrix("c1", exact=True)
    x = gen.x_values((0, n), exact=True)
    plans = O2.plan_all(rp, col, n, 3)
    V, E, _ = S.fine_dag([1])
    y = O2.simulate(plans, val, x, [(v,) for v in S.topological_orders(E, V)[0]])
    assert np.isnan(y).any()


def test_fine_validate_and_derive():
    V, E, Dl = S.fine_dag([-1, 1])
    rng = random.Random(7)
    for _ in range(20):
        order = random_topo(V, E, rng)
        streams = {v: rng.randrange(2) for v in V if S.base(v) in S.GPU_VERTICES}
        ops = S.derive(order, streams)
        assert S.validate(ops, 2) == (True, "", "")
    ops = S.derive(random_topo(V, E, rng), {v: 0 for v in V})
    # mixed granularity
    mixed = [("Pack", 0) if op[0] == "Pack[+1]" else op for op in ops]
    assert S.validate(mixed, 2)[:2] == (False, "schedule")
    # a vertex of one side missing
    assert S.validate([op for op in ops if op[0] != "Unpack[+1]"], 2)[:2] == (False, "schedule")
    # deadlock edge violated (WaitRecv[-1] moved before PostSend[+1])
    order = [v for v in V]
    order = random_topo(V, [e for e in E if e not in Dl], rng)
    while not any(order.index(u) > order.index(v) for u, v in Dl):
        order = random_topo(V, [e for e in E if e not in Dl], rng)
    dead = S.derive(order, {v: 0 for v in V}, [e for e in E if e not in Dl])
    assert S.validate(dead, 2)[:2] == (False, "deadlock")
