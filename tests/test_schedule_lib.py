"""The library's schedule layer (vector-clock validator, tab:sync derivation,
S:197 text format) against the oracle's happens-before graph enumerator."""
import itertools

import numpy as np
import random

import pytest

from oracle import schedules as S
from paper_2203_02530_b200 import dspmv as D

KIND = {v: i for i, v in enumerate(S.VERTICES)}
GPUS = ["Pack", "y_L", "Unpack", "y_R"]


def to_lib(ops):
    out = []
    for op in ops:
        n = op[0]
        b, d = S.split_name(n)
        if b in KIND:
            out.append((KIND[b], op[1] if b in S.GPU_VERTICES else 0, 0, d))
        elif n == "CER":
            out.append((D.DSPMV_OP_EVENT_RECORD, op[1], op[2], 0))
        elif n == "CES":
            out.append((D.DSPMV_OP_EVENT_SYNC, 0, op[1], 0))
        else:
            out.append((D.DSPMV_OP_STREAM_WAIT_EVENT, op[1], op[2], 0))
    return out


def lib_status(ops, n_streams=2):
    try:
        D.dspmv_schedule_validate(to_lib(ops), n_streams)
        return "ok"
    except D.DspmvError as e:
        return {D.DSPMV_ERR_SCHEDULE: "schedule", D.DSPMV_ERR_DEADLOCK: "deadlock"}[e.status]


def oracle_status(ops, n_streams=2):
    ok, kind, _ = S.validate(ops, n_streams)
    return "ok" if ok else kind


def test_derive_matches_oracle_for_every_order_and_stream_assignment():
    for edges in (S.EDGES,):
        for order in S.topological_orders(edges):
            for assign in itertools.product(range(2), repeat=4):
                streams = dict(zip(GPUS, assign))
                want = to_lib(S.derive(order, streams, edges))
                got = D.dspmv_schedule_derive([KIND[v] for v in order],
                                              [streams.get(v, 0) for v in order], 2)
                assert [tuple(r) for r in got] == want, order


def test_validator_agrees_with_oracle_on_all_derived_schedules():
    for ops in S.enumerate_derived(2, S.EDGES):
        assert lib_status(ops) == "ok"
    for ops in S.enumerate_derived(2, S.EDGES_A):      # 1408 of 2240 deadlock (R-Q13)
        assert lib_status(ops) == oracle_status(ops)


def _mutations(ops, rng):
    ops = list(ops)
    yield ops[:]                                         # identity
    for t in range(len(ops)):                            # drop one op
        yield ops[:t] + ops[t + 1:]
    for t in range(len(ops) - 1):                        # swap neighbours
        m = ops[:]
        m[t], m[t + 1] = m[t + 1], m[t]
        yield m
    for t, op in enumerate(ops):                         # re-stream one op
        if op[0] in S.GPU_VERTICES:
            yield ops[:t] + [(op[0], 1 - op[1])] + ops[t + 1:]
        if op[0] in ("CER", "CSWE"):
            yield ops[:t] + [(op[0], 1 - op[1], op[2])] + ops[t + 1:]
    for _ in range(5):                                   # move a sync op
        syncs = [t for t, o in enumerate(ops) if o[0] in ("CER", "CES", "CSWE")]
        if not syncs:
            break
        t = rng.choice(syncs)
        m = ops[:t] + ops[t + 1:]
        m.insert(rng.randrange(1, len(m)), ops[t])
        yield m


def test_validator_agrees_with_oracle_on_mutations():
    rng = random.Random(2203)
    scheds = S.enumerate_derived(2, S.EDGES)
    rng.shuffle(scheds)
    n = 0
    for ops in scheds[:250]:
        for m in _mutations(ops, rng):
            assert lib_status(m) == oracle_status(m), m
            n += 1
    assert n > 5000


def test_paper_sequences_and_parse_roundtrip():
    seq2 = ["start", "PostRecv", "y_L", "Pack", "PostSend", "WaitRecv", "WaitSend",
            "Unpack", "y_R", "end"]
    ops = D.dspmv_schedule_derive([KIND[v] for v in seq2], [0, 0, 1, 0, 0, 0, 0, 0, 1, 0], 2)
    D.dspmv_schedule_validate(ops, 2)
    text = D.dspmv_schedule_format(ops)
    assert "CES-b4-PostSend EventSync" in text
    back, ns = D.dspmv_schedule_parse(text)
    assert ns == 2 and (back == ops).all()


def test_parse_spec_format_example():
    text = """# S:197 external schedule format
start Cpu
Pack BoundGpu stream=0
CER-after-Pack EventRecord stream=0 event=0
CES-b4-PostSend EventSync event=0
PostSend PostSend
PostRecv PostRecv
WaitSend WaitSend
WaitRecv WaitRecv
y_L BoundGpu stream=1
Unpack BoundGpu stream=0
y_R BoundGpu stream=0
CER-after-y_R EventRecord stream=0 event=1
CES-b4-end EventSync event=1
CER-after-y_L EventRecord stream=1 event=2
CES-b4-end EventSync event=2
end Cpu
"""
    ops, ns = D.dspmv_schedule_parse(text)
    assert ns == 2 and len(ops) == 16
    D.dspmv_schedule_validate(ops, ns)
    with pytest.raises(D.DspmvError):
        D.dspmv_schedule_parse("Pack Cpu\n")             # kind/vertex mismatch
    with pytest.raises(D.DspmvError):
        D.dspmv_schedule_parse("foo BoundGpu stream=0\n")


def test_error_cases_of_the_boundary_table():
    good = D.dspmv_schedule_derive(list(range(10)), [0] * 10, 2)
    D.dspmv_schedule_validate(good, 2)

    def status(ops, ns=2):
        try:
            D.dspmv_schedule_validate(ops, ns)
            return D.DSPMV_OK
        except D.DspmvError as e:
            return e.status

    dup = list(map(tuple, good)) + [(D.DSPMV_OP_PACK, 0, 0, 0)]
    assert status(dup) == D.DSPMV_ERR_SCHEDULE                  # duplicated DAG op
    missing = [tuple(o) for o in good if o[0] != D.DSPMV_OP_UNPACK]
    assert status(missing) == D.DSPMV_ERR_SCHEDULE              # missing DAG op
    bad_stream = [tuple(o) for o in good]
    i = [o[0] for o in bad_stream].index(D.DSPMV_OP_PACK)
    bad_stream[i] = (D.DSPMV_OP_PACK, 3, 0, 0)
    assert status(bad_stream) == D.DSPMV_ERR_SCHEDULE           # stream >= n_streams
    unrec = [tuple(o) for o in good]
    j = [o[0] for o in unrec].index(D.DSPMV_OP_EVENT_SYNC)
    unrec[j] = (D.DSPMV_OP_EVENT_SYNC, 0, 33, 0)
    assert status(unrec) == D.DSPMV_ERR_SCHEDULE                # CES on unrecorded event
    nosync = [tuple(o) for o in good if o[0] < 10]
    assert status(nosync) == D.DSPMV_ERR_SCHEDULE               # missing tab:sync sync
    order = ["start", "PostRecv", "WaitRecv", "Pack", "PostSend", "WaitSend", "Unpack",
             "y_L", "y_R", "end"]
    dead = to_lib(S.derive(order, dict.fromkeys(GPUS, 0), S.EDGES_A))
    assert status(dead) == D.DSPMV_ERR_DEADLOCK                 # WaitRecv before PostSend


def test_product_enumerator_equals_oracle_enumerator():
    """The sweep's enumerator (package, library-derived syncs) yields exactly
    the oracle's brute-force set of 768 canonical schedules."""
    from paper_2203_02530_b200 import schedules as PS
    mine = {PS.canonical_key(o) for o in PS.enumerate_derived(2)}
    ref = {PS.canonical_key(np.array(to_lib(o), np.int32)) for o in S.enumerate_derived(2, S.EDGES)}
    assert len(mine) == 768 and mine == ref
    assert len(PS.topological_orders()) == 96


def _random_schedule(rng):
    """A random op list: a random order of the 10 vertices (not necessarily
    topological), random streams, and random CER / CES / CSWE insertions."""
    verts = S.VERTICES[1:-1]
    rng.shuffle(verts)
    ops = [("start",)]
    ev = 0
    recorded = []
    for v in verts:
        for _ in range(rng.choice([0, 0, 1, 2])):
            kind = rng.choice(["CER", "CES", "CSWE"])
            if kind == "CER" or not recorded:
                ops.append(("CER", rng.randrange(2), ev))
                recorded.append(ev)
                ev += 1
            elif kind == "CES":
                ops.append(("CES", rng.choice(recorded)))
            else:
                ops.append(("CSWE", rng.randrange(2), rng.choice(recorded)))
        ops.append((v, rng.randrange(2)) if v in S.GPU_VERTICES else (v,))
    for _ in range(rng.choice([1, 2, 3])):
        s_ = rng.randrange(2)
        ops.append(("CER", s_, ev))
        ops.append(("CES", ev))
        ev += 1
    ops.append(("end",))
    return ops


def test_validator_fuzz_random_schedules_vs_oracle():
    """Library validator (vector clocks) == oracle validator (explicit
    happens-before reachability) on 20000 random op lists."""
    rng = random.Random(2530)
    orders = S.topological_orders()
    n_ok = 0
    for i in range(20000):
        if i % 2:
            ops = _random_schedule(rng)
        else:
            # a derived schedule with one sync dropped and/or a random extra sync
            order = rng.choice(orders)
            streams = [rng.randrange(2) if v in S.GPU_VERTICES else 0 for v in order]
            ops = S.derive(order, dict(zip(order, streams)))
            if rng.random() < 0.5:
                syncs = [t for t, o in enumerate(ops) if o[0] in ("CER", "CES", "CSWE")]
                if syncs:
                    del ops[rng.choice(syncs)]
            if rng.random() < 0.5:
                recs = [o[-1] for o in ops if o[0] == "CER"]
                if recs:
                    t = rng.randrange(1, len(ops) - 1)
                    ops.insert(t, ("CES", rng.choice(recs)) if rng.random() < 0.5
                               else ("CSWE", rng.randrange(2), rng.choice(recs)))
        a, b = lib_status(ops), oracle_status(ops)
        assert a == b, ops
        n_ok += a == "ok"
    assert n_ok > 2000    # both valid and invalid schedules are exercised


def test_parse_rejects_garbage_without_crashing():
    rng = random.Random(7)
    words = ["start", "Pack", "y_L", "Cpu", "BoundGpu", "EventRecord", "EventSync", "StreamWaitEvent",
             "stream=1", "event=3", "stream=-1", "event=x", "#", "end", "PostSend"]
    for _ in range(3000):
        text = "\n".join(" ".join(rng.choice(words) for _ in range(rng.randrange(0, 5)))
                         for _ in range(rng.randrange(0, 20)))
        try:
            ops, ns = D.dspmv_schedule_parse(text)
            try:
                D.dspmv_schedule_validate(ops, ns)
            except D.DspmvError:
                pass
        except D.DspmvError:
            pass


# ------------------------------------------------ per-destination schedules
def _rand_topo(V, E, rng):
    pred = {v: {u for u, w in E if w == v} for v in V}
    done, out = set(), []
    while len(out) < len(V):
        v = rng.choice([v for v in V if v not in done and pred[v] <= done])
        out.append(v)
        done.add(v)
    return out


@pytest.mark.parametrize("offsets", [[1], [-1, 1], [-2, -1, 1, 2], [-3, 1]])
def test_fine_derive_matches_oracle(offsets):
    """dspmv_schedule_derive_peers == oracle derive on random traversals of the
    per-destination DAG (R-N4), every stream assignment sampled."""
    V, E, _ = S.fine_dag(offsets)
    rng = random.Random(len(offsets))
    for _ in range(300):
        order = _rand_topo(V, E, rng)
        streams = {v: rng.randrange(2) for v in order if S.base(v) in S.GPU_VERTICES}
        want = to_lib(S.derive(order, streams))
        kinds = [KIND[S.base(v)] for v in order]
        peers = [S.split_name(v)[1] for v in order]
        got = D.dspmv_schedule_derive_peers(kinds, [streams.get(v, 0) for v in order], peers, 2)
        assert [tuple(r) for r in got] == want, order
        assert lib_status(S.derive(order, streams)) == "ok"


def test_fine_validator_fuzz_vs_oracle():
    """Vector-clock validator == happens-before oracle on per-destination
    schedules: derived ones, derived with a sync dropped / a vertex moved /
    a vertex restreamed, and traversals that ignore the deadlock edges."""
    rng = random.Random(99)
    n_ok = n_dead = 0
    for i in range(3000):
        offsets = rng.choice([[-1, 1], [-2, -1, 1, 2], [2], [-3, 1]])
        V, E, Dl = S.fine_dag(offsets)
        edges = E if i % 3 else [e for e in E if e not in Dl]
        order = _rand_topo(V, edges, rng)
        streams = {v: rng.randrange(2) for v in order if S.base(v) in S.GPU_VERTICES}
        ops = S.derive(order, streams, edges)
        r = rng.random()
        if r < 0.25:
            syncs = [t for t, o in enumerate(ops) if o[0] in ("CER", "CES", "CSWE")]
            if syncs:
                del ops[rng.choice(syncs)]
        elif r < 0.5:
            t = rng.randrange(1, len(ops) - 1)
            op = ops.pop(t)
            ops.insert(rng.randrange(1, len(ops)), op)
        elif r < 0.6:
            t = rng.randrange(len(ops))
            if S.base(ops[t][0]) in S.GPU_VERTICES:
                ops[t] = (ops[t][0], 1 - ops[t][1])
        a, b = lib_status(ops), oracle_status(ops)
        assert a == b, ops
        n_ok += a == "ok"
        n_dead += a == "deadlock"
    assert n_ok > 500 and n_dead > 100


def test_fine_schedule_errors():
    V, E, _ = S.fine_dag([-1, 1])
    ops = S.derive(S.topological_orders(E, V)[0], {v: 0 for v in V})
    lib = to_lib(ops)
    D.dspmv_schedule_validate(lib, 1)
    mixed = [(k, s_, e, 0) if k == D.DSPMV_OP_PACK and p == 1 else (k, s_, e, p) for k, s_, e, p in lib]
    with pytest.raises(D.DspmvError, match="mixed"):
        D.dspmv_schedule_validate(mixed, 1)
    bad_peer = [(k, s_, e, 3) if k == D.DSPMV_OP_SPMV_LOCAL else (k, s_, e, p) for k, s_, e, p in lib]
    with pytest.raises(D.DspmvError, match="no peer offset"):
        D.dspmv_schedule_validate(bad_peer, 1)
    dup = lib[:2] + [lib[1]] + lib[2:]
    with pytest.raises(D.DspmvError):
        D.dspmv_schedule_validate(dup, 1)


def test_fine_parse_format_roundtrip():
    V, E, _ = S.fine_dag([-2, 1])
    rng = random.Random(3)
    for _ in range(50):
        order = _rand_topo(V, E, rng)
        ops = np.array(to_lib(S.derive(order, {v: rng.randrange(2) for v in V})), np.int32)
        text = D.dspmv_schedule_format(ops)
        assert "Pack[+1]" in text and "Unpack[+2]" in text
        back, ns = D.dspmv_schedule_parse(text)
        assert np.array_equal(back, ops)
    back, _ = D.dspmv_schedule_parse("start Cpu\nPack BoundGpu stream=0 peer=-1\n")
    assert back[1].tolist() == [D.DSPMV_OP_PACK, 0, 0, -1]


@pytest.mark.parametrize("offsets", [[], [1], [-1, 1], [-3, -1, 2]])
def test_library_dag_equals_oracle_dag(offsets):
    """dspmv_schedule_dag (used by the sweep / MCTS / rules) has exactly the
    oracle's vertices, edges and deadlock edges, with each vertex's
    predecessors in the oracle's order (it fixes the derived-sync order)."""
    verts, edges = D.dspmv_schedule_dag(offsets)
    names = [D.vertex_label(k, p) for k, p in verts]
    if offsets:
        V, E, Dl = S.fine_dag(offsets)
    else:
        V, E, Dl = S.VERTICES, S.EDGES, S.DEADLOCK_EDGES
    assert sorted(names) == sorted(V)
    got = [(names[u], names[v]) for u, v, _ in edges]
    assert set(got) == set(E) and len(got) == len(E)
    assert {(names[u], names[v]) for u, v, dead in edges if dead} == set(Dl)
    for v in V:
        assert [a for a, b in got if b == v] == S.preds(v, E)


def test_orderable_moves_and_space_match_oracle():
    """dspmv_schedule_moves (vector clocks) offers exactly the oracle's
    orderable_moves (happens-before graph) along every prefix, and the two
    enumerations give the same 4,780 schedules (R-N5)."""
    from paper_2203_02530_b200 import schedules as PS
    lib_space = PS.enumerate_orderable(2)
    assert len(lib_space) == 4780
    ora = S.enumerate_orderable(2)
    assert {PS.canonical_key(o) for o in lib_space} == {PS.canonical_key(to_lib(o)) for o in ora}
    rng = random.Random(1)
    for o in rng.sample(ora, 200):
        for t in range(len(o)):
            want = {tuple(m) for m in to_lib(S.orderable_moves(o[:t], 2))}
            got = {tuple(m) for m in D.dspmv_schedule_moves(to_lib(o[:t]), 2).tolist()}
            assert got == want, (o[:t], got, want)
        D.dspmv_schedule_validate(to_lib(o), 2)


def test_orderable_moves_per_destination_match_oracle():
    V, E, _ = S.fine_dag([-1, 1])
    rng = random.Random(4)
    for _ in range(40):
        ops = []
        while not ops or ops[-1][0] != "end":
            want = S.orderable_moves(ops, 2, E, V)
            got = {tuple(m) for m in D.dspmv_schedule_moves(to_lib(ops), 2, [-1, 1]).tolist()}
            assert got == {tuple(m) for m in to_lib(want)}, ops
            ops = ops + [rng.choice(want)]
        assert S.validate(ops, 2) == (True, "", "")
        D.dspmv_schedule_validate(to_lib(ops), 2)
