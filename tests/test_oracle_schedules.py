"""Pins for oracle/schedules.py: Appendix-A counts, paper sequences, tab:sync."""
import os

import pytest

from oracle import schedules as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_counts():
    out = []
    for line in open(os.path.join(GOLDEN, "schedule_counts.txt")):
        if line.startswith("#") or not line.strip():
            continue
        a, b, c = line.split()
        out.append((a, int(b), int(c)))
    return out


@pytest.mark.parametrize("reading,n_streams,count", _golden_counts())
def test_counts_match_appendix_a(reading, n_streams, count):
    if reading == "topo_orders_A":
        assert len(S.topological_orders(S.EDGES_A)) == count
        return
    edges = S.EDGES_A if reading == "A" else S.EDGES
    assert len(S.enumerate_derived(n_streams, edges)) == count


def _paper_seqs():
    seqs = []
    for line in open(os.path.join(GOLDEN, "paper_sequences.txt")):
        if line.startswith("#") or not line.strip():
            continue
        seqs.append(line.split())
    return seqs


@pytest.mark.parametrize("seq", _paper_seqs())
@pytest.mark.parametrize("streams", [(0, 0, 0, 0), (0, 1, 0, 1), (1, 0, 0, 1)])
def test_paper_sequences_valid(seq, streams):
    """both example sequences are valid traversals."""
    assert S.topological_orders  # noqa
    pos = {v: i for i, v in enumerate(seq)}
    for (u, v) in S.EDGES:
        assert pos[u] < pos[v]
    ops = S.derive(seq, dict(zip(["Pack", "y_L", "Unpack", "y_R"], streams)))
    assert S.validate(ops, 2) == (True, "", "")


def test_pack_to_postsend_inserts_cer_ces():
    """edge (2)->(4) requires a synchronisation; tab:sync row 2:
    cudaEventRecord -> cudaEventSynchronize (named CER-after-Pack /
    CES-b4-PostSend)."""
    seq = _paper_seqs()[0]
    ops = S.derive(seq, {"Pack": 0, "y_L": 0, "Unpack": 0, "y_R": 0})
    i = ops.index(("PostSend",))
    assert ops[i - 2][0] == "CER" and ops[i - 2][1] == 0
    assert ops[i - 1][0] == "CES" and ops[i - 1][1] == ops[i - 2][2]


def test_same_stream_needs_nothing_cross_stream_needs_cswe():
    """tab:sync rows 3-4: GPU_i->GPU_i none; GPU_i->GPU_j CER -> CSWE."""
    seq = ["start", "PostRecv", "Pack", "PostSend", "WaitRecv", "Unpack", "y_R",
           "y_L", "WaitSend", "end"]
    same = S.derive(seq, {"Pack": 0, "y_L": 0, "Unpack": 0, "y_R": 0})
    i = same.index(("y_R", 0))
    assert same[i - 1] == ("Unpack", 0)
    cross = S.derive(seq, {"Pack": 0, "y_L": 0, "Unpack": 0, "y_R": 1})
    i = cross.index(("y_R", 1))
    assert cross[i - 2][0] == "CER" and cross[i - 2][1] == 0
    assert cross[i - 1] == ("CSWE", 1, cross[i - 2][2])


def test_every_derived_schedule_valid_and_needs_its_syncs():
    """Every derived schedule validates; removing CES-b4-PostSend (the
    P:432 sync) or every sync op breaks it; removing a CER whose event is
    consumed is a structural error."""
    scheds = S.enumerate_derived(2, S.EDGES)
    for ops in scheds:
        assert S.validate(ops, 2)[0]
        i = ops.index(("PostSend",))
        assert ops[i - 1][0] == "CES"
        assert not S.validate(ops[:i - 1] + ops[i:], 2)[0]
        nosync = [o for o in ops if o[0] not in ("CER", "CES", "CSWE")]
        assert not S.validate(nosync, 2)[0]
        for t, op in enumerate(ops):
            if op[0] == "CER":
                assert not S.validate(ops[:t] + ops[t + 1:], 2)[0]


def test_canonical_key_invariant_under_stream_swap():
    for ops in S.enumerate_derived(2, S.EDGES)[:200]:
        sw = []
        for op in ops:
            if op[0] in S.GPU_VERTICES:
                sw.append((op[0], 1 - op[1]))
            elif op[0] in ("CER", "CSWE"):
                sw.append((op[0], 1 - op[1], op[2]))
            else:
                sw.append(op)
        assert S.canonical(sw) == S.canonical(ops)
        assert S.canonical(S.canonical(ops)) == S.canonical(ops)


def test_deadlock_orders_classified():
    seq = ["start", "PostRecv", "WaitRecv", "Pack", "PostSend", "WaitSend",
           "Unpack", "y_L", "y_R", "end"]
    ops = S.derive(seq, {"Pack": 0, "y_L": 0, "Unpack": 0, "y_R": 0}, S.EDGES_A)
    ok, kind, _ = S.validate(ops, 2)
    assert not ok and kind == "deadlock"


def test_validator_rejects_structural_errors():
    good = S.derive(_paper_seqs()[0], {"Pack": 0, "y_L": 1, "Unpack": 0, "y_R": 1})
    assert S.validate(good, 2)[0]
    assert not S.validate(good, 1)[0]                        # stream out of range
    assert not S.validate(good[:-1], 2)[0]                   # missing end
    assert not S.validate(good + [("end",)], 2)[0]           # duplicate
    ces = next(t for t, o in enumerate(good) if o[0] == "CES")
    bad = list(good)
    bad[ces] = ("CES", 99)                                   # unrecorded event
    assert not S.validate(bad, 2)[0]


def _orderable_golden():
    out = []
    for line in open(os.path.join(GOLDEN, "orderable_counts.txt")):
        if line.startswith("#") or not line.strip():
            continue
        a, b = line.split()
        out.append((a, int(b)))
    return out


@pytest.mark.parametrize("reading,count", _orderable_golden())
def test_orderable_sync_counts_match_appendix_a(reading, count):
    """Syncs as moves of their own (R-N5 "first-unmet"): the
    number of distinct schedules equals the surveyor's independent count."""
    edges = {"A+both": S.EDGES, "A+PostSend->WaitRecv": S.EDGES_A + [("PostSend", "WaitRecv")]}[reading]
    assert len(S.enumerate_orderable(2, edges)) == count


def test_orderable_space_covers_the_derived_space_and_is_valid():
    """Every traversal + stream binding of the derived space is reached (the
    syncs may differ: an event already recorded after u is reused), and every
    orderable schedule is valid."""
    orderable = S.enumerate_orderable(2)

    def proj(o):
        return tuple(op for op in S.canonical(o) if op[0] in S.VERTICES)
    keys = {proj(o) for o in orderable}
    assert all(proj(o) in keys for o in S.enumerate_derived(2))
    assert all(S.validate(o, 2) == (True, "", "") for o in orderable)
    # a sync placed away from its consumer exists (what the derived space lacks)
    assert any(o[i][0] == "CER" and o[i + 1][0] not in ("CES", "CSWE") for o in orderable for i in range(len(o) - 1))
