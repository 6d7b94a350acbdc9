"""Schedule-space enumeration for the design-space sweep (host logic).

The paper's design space is every traversal of the program DAG with every
stream assignment of its GPU vertices, synchronisation inserted per tab:sync
(§III-A/§III-C), streams pruned under
bijection.  Syncs are derived by the library
(``dspmv_schedule_derive``); this module only walks orders and stream
assignments and deduplicates by the first-use canonical form.  Under the
DESIGN.md R-Q13 DAG with two streams the space has 768 schedules.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import dspmv as D

V = D  # op-kind constants
VERTICES = list(range(10))
GPU = [D.DSPMV_OP_PACK, D.DSPMV_OP_SPMV_LOCAL, D.DSPMV_OP_UNPACK, D.DSPMV_OP_SPMV_REMOTE]
# SPEC.md S:125 + R-Q13 (same list as csrc/schedule.cpp kEdges)
EDGES = [(D.DSPMV_OP_START, D.DSPMV_OP_PACK), (D.DSPMV_OP_START, D.DSPMV_OP_SPMV_LOCAL),
         (D.DSPMV_OP_START, D.DSPMV_OP_POST_RECV), (D.DSPMV_OP_PACK, D.DSPMV_OP_POST_SEND),
         (D.DSPMV_OP_POST_SEND, D.DSPMV_OP_WAIT_SEND), (D.DSPMV_OP_POST_RECV, D.DSPMV_OP_WAIT_RECV),
         (D.DSPMV_OP_WAIT_RECV, D.DSPMV_OP_UNPACK), (D.DSPMV_OP_UNPACK, D.DSPMV_OP_SPMV_REMOTE),
         (D.DSPMV_OP_SPMV_LOCAL, D.DSPMV_OP_END), (D.DSPMV_OP_SPMV_REMOTE, D.DSPMV_OP_END),
         (D.DSPMV_OP_WAIT_SEND, D.DSPMV_OP_END),
         (D.DSPMV_OP_POST_SEND, D.DSPMV_OP_WAIT_RECV), (D.DSPMV_OP_POST_RECV, D.DSPMV_OP_WAIT_SEND)]


def topological_orders(edges=EDGES):
    pred = {v: {u for (u, w) in edges if w == v} for v in VERTICES}
    out, prefix, done = [], [], set()

    def rec():
        if len(prefix) == len(VERTICES):
            out.append(list(prefix))
            return
        for v in VERTICES:
            if v not in done and pred[v] <= done:
                prefix.append(v)
                done.add(v)
                rec()
                done.discard(v)
                prefix.pop()

    rec()
    return out


def canonical_key(ops) -> tuple:
    """First-use stream relabelling + sequential event ids."""
    smap, emap, key = {}, {}, []
    for k, s, e, _ in np.asarray(ops).tolist():
        if k in GPU or k in (D.DSPMV_OP_EVENT_RECORD, D.DSPMV_OP_STREAM_WAIT_EVENT):
            s = smap.setdefault(s, len(smap))
        else:
            s = 0
        if k == D.DSPMV_OP_EVENT_RECORD:
            e = emap.setdefault(e, len(emap))
        elif k in (D.DSPMV_OP_EVENT_SYNC, D.DSPMV_OP_STREAM_WAIT_EVENT):
            e = emap[e]
        else:
            e = 0
        key.append((k, s, e))
    return tuple(key)


def canonical_ops(ops) -> np.ndarray:
    """The representative of a schedule's bijection class: streams relabelled
    by first use (the first GPU op runs on stream 0, which can be the caller's
    stream) and events numbered in record order."""
    return np.array([(k, s, e, 0) for k, s, e in canonical_key(ops)], np.int32)


def enumerate_derived(n_streams: int = 2):
    """Every distinct schedule with derived syncs, as canonical ops arrays."""
    seen = {}
    for order in topological_orders():
        for assign in itertools.product(range(n_streams), repeat=len(GPU)):
            st = dict(zip(GPU, assign))
            ops = D.dspmv_schedule_derive(order, [st.get(v, 0) for v in order], n_streams)
            key = canonical_key(ops)
            if key not in seen:
                seen[key] = canonical_ops(ops)
    return list(seen.values())


def describe(ops) -> str:
    """Compact one-line description: vertices in order with streams."""
    parts = []
    for k, s, e, _ in np.asarray(ops).tolist():
        if k < 10:
            parts.append(D.VERTEX_NAMES[k] + (f"@s{s}" if k in GPU else ""))
        elif k == D.DSPMV_OP_EVENT_RECORD:
            parts.append(f"CER(s{s},e{e})")
        elif k == D.DSPMV_OP_EVENT_SYNC:
            parts.append(f"CES(e{e})")
        else:
            parts.append(f"CSWE(s{s},e{e})")
    return " ".join(parts)
