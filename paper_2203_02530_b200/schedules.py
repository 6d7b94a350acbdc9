"""Schedule-space enumeration for the design-space sweep (host logic).

The paper's design space is every traversal of the program DAG with every
stream assignment of its GPU vertices, synchronisation inserted per tab:sync
(§III-A/§III-C), streams pruned under
bijection.  Syncs are derived by the library
(``dspmv_schedule_derive_peers``); this module only walks orders and stream
assignments and deduplicates by the first-use canonical form.  Under the
DESIGN.md R-Q13 DAG with two streams the coarse space has 768 schedules.

A ``Space`` is the DAG of one granularity, taken from the library
(``dspmv_schedule_dag``): the coarse DAG, or the per-destination DAG of a set
of peer offsets (DESIGN.md R-N4) whose traversal space is far too
large to enumerate -- the MCTS (``mcts.py``) samples it instead.
"""
from __future__ import annotations

import itertools

import numpy as np

from . import dspmv as D

VERTICES = list(range(10))
GPU = [D.DSPMV_OP_PACK, D.DSPMV_OP_SPMV_LOCAL, D.DSPMV_OP_UNPACK, D.DSPMV_OP_SPMV_REMOTE]
SEND_SIDE = (D.DSPMV_OP_PACK, D.DSPMV_OP_POST_SEND, D.DSPMV_OP_WAIT_SEND)
RECV_SIDE = (D.DSPMV_OP_POST_RECV, D.DSPMV_OP_WAIT_RECV, D.DSPMV_OP_UNPACK)


class Space:
    """Vertices (kind, peer), edges and predecessor sets of one granularity."""

    def __init__(self, offsets=()):
        self.offsets = sorted(set(int(d) for d in offsets))
        self.vertices, edges = D.dspmv_schedule_dag(self.offsets)
        self.edges = [(u, v) for u, v, _ in edges]
        self.deadlock_edges = [(u, v) for u, v, dead in edges if dead]
        self.index = {vp: i for i, vp in enumerate(self.vertices)}
        self.pred = {i: set() for i in range(len(self.vertices))}
        for u, v in self.edges:
            self.pred[v].add(u)
        self.gpu = {i for i, (k, _) in enumerate(self.vertices) if k in GPU}
        self.names = [D.vertex_label(k, p) for k, p in self.vertices]

    @classmethod
    def of_ops(cls, ops):
        """The space a schedule belongs to (its peer offsets)."""
        offs = set()
        for k, _, _, p in np.asarray(ops).tolist():
            if p and k in SEND_SIDE:
                offs.add(p)
            elif p and k in RECV_SIDE:
                offs.add(-p)
        return cls(sorted(offs))

    def derive(self, order, streams, n_streams: int) -> np.ndarray:
        """ops of a traversal (vertex indices) with a stream per vertex."""
        kinds = [self.vertices[i][0] for i in order]
        peers = [self.vertices[i][1] for i in order]
        return D.dspmv_schedule_derive_peers(kinds, streams, peers, n_streams)

    def topological_orders(self):
        out, prefix, done = [], [], set()
        n = len(self.vertices)

        def rec():
            if len(prefix) == n:
                out.append(list(prefix))
                return
            for v in range(n):
                if v not in done and self.pred[v] <= done:
                    prefix.append(v)
                    done.add(v)
                    rec()
                    done.discard(v)
                    prefix.pop()

        rec()
        return out


COARSE = Space()
# SPEC.md S:125 + R-Q13 as (kind, kind) pairs (same list as csrc/schedule.cpp)
EDGES = [(COARSE.vertices[u][0], COARSE.vertices[v][0]) for u, v in COARSE.edges]


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
    for k, s, e, p in np.asarray(ops).tolist():
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
        key.append((k, s, e, p if k < 10 else 0))
    return tuple(key)


def canonical_ops(ops) -> np.ndarray:
    """The representative of a schedule's bijection class: streams relabelled
    by first use (the first GPU op runs on stream 0, which can be the caller's
    stream) and events numbered in record order."""
    return np.array(canonical_key(ops), np.int32).reshape(-1, 4)


def enumerate_derived(n_streams: int = 2, space: Space = COARSE):
    """Every distinct schedule with derived syncs, as canonical ops arrays."""
    seen = {}
    gpu = sorted(space.gpu)
    for order in space.topological_orders():
        for assign in itertools.product(range(n_streams), repeat=len(gpu)):
            st = dict(zip(gpu, assign))
            ops = space.derive(order, [st.get(v, 0) for v in order], n_streams)
            key = canonical_key(ops)
            if key not in seen:
                seen[key] = canonical_ops(ops)
    return list(seen.values())


def enumerate_orderable(n_streams: int = 2, space: Space = COARSE):
    """Every distinct schedule when synchronisation operations are moves of
    their own (DESIGN.md R-N5; ``dspmv_schedule_moves``), as
    canonical ops arrays.  Coarse DAG, two streams: 4,780 schedules."""
    seen = {}

    def dfs(prefix):
        if prefix and prefix[-1][0] == D.DSPMV_OP_END:
            key = canonical_key(prefix)
            if key not in seen:
                seen[key] = canonical_ops(prefix)
            return
        for m in D.dspmv_schedule_moves(prefix, n_streams, space.offsets).tolist():
            dfs(prefix + [tuple(m)])

    dfs([])
    return list(seen.values())


def describe(ops) -> str:
    """Compact one-line description: vertices in order with streams."""
    parts = []
    for k, s, e, p in np.asarray(ops).tolist():
        if k < 10:
            parts.append(D.vertex_label(k, p) + (f"@s{s}" if k in GPU else ""))
        elif k == D.DSPMV_OP_EVENT_RECORD:
            parts.append(f"CER(s{s},e{e})")
        elif k == D.DSPMV_OP_EVENT_SYNC:
            parts.append(f"CES(e{e})")
        else:
            parts.append(f"CSWE(s{s},e{e})")
    return " ".join(parts)
