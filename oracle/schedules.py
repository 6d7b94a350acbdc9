"""The SpMV program DAG, tab:sync synchronisation insertion, a happens-before
validator, and a brute-force schedule enumerator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sources
-------
* DAG vertices / vertex types: PAPER.md §III-A ``tab:vertices`` P:250-264 and
  the SpMV description P:270-287 (Pack P:278, PostSends/PostRecvs P:279,
  start/end P:286-287).  Fig. 3c itself is a ``[FIGURE]`` placeholder, so the
  edge list is SPEC.md's inferred list plus, per the DESIGN.md reading
  R-Q13, PostSend->WaitRecv and PostRecv->WaitSend (every rank runs the same P,
  P:460, so a Wait before the matching Post on every rank can never finish).
* Synchronisation: PAPER.md ``tab:sync`` P:436-451 --
  CPU->*: none; GPU_i->CPU: cudaEventRecord -> cudaEventSynchronize;
  GPU_i->GPU_i: none; GPU_i->GPU_j: cudaEventRecord -> cudaStreamWaitEvent.
* Stream-bijection pruning: P:426-428 ("children that represent equivalent P_k
  under a stream bijection are pruned") -- first-use relabelling.
* Per-destination granularity (NEXT-3 (i)): P:281-284 -- "SpMV could have been
  implemented with a set of parallel independent vertices for each separate
  pack and MPI_Isend instead of collecting them into single Pack and PostSends
  vertices".  DESIGN.md reading R-N4: an SPMD schedule names a peer by its rank
  offset d (the exchange with rank r+d), written ``Pack[+1]``; the send side
  (Pack, PostSend, WaitSend) has one vertex per offset d in S, the receive
  side (PostRecv, WaitRecv, Unpack) one per offset in -S (rank r's send to
  r+d is received by rank r+d from offset -d).  The R-Q13 edges become
  PostSend[-e] -> WaitRecv[e] and PostRecv[-d] -> WaitSend[d].

A schedule here is a list of tuples:
  (name,)                    CPU vertex  (start, PostSend, PostRecv, WaitSend, WaitRecv, end)
  (name, stream)             GPU vertex  (Pack, y_L, Unpack, y_R) bound to a stream
                             (fine granularity: name = "Pack[+1]", "WaitRecv[-1]", ...)
  ("CER", stream, event)     cudaEventRecord on ``stream``
  ("CES", event)             cudaEventSynchronize (host blocks)
  ("CSWE", stream, event)    cudaStreamWaitEvent(stream, event)
"""
from __future__ import annotations

import itertools

VERTICES = ["start", "Pack", "y_L", "PostSend", "PostRecv", "WaitSend", "WaitRecv",
            "Unpack", "y_R", "end"]
GPU_VERTICES = {"Pack", "y_L", "Unpack", "y_R"}          # P:278, P:273 (GPU kernels)
CPU_VERTICES = set(VERTICES) - GPU_VERTICES               # MPI calls, start/end are CPU

# SPEC.md S:125 (Fig. 3c inferred)
EDGES_A = [("start", "Pack"), ("start", "y_L"), ("start", "PostRecv"),
           ("Pack", "PostSend"), ("PostSend", "WaitSend"), ("PostRecv", "WaitRecv"),
           ("WaitRecv", "Unpack"), ("Unpack", "y_R"),
           ("y_L", "end"), ("y_R", "end"), ("WaitSend", "end")]
# DESIGN.md reading R-Q13: SPMD deadlock-freedom edges
DEADLOCK_EDGES = [("PostSend", "WaitRecv"), ("PostRecv", "WaitSend")]
EDGES = EDGES_A + DEADLOCK_EDGES


SEND_SIDE = ("Pack", "PostSend", "WaitSend")
RECV_SIDE = ("PostRecv", "WaitRecv", "Unpack")


def vname(base: str, d: int) -> str:
    """Per-destination vertex name, e.g. vname("Pack", 1) == "Pack[+1]"."""
    return f"{base}[{d:+d}]"


def split_name(name: str):
    """("Pack[+1]" -> ("Pack", 1); "Pack" -> ("Pack", 0))."""
    if name.endswith("]") and "[" in name:
        b, d = name[:-1].split("[")
        return b, int(d)
    return name, 0


def base(name: str) -> str:
    return split_name(name)[0]


def fine_dag(S):
    """(vertices, edges, deadlock_edges) of the per-destination DAG for the
    send-offset set S (reading R-N4).  With S = {d} the DAG is the
    coarse one with every exchange vertex renamed."""
    S = sorted(set(int(d) for d in S))
    if not S or 0 in S:
        raise ValueError("offsets must be non-empty and non-zero")
    R = sorted(-d for d in S)
    V = (["start"] + [vname(b, d) for d in S for b in SEND_SIDE] + ["y_L"]
         + [vname(b, e) for e in R for b in RECV_SIDE] + ["y_R", "end"])
    E = [("start", "y_L"), ("y_L", "end"), ("y_R", "end")]
    for d in S:
        E += [("start", vname("Pack", d)), (vname("Pack", d), vname("PostSend", d)),
              (vname("PostSend", d), vname("WaitSend", d)), (vname("WaitSend", d), "end")]
    for e in R:
        E += [("start", vname("PostRecv", e)), (vname("PostRecv", e), vname("WaitRecv", e)),
              (vname("WaitRecv", e), vname("Unpack", e)), (vname("Unpack", e), "y_R")]
    # a Wait needs the peer's matching Post, and every rank runs the same P
    Dl = ([(vname("PostSend", -e), vname("WaitRecv", e)) for e in R]
          + [(vname("PostRecv", -d), vname("WaitSend", d)) for d in S])
    return V, E + Dl, Dl


def dag_of(ops):
    """The DAG a schedule is checked against: the coarse one unless its
    exchange vertices carry offsets; then fine_dag(S) with S = the send-side
    offsets and the negated receive-side offsets (a vertex missing from
    either side is reported by validate).  Raises ValueError on mixed
    granularity."""
    names = [op[0] for op in ops if base(op[0]) in VERTICES]
    fine = {n for n in names if split_name(n)[1] != 0}
    if not fine:
        return VERTICES, EDGES, DEADLOCK_EDGES
    if any(base(n) in SEND_SIDE + RECV_SIDE and split_name(n)[1] == 0 for n in names):
        raise ValueError("mixed coarse and per-destination exchange vertices")
    S = set()
    for n in fine:
        b, d = split_name(n)
        S.add(d if b in SEND_SIDE else -d)
    return fine_dag(S)


def preds(v, edges=EDGES):
    return [u for (u, w) in edges if w == v]


# ------------------------------------------------------------------ topology
def topological_orders(edges=EDGES, vertices=VERTICES):
    """All topological orders of the DAG (plain recursive enumeration)."""
    pred = {v: set(preds(v, edges)) for v in vertices}
    out = []

    def rec(prefix, done):
        if len(prefix) == len(vertices):
            out.append(list(prefix))
            return
        for v in vertices:  # declaration order
            if v not in done and pred[v] <= done:
                prefix.append(v)
                done.add(v)
                rec(prefix, done)
                done.remove(v)
                prefix.pop()

    rec([], set())
    return out


# ----------------------------------------------------------- happens-before
def _hb_graph(ops):
    """Nodes: ('H', t) host point after op t; ('C', t) CPU vertex; ('G', t) GPU
    op completion; ('R', e) event record; ('W', t) stream wait.  Returns
    (succ dict, node-of-op dict)."""
    succ = {}

    def edge(a, b):
        succ.setdefault(a, set()).add(b)
        succ.setdefault(b, set())

    prev_on_stream = {}
    rec = {}
    node_of = {}
    hprev = ("H", -1)
    succ[hprev] = set()
    for t, op in enumerate(ops):
        h = ("H", t)
        edge(hprev, h)
        name = base(op[0])
        if name in CPU_VERTICES:
            c = ("C", t)
            edge(hprev, c)
            edge(c, h)
            node_of[t] = c
        elif name in GPU_VERTICES:
            g = ("G", t)
            edge(hprev, g)
            s = op[1]
            if s in prev_on_stream:
                edge(prev_on_stream[s], g)
            prev_on_stream[s] = g
            node_of[t] = g
        elif name == "CER":
            _, s, e = op
            r = ("R", e)
            edge(hprev, r)
            if s in prev_on_stream:
                edge(prev_on_stream[s], r)
            prev_on_stream[s] = r
            rec[e] = r
            node_of[t] = r
        elif name == "CES":
            _, e = op
            if e in rec:
                edge(rec[e], h)
            node_of[t] = h
        elif name == "CSWE":
            _, s, e = op
            w = ("W", t)
            edge(hprev, w)
            if s in prev_on_stream:
                edge(prev_on_stream[s], w)
            if e in rec:
                edge(rec[e], w)
            prev_on_stream[s] = w
            node_of[t] = w
        else:
            raise ValueError(f"unknown op {op!r}")
        hprev = h
    return succ, node_of


def _reaches(succ, a, b):
    seen = {a}
    stack = [a]
    while stack:
        u = stack.pop()
        if u == b:
            return True
        for w in succ.get(u, ()):
            if w not in seen:
                seen.add(w)
                stack.append(w)
    return False


def edge_satisfied(ops, iu, iv):
    """DAG edge ops[iu] -> ops[iv] is enforced by host order, stream order and
    the inserted syncs (tab:sync P:444-448)."""
    succ, node_of = _hb_graph(ops)
    return _reaches(succ, node_of[iu], node_of[iv])


def validate(ops, n_streams, edges=None):
    """Return (True, '') or (False, 'schedule'|'deadlock', reason).  The DAG is
    ``dag_of(ops)`` (coarse or per-destination) unless ``edges`` is given."""
    try:
        vertices, dag_edges, dead = dag_of(ops)
    except ValueError as e:
        return (False, "schedule", str(e))
    if edges is None:
        edges = dag_edges
    pos = {}
    recorded = set()
    for t, op in enumerate(ops):
        name = op[0]
        if base(name) in VERTICES:
            if name not in vertices:
                return (False, "schedule", f"unknown vertex {name}")
            if name in pos:
                return (False, "schedule", f"duplicate vertex {name}")
            pos[name] = t
            if base(name) in GPU_VERTICES and not (0 <= op[1] < n_streams):
                return (False, "schedule", f"{name}: stream {op[1]} out of range")
        elif name == "CER":
            if not (0 <= op[1] < n_streams):
                return (False, "schedule", "CER stream out of range")
            if op[2] in recorded:
                return (False, "schedule", f"event {op[2]} recorded twice")
            recorded.add(op[2])
        elif name in ("CES", "CSWE"):
            e = op[-1]
            if e not in recorded:
                return (False, "schedule", f"event {e} used before record")
            if name == "CSWE" and not (0 <= op[1] < n_streams):
                return (False, "schedule", "CSWE stream out of range")
        else:
            return (False, "schedule", f"unknown op {name}")
    for v in vertices:
        if v not in pos:
            return (False, "schedule", f"missing vertex {v}")
    if pos["start"] != 0:
        return (False, "schedule", "start is not first")
    if pos["end"] != len(ops) - 1:
        return (False, "schedule", "end is not last")
    for (u, v) in edges:
        if pos[u] > pos[v]:
            kind = "deadlock" if (u, v) in dead else "schedule"
            return (False, kind, f"{v} before {u}")
    succ, node_of = _hb_graph(ops)
    for (u, v) in edges:
        if not _reaches(succ, node_of[pos[u]], node_of[pos[v]]):
            return (False, "schedule", f"edge {u}->{v} not synchronised")
    return (True, "", "")


# ------------------------------------------------------------ sync insertion
def derive(order, streams, edges=None):
    """Schedule from a vertex order and a {GPU vertex: stream} map, inserting
    syncs per tab:sync immediately before the vertex that needs them
    (already-satisfied edges insert nothing).  Events get
    sequential ids in emission order.  ``edges`` defaults to the DAG of the
    order's vertices (coarse or per-destination)."""
    if edges is None:
        edges = dag_of([(v,) for v in order])[1]
    ops = []
    ev = 0
    for v in order:
        vop = (v, streams[v]) if base(v) in GPU_VERTICES else (v,)
        for u in preds(v, edges):
            iu = next(t for t, op in enumerate(ops) if op[0] == u)
            trial = ops + [vop]
            if edge_satisfied(trial, iu, len(ops)):
                continue
            su = ops[iu][1]
            ops.append(("CER", su, ev))
            if base(v) in GPU_VERTICES:
                ops.append(("CSWE", streams[v], ev))
            else:
                ops.append(("CES", ev))
            ev += 1
        ops.append(vop)
    return ops


def canonical(ops):
    """First-use stream relabelling and sequential event ids."""
    smap, emap = {}, {}
    out = []
    for op in ops:
        name = op[0]
        if base(name) in GPU_VERTICES:
            s = smap.setdefault(op[1], len(smap))
            out.append((name, s))
        elif name == "CER":
            s = smap.setdefault(op[1], len(smap))
            e = emap.setdefault(op[2], len(emap))
            out.append(("CER", s, e))
        elif name == "CSWE":
            s = smap.setdefault(op[1], len(smap))
            out.append(("CSWE", s, emap[op[2]]))
        elif name == "CES":
            out.append(("CES", emap[op[1]]))
        else:
            out.append(op)
    return tuple(out)


def enumerate_derived(n_streams=2, edges=EDGES):
    """Brute force: every topological order x every stream assignment of the
    four GPU vertices, syncs derived, deduplicated by canonical form."""
    seen = {}
    gpus = [v for v in VERTICES if v in GPU_VERTICES]
    for order in topological_orders(edges):
        for assign in itertools.product(range(n_streams), repeat=len(gpus)):
            ops = derive(order, dict(zip(gpus, assign)), edges)
            key = canonical(ops)
            seen.setdefault(key, ops)
    return list(seen.values())


# ------------------------------------------------------ orderable syncs
def _sync_move(ops, u, iu, v_stream):
    """Next synchronisation step for an unmet edge u -> v (tab:sync): a
    cudaEventRecord on u's stream if no event recorded there after u yet,
    else the wait (CES for a CPU v, CSWE on v's stream for a GPU v) on the
    latest such event."""
    su = ops[iu][1]
    evs = [op[2] for t, op in enumerate(ops) if op[0] == "CER" and op[1] == su and t > iu]
    if not evs:
        n_ev = sum(1 for op in ops if op[0] == "CER")
        return ("CER", su, n_ev)
    return ("CES", evs[-1]) if v_stream is None else ("CSWE", v_stream, evs[-1])


def orderable_moves(ops, n_streams, edges=None, vertices=None):
    """Legal next ops of a prefix when synchronisation operations are moves
    of their own ("some prefixes may require synchronization
    operations before proceeding to the next vertex"; DESIGN.md R-N5, the
    "first-unmet" reading of SURVEY Appendix A).  For every frontier vertex v
    (all DAG predecessors in the prefix) and stream choice s (first-use
    bijection pruning): v itself if every edge u -> v is already
    enforced, else the next sync step of the first unmet predecessor."""
    if not ops:
        return [("start",)]
    if edges is None:                 # the coarse DAG unless given (a prefix may
        vertices, edges = VERTICES, EDGES   # not show its granularity yet)
    elif vertices is None:
        vertices = VERTICES
    done = {op[0] for op in ops if base(op[0]) in VERTICES}
    used = len({op[1] for op in ops
                if (base(op[0]) in GPU_VERTICES) or op[0] in ("CER", "CSWE")})
    moves = []
    for v in vertices:
        pv = preds(v, edges)
        if v in done or not all(u in done for u in pv):
            continue
        opts = range(min(used + 1, n_streams)) if base(v) in GPU_VERTICES else [None]
        for s in opts:
            vop = (v, s) if s is not None else (v,)
            m = vop
            for u in pv:
                iu = next(t for t, op in enumerate(ops) if op[0] == u)
                if not edge_satisfied(ops + [vop], iu, len(ops)):
                    m = _sync_move(ops, u, iu, s)
                    break
            if m not in moves:
                moves.append(m)
    return moves


def enumerate_orderable(n_streams=2, edges=EDGES):
    """Every distinct complete schedule reachable through orderable_moves,
    deduplicated by the canonical form (brute-force DFS)."""
    seen = {}

    def dfs(ops):
        if ops and ops[-1][0] == "end":
            seen.setdefault(canonical(ops), ops)
            return
        for m in orderable_moves(ops, n_streams, edges):
            dfs(ops + [m])

    dfs([])
    return list(seen.values())
