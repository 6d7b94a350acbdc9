"""O2 -- the simulated multi-rank distributed SpMV (§III-A).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the paper's problem statement step by step, in its order and notation:

1. ``partition`` -- "evenly divides contiguous rows of A, x, and y evenly across
   MPI ranks"; reading R-Q3 for n mod P != 0.
2. ``plan_rank`` -- "A_L has the column entries of A that correspond to x_L,
   the locally-held rows of x; A_R has the rest, corresponding to x_R"
   (P:273-275); "A is considered to be static, so the entries that make up x_R
   are fixed"; "each rank must copy a subset of its x_L entries into one
   buffer for each other rank (the Pack vertex)".  Readings R-Q4
   (halo ascending by global id), R-Q6 (compressed A_R rows), R-Q7 (pack map:
   destinations ascending, then ascending local index).
3. ``simulate`` -- executes one schedule's DAG vertices (coarse or
   per-destination) in lock-step over all
   ranks (op k on every rank before op k+1: a legal serialisation of the SPMD
   run), with MPI_Isend/Irecv/Wait semantics; sync ops
   are no-ops in this sequential semantics.  y_L and y_R are O1 loops; the
   accumulate is y_i = fl(y_L,i + y_R,i) on rows with remote entries (P:273
   "sum of"; reading R-Q9), y_i = y_L,i elsewhere.
"""
from __future__ import annotations

import numpy as np

from . import spmv as O1


def partition(n: int, P: int):
    """row_begin[r] = r*floor(n/P) + min(r, n mod P), r = 0..P."""
    q, rem = divmod(n, P)
    return [r * q + min(r, rem) for r in range(P + 1)]


def owner(j: int, row_begin) -> int:
    """Rank whose contiguous row block holds global index j."""
    for p in range(len(row_begin) - 1):
        if row_begin[p] <= j < row_begin[p + 1]:
            return p
    raise ValueError(j)


def plan_rank(rowptr_g, col_g, n: int, P: int, r: int):
    """Split rank r's rows into A_L / A_R and build its halo list.

    Returns a dict of int arrays (values are carried by index maps
    ``al_src`` / ``ar_src``: positions of each A_L / A_R entry in the global
    CSR, so the caller can gather any value array bit-exactly)."""
    rb = partition(n, P)
    b, e = rb[r], rb[r + 1]
    al_rowptr = [0]
    al_col, al_src = [], []
    ar_rows, ar_rowptr, ar_gcol, ar_src = [], [0], [], []
    remote = set()
    for i in range(b, e):
        had_remote = False
        for p in range(int(rowptr_g[i]), int(rowptr_g[i + 1])):
            j = int(col_g[p])
            if b <= j < e:                      # column of x_L: local
                al_col.append(j - b)
                al_src.append(p)
            else:                               # column of x_R: remote
                ar_gcol.append(j)
                ar_src.append(p)
                remote.add(j)
                had_remote = True
        al_rowptr.append(len(al_col))
        if had_remote:
            ar_rows.append(i - b)
            ar_rowptr.append(len(ar_gcol))
    halo = sorted(remote)                       # R-Q4: ascending global id
    hpos = {j: k for k, j in enumerate(halo)}
    ar_col = [hpos[j] for j in ar_gcol]
    recv_count = [0] * P
    for j in halo:
        recv_count[owner(j, rb)] += 1
    recv_displ = [0] * P
    for p in range(1, P):
        recv_displ[p] = recv_displ[p - 1] + recv_count[p - 1]
    I32 = np.int32
    return dict(row_begin=b, row_end=e,
                al_rowptr=np.array(al_rowptr, I32), al_col=np.array(al_col, I32),
                al_src=np.array(al_src, np.int64),
                ar_rows=np.array(ar_rows, I32), ar_rowptr=np.array(ar_rowptr, I32),
                ar_col=np.array(ar_col, I32), ar_src=np.array(ar_src, np.int64),
                halo_gid=np.array(halo, I32),
                recv_count=np.array(recv_count, I32), recv_displ=np.array(recv_displ, I32))


def plan_all(rowptr_g, col_g, n: int, P: int):
    """Plans of every rank, plus send lists / pack maps (R-Q7).

    send list p -> r = (H_r intersect [begin_p, end_p)) - begin_p; rank p's
    pack map is the concatenation over destinations r in ascending order."""
    plans = [plan_rank(rowptr_g, col_g, n, P, r) for r in range(P)]
    rb = partition(n, P)
    for p in range(P):
        send_count = [0] * P
        pack = []
        for r in range(P):
            lst = [int(j) - rb[p] for j in plans[r]["halo_gid"] if rb[p] <= j < rb[p + 1]]
            send_count[r] = len(lst)
            pack.extend(lst)
        send_displ = [0] * P
        for r in range(1, P):
            send_displ[r] = send_displ[r - 1] + send_count[r - 1]
        plans[p]["send_count"] = np.array(send_count, np.int32)
        plans[p]["send_displ"] = np.array(send_displ, np.int32)
        plans[p]["pack_map"] = np.array(pack, np.int32)
    return plans


class Deadlock(Exception):
    pass


def simulate(plans, val_g, x_g, ops):
    """Run one schedule (oracle.schedules tuple format) on every rank in
    lock-step and return the global y (fp64).  Raises Deadlock when a Wait
    finds its matching communication not posted by the peer.

    Exchange vertices are coarse (every peer) or per-destination (P:281-284,
    reading R-N4): ``Pack[+1]`` packs only the segment for rank r+1,
    ``PostRecv[-1]`` posts only the receive from rank r-1, and so on; a
    per-destination vertex whose peer r+d does not exist does nothing.  Halo
    entries no Unpack vertex wrote stay NaN."""
    from .schedules import split_name
    P = len(plans)
    val_g = np.asarray(val_g, np.float64)
    x_g = np.asarray(x_g, np.float64)
    st = []
    for pl in plans:
        b, e = pl["row_begin"], pl["row_end"]
        st.append(dict(x=x_g[b:e].copy(), sendbuf=np.full(len(pl["pack_map"]), np.nan),
                       recvbuf=np.full(len(pl["halo_gid"]), np.nan),
                       x_halo=np.full(len(pl["halo_gid"]), np.nan),
                       posted_send=[False] * P, posted_recv=[False] * P,
                       arrived=[False] * P, yL=None, yR=None, y=None))

    def deliver(p, r):
        cnt = int(plans[p]["send_count"][r])
        assert cnt == int(plans[r]["recv_count"][p])
        so = int(plans[p]["send_displ"][r])
        ro = int(plans[r]["recv_displ"][p])
        st[r]["recvbuf"][ro:ro + cnt] = st[p]["sendbuf"][so:so + cnt]
        st[r]["arrived"][p] = True

    def peers(r, d):
        """Ranks a vertex with offset d addresses on rank r (d = 0: all)."""
        if d == 0:
            return [q for q in range(P) if q != r]
        return [r + d] if 0 <= r + d < P else []

    for op in ops:
        name, d = split_name(op[0])
        for r in range(P):
            pl, s = plans[r], st[r]
            if name == "Pack":
                for q in peers(r, d):
                    a, c = int(pl["send_displ"][q]), int(pl["send_count"][q])
                    s["sendbuf"][a:a + c] = s["x"][pl["pack_map"][a:a + c]]
            elif name == "PostSend":
                for q in peers(r, d):
                    s["posted_send"][q] = True
                    if pl["send_count"][q] > 0 and st[q]["posted_recv"][r]:
                        deliver(r, q)
            elif name == "PostRecv":
                for p in peers(r, d):
                    s["posted_recv"][p] = True
                    if pl["recv_count"][p] > 0 and st[p]["posted_send"][r]:
                        deliver(p, r)
            elif name == "WaitRecv":
                for p in peers(r, d):
                    if pl["recv_count"][p] > 0 and not s["arrived"][p]:
                        raise Deadlock(f"rank {r} WaitRecv: nothing from {p}")
            elif name == "WaitSend":
                for q in peers(r, d):
                    if pl["send_count"][q] > 0 and not st[q]["arrived"][r]:
                        raise Deadlock(f"rank {r} WaitSend: {q} never received")
            elif name == "Unpack":
                for p in peers(r, d):
                    a, c = int(pl["recv_displ"][p]), int(pl["recv_count"][p])
                    s["x_halo"][a:a + c] = s["recvbuf"][a:a + c]
            elif name == "y_L":
                s["yL"] = O1.o1_spmv(pl["al_rowptr"].astype(np.int64), pl["al_col"],
                                     val_g[pl["al_src"]], s["x"])
            elif name == "y_R":
                s["yR"] = O1.o1_spmv(pl["ar_rowptr"].astype(np.int64), pl["ar_col"],
                                     val_g[pl["ar_src"]], s["x_halo"])
            elif name == "end":
                y = s["yL"].copy()
                for k, i in enumerate(pl["ar_rows"]):
                    y[i] = s["yL"][i] + s["yR"][k]
                s["y"] = y
    return np.concatenate([s["y"] for s in st]) if P else np.zeros(0)


def paper_sequence_1():
    """1-2-3-4-5-6-7-8-9-10 (start, Pack, y_L, PostSend, PostRecv,
    WaitSend, WaitRecv, Unpack, y_R, end) -- one stream, syncs derived."""
    return ["start", "Pack", "y_L", "PostSend", "PostRecv", "WaitSend", "WaitRecv",
            "Unpack", "y_R", "end"]


def paper_sequence_2():
    """1-5-3-2-4-7-6-8-9-10."""
    return ["start", "PostRecv", "y_L", "Pack", "PostSend", "WaitRecv", "WaitSend",
            "Unpack", "y_R", "end"]
