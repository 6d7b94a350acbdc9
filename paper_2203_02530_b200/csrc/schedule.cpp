// schedule.cpp -- schedule validation, tab:sync derivation, text format.
//
// A schedule is a traversal P of the program DAG G_P (PAPER.md P:239-248,
// P:289-292) whose GPU vertices are bound to streams (BoundGPU_s,
// tab:vertices P:250-264) and whose cross-resource dependencies are enforced
// by the synchronisation operations of tab:sync:
//   CPU -> *            : none (CPU vertices are synchronous)
//   GPU_i -> CPU        : cudaEventRecord -> cudaEventSynchronize
//   GPU_i -> GPU_i      : none (stream order)
//   GPU_i -> GPU_j      : cudaEventRecord -> cudaStreamWaitEvent
// The validator tracks happens-before with vector clocks: each stream s has
// VC[s][i] = number of items of stream i known complete before s's next item;
// the host has H[i]; an event snapshots its stream's clock at record time.
// Every enqueue on a stream inherits the host's knowledge (it is issued after
// everything the host has synchronised).  Edge u->v is enforced iff the
// consumer's clock covers u's position.
// Exchange vertices may be per destination (dspmv_op.peer = rank offset,
// P:281-284, DESIGN.md R-N4); build_dag derives the DAG of the granularity a
// schedule uses.
#include <algorithm>
#include <array>
#include <cstdio>
#include <sstream>

#include "internal.h"

namespace dspmv {

namespace {
constexpr int NV = 10;  // op kinds 0..9 are DAG vertex kinds

const char* kNames[NV] = {"start", "Pack", "y_L", "PostSend", "PostRecv",
                          "WaitSend", "WaitRecv", "Unpack", "y_R", "end"};

bool send_side(int k) { return k == DSPMV_OP_PACK || k == DSPMV_OP_POST_SEND || k == DSPMV_OP_WAIT_SEND; }
bool recv_side(int k) { return k == DSPMV_OP_POST_RECV || k == DSPMV_OP_WAIT_RECV || k == DSPMV_OP_UNPACK; }

using Clock = std::array<int32_t, DSPMV_MAX_STREAMS>;

inline void merge(Clock& a, const Clock& b) {
    for (int i = 0; i < DSPMV_MAX_STREAMS; ++i) a[i] = std::max(a[i], b[i]);
}

// Incremental happens-before state over a prefix of a schedule; DAG vertex
// instances are indexed by Dag ids.
struct HB {
    Clock host{};
    std::array<Clock, DSPMV_MAX_STREAMS> vc{};
    std::array<int32_t, DSPMV_MAX_STREAMS> len{};
    std::array<Clock, DSPMV_MAX_EVENTS> ev{};
    std::vector<int> stream_of;   // instance -> stream (GPU vertices)
    std::vector<int32_t> pos;     // instance -> position in its stream
    std::vector<bool> done;
    const Dag* dag;

    explicit HB(const Dag& d) : stream_of(d.v.size(), 0), pos(d.v.size(), 0), done(d.v.size(), false), dag(&d) {}
    void enqueue(int s) { merge(vc[s], host); }
    // would a DAG edge u->v be enforced if v (on stream sv, or CPU if sv<0) ran now?
    bool enforced(int u, int sv) const {
        if (!is_gpu_vertex(dag->v[u].kind)) return true;
        const int su = stream_of[u];
        if (sv < 0) return host[su] >= pos[u];
        if (sv == su) return true;
        Clock c = vc[sv];
        merge(c, host);
        return c[su] >= pos[u];
    }
    void vertex(int id, int stream) {
        if (is_gpu_vertex(dag->v[id].kind)) {
            enqueue(stream);
            pos[id] = ++len[stream];
            stream_of[id] = stream;
        }
        done[id] = true;
    }
    void sync(const dspmv_op& op) {
        const int k = op.kind;
        if (k == DSPMV_OP_EVENT_RECORD) {
            enqueue(op.stream);
            Clock c = vc[op.stream];
            c[op.stream] = len[op.stream];
            ev[op.event] = c;
        } else if (k == DSPMV_OP_EVENT_SYNC) {
            merge(host, ev[op.event]);
        } else if (k == DSPMV_OP_STREAM_WAIT_EVENT) {
            enqueue(op.stream);
            merge(vc[op.stream], ev[op.event]);
        }
    }
};
}  // namespace

bool is_dag_vertex(int kind) { return kind >= 0 && kind < NV; }
bool is_gpu_vertex(int kind) {
    return kind == DSPMV_OP_PACK || kind == DSPMV_OP_SPMV_LOCAL || kind == DSPMV_OP_UNPACK ||
           kind == DSPMV_OP_SPMV_REMOTE;
}
bool is_exchange_vertex(int kind) { return send_side(kind) || recv_side(kind); }
const char* vertex_name(int kind) { return is_dag_vertex(kind) ? kNames[kind] : "?"; }
std::string vertex_label(int kind, int peer) {
    std::string s = vertex_name(kind);
    if (peer) s += std::string("[") + (peer > 0 ? "+" : "") + std::to_string(peer) + "]";
    return s;
}

int Dag::find(int kind, int peer) const {
    for (size_t i = 0; i < v.size(); ++i)
        if (v[i].kind == kind && v[i].peer == peer) return int(i);
    return -1;
}

// The program DAG for the granularity of `present` (the DAG vertices a
// schedule names).  Coarse (every exchange vertex peer 0): SPEC S:125 +
// R-Q13.  Per destination (reading R-N4): the send-offset set S is
// the offsets of the send-side vertices and the negated offsets of the
// receive-side ones; each d in S contributes Pack/PostSend/WaitSend[d] and
// PostRecv/WaitRecv/Unpack[-d], with PostSend[d] -> WaitRecv[-d] and
// PostRecv[-d] -> WaitSend[d] as the deadlock edges.  Edges are emitted so
// that every vertex sees its predecessors in the oracle's order.
bool build_dag(const std::vector<DagVertex>& present, Dag& g, std::string& why) {
    g = Dag{};
    bool any_fine = false, any_coarse = false;
    std::vector<int> S;
    for (const DagVertex& x : present) {
        if (!is_dag_vertex(x.kind)) {
            why = "not a DAG vertex";
            return false;
        }
        if (!is_exchange_vertex(x.kind)) {
            if (x.peer != 0) {
                why = std::string(kNames[x.kind]) + " takes no peer offset";
                return false;
            }
            continue;
        }
        if (x.peer == 0) {
            any_coarse = true;
        } else {
            if (x.peer < -(1 << 20) || x.peer > (1 << 20)) {
                why = "peer offset out of range";
                return false;
            }
            any_fine = true;
            S.push_back(send_side(x.kind) ? x.peer : -x.peer);
        }
    }
    if (any_fine && any_coarse) {
        why = "mixed coarse and per-destination exchange vertices";
        return false;
    }
    g.fine = any_fine;
    if (!g.fine) S = {0};
    std::sort(S.begin(), S.end());
    S.erase(std::unique(S.begin(), S.end()), S.end());
    g.offsets = S;
    std::vector<int> R;
    for (int d : S) R.push_back(-d);
    std::sort(R.begin(), R.end());
    auto add = [&](int k, int d) {
        g.v.push_back({k, d});
        return int(g.v.size()) - 1;
    };
    const int vs = add(DSPMV_OP_START, 0);
    for (int d : S)
        for (int k : {DSPMV_OP_PACK, DSPMV_OP_POST_SEND, DSPMV_OP_WAIT_SEND}) add(k, d);
    const int vl = add(DSPMV_OP_SPMV_LOCAL, 0);
    for (int e : R)
        for (int k : {DSPMV_OP_POST_RECV, DSPMV_OP_WAIT_RECV, DSPMV_OP_UNPACK}) add(k, e);
    const int vr = add(DSPMV_OP_SPMV_REMOTE, 0), ve = add(DSPMV_OP_END, 0);
    auto E = [&](int u, int v, bool dead = false) { g.edges.push_back({u, v, dead ? 1 : 0}); };
    auto I = [&](int k, int d) { return g.find(k, d); };
    if (!g.fine) {
        // SPEC S:125 order (kept for the derived-sync order of the coarse space)
        E(vs, I(DSPMV_OP_PACK, 0));
        E(vs, vl);
        E(vs, I(DSPMV_OP_POST_RECV, 0));
        E(I(DSPMV_OP_PACK, 0), I(DSPMV_OP_POST_SEND, 0));
        E(I(DSPMV_OP_POST_SEND, 0), I(DSPMV_OP_WAIT_SEND, 0));
        E(I(DSPMV_OP_POST_RECV, 0), I(DSPMV_OP_WAIT_RECV, 0));
        E(I(DSPMV_OP_WAIT_RECV, 0), I(DSPMV_OP_UNPACK, 0));
        E(I(DSPMV_OP_UNPACK, 0), vr);
        E(vl, ve);
        E(vr, ve);
        E(I(DSPMV_OP_WAIT_SEND, 0), ve);
    } else {
        E(vs, vl);
        E(vl, ve);
        E(vr, ve);
        for (int d : S) {
            E(vs, I(DSPMV_OP_PACK, d));
            E(I(DSPMV_OP_PACK, d), I(DSPMV_OP_POST_SEND, d));
            E(I(DSPMV_OP_POST_SEND, d), I(DSPMV_OP_WAIT_SEND, d));
            E(I(DSPMV_OP_WAIT_SEND, d), ve);
        }
        for (int e : R) {
            E(vs, I(DSPMV_OP_POST_RECV, e));
            E(I(DSPMV_OP_POST_RECV, e), I(DSPMV_OP_WAIT_RECV, e));
            E(I(DSPMV_OP_WAIT_RECV, e), I(DSPMV_OP_UNPACK, e));
            E(I(DSPMV_OP_UNPACK, e), vr);
        }
    }
    // R-Q13 / R-N4: a Wait needs the peer's matching Post (SPMD)
    for (int e : R) E(I(DSPMV_OP_POST_SEND, -e), I(DSPMV_OP_WAIT_RECV, e), true);
    for (int d : S) E(I(DSPMV_OP_POST_RECV, -d), I(DSPMV_OP_WAIT_SEND, d), true);
    return true;
}

SchedCheck validate_schedule(const dspmv_op* ops, int n_ops, int n_streams) {
    SchedCheck r;
    auto bad = [&](dspmv_status st, const std::string& why) {
        r.st = st;
        r.why = why;
        return r;
    };
    if (!ops || n_ops <= 0) return bad(DSPMV_ERR_ARG, "empty schedule");
    if (n_ops > DSPMV_MAX_OPS) return bad(DSPMV_ERR_SCHEDULE, "too many ops");
    if (n_streams < 1 || n_streams > DSPMV_MAX_STREAMS) return bad(DSPMV_ERR_ARG, "n_streams out of range");
    std::array<bool, DSPMV_MAX_EVENTS> rec{};
    std::vector<DagVertex> present;
    for (int t = 0; t < n_ops; ++t) {
        const dspmv_op& o = ops[t];
        const std::string at = "op " + std::to_string(t) + ": ";
        if (is_dag_vertex(o.kind)) {
            if (is_gpu_vertex(o.kind) && (o.stream < 0 || o.stream >= n_streams))
                return bad(DSPMV_ERR_SCHEDULE, at + "stream out of range");
            for (const DagVertex& x : present)
                if (x.kind == o.kind && x.peer == o.peer)
                    return bad(DSPMV_ERR_SCHEDULE, at + "duplicate " + vertex_label(o.kind, o.peer));
            present.push_back({o.kind, o.peer});
        } else if (o.kind == DSPMV_OP_EVENT_RECORD || o.kind == DSPMV_OP_EVENT_SYNC ||
                   o.kind == DSPMV_OP_STREAM_WAIT_EVENT) {
            if (o.event < 0 || o.event >= DSPMV_MAX_EVENTS) return bad(DSPMV_ERR_SCHEDULE, at + "event id out of range");
            if (o.kind != DSPMV_OP_EVENT_SYNC && (o.stream < 0 || o.stream >= n_streams))
                return bad(DSPMV_ERR_SCHEDULE, at + "stream out of range");
            if (o.kind == DSPMV_OP_EVENT_RECORD) {
                if (rec[o.event]) return bad(DSPMV_ERR_SCHEDULE, at + "event recorded twice");
                rec[o.event] = true;
            } else if (!rec[o.event]) {
                return bad(DSPMV_ERR_SCHEDULE, at + "event used before it is recorded");
            }
        } else {
            return bad(DSPMV_ERR_SCHEDULE, at + "unknown op kind " + std::to_string(o.kind));
        }
    }
    std::string why;
    if (!build_dag(present, r.dag, why)) return bad(DSPMV_ERR_SCHEDULE, why);
    const Dag& g = r.dag;
    std::vector<int> where(g.v.size(), -1);
    r.inst.assign(n_ops, -1);
    for (int t = 0; t < n_ops; ++t) {
        if (!is_dag_vertex(ops[t].kind)) continue;
        const int id = g.find(ops[t].kind, ops[t].peer);
        where[id] = t;
        r.inst[t] = id;
    }
    for (size_t i = 0; i < g.v.size(); ++i)
        if (where[i] < 0) return bad(DSPMV_ERR_SCHEDULE, "missing vertex " + vertex_label(g.v[i].kind, g.v[i].peer));
    if (where[g.find(DSPMV_OP_START, 0)] != 0) return bad(DSPMV_ERR_SCHEDULE, "start is not the first op");
    if (where[g.find(DSPMV_OP_END, 0)] != n_ops - 1) return bad(DSPMV_ERR_SCHEDULE, "end is not the last op");
    for (const auto& e : g.edges) {
        if (where[e[0]] > where[e[1]])
            return bad(e[2] ? DSPMV_ERR_DEADLOCK : DSPMV_ERR_SCHEDULE,
                       vertex_label(g.v[e[1]].kind, g.v[e[1]].peer) + " before " +
                           vertex_label(g.v[e[0]].kind, g.v[e[0]].peer));
    }
    HB hb(g);
    for (int t = 0; t < n_ops; ++t) {
        const dspmv_op& o = ops[t];
        if (is_dag_vertex(o.kind)) {
            const int id = r.inst[t];
            const int sv = is_gpu_vertex(o.kind) ? o.stream : -1;
            for (const auto& e : g.edges) {
                if (e[1] != id) continue;
                if (!hb.enforced(e[0], sv))
                    return bad(DSPMV_ERR_SCHEDULE, "edge " + vertex_label(g.v[e[0]].kind, g.v[e[0]].peer) + "->" +
                                                       vertex_label(o.kind, o.peer) + " not synchronised (tab:sync)");
            }
            hb.vertex(id, o.stream);
        } else {
            hb.sync(o);
        }
    }
    return r;
}

}  // namespace dspmv

using namespace dspmv;

extern "C" dspmv_status dspmv_schedule_validate(const dspmv_op* ops, int n_ops, int n_streams) {
    SchedCheck c = validate_schedule(ops, n_ops, n_streams);
    if (c.st != DSPMV_OK) return fail(c.st, c.why);
    return DSPMV_OK;
}

extern "C" dspmv_status dspmv_schedule_dag(const int32_t* offsets, int n_offsets, int32_t* kinds, int32_t* peers,
                                          int cap_v, int* n_v, int32_t* edges, int cap_e, int* n_e) {
    if (!n_v || !n_e || n_offsets < 0 || (n_offsets > 0 && !offsets)) return fail(DSPMV_ERR_ARG, "bad argument");
    std::vector<DagVertex> present;
    for (int i = 0; i < n_offsets; ++i) {
        if (offsets[i] == 0) return fail(DSPMV_ERR_ARG, "offsets must be non-zero");
        present.push_back({DSPMV_OP_PACK, offsets[i]});
    }
    Dag g;
    std::string why;
    if (!build_dag(present, g, why)) return fail(DSPMV_ERR_ARG, why);
    *n_v = int(g.v.size());
    *n_e = int(g.edges.size());
    if ((kinds || peers) && cap_v < *n_v) return fail(DSPMV_ERR_ARG, "vertex capacity too small");
    if (edges && cap_e < *n_e) return fail(DSPMV_ERR_ARG, "edge capacity too small");
    for (int i = 0; i < *n_v; ++i) {
        if (kinds) kinds[i] = g.v[i].kind;
        if (peers) peers[i] = g.v[i].peer;
    }
    if (edges)
        for (int i = 0; i < *n_e; ++i)
            for (int j = 0; j < 3; ++j) edges[3 * i + j] = g.edges[i][j];
    return DSPMV_OK;
}

extern "C" dspmv_status dspmv_schedule_moves(const int32_t* offsets, int n_offsets, const dspmv_op* prefix,
                                            int n_prefix, int n_streams, dspmv_op* out, int cap, int* n_out) {
    if (!n_out || n_prefix < 0 || (n_prefix > 0 && !prefix) || n_offsets < 0 || (n_offsets > 0 && !offsets))
        return fail(DSPMV_ERR_ARG, "bad argument");
    if (n_streams < 1 || n_streams > DSPMV_MAX_STREAMS) return fail(DSPMV_ERR_ARG, "n_streams out of range");
    std::vector<dspmv_op> moves;
    auto emit = [&](const dspmv_op& m) {
        for (const dspmv_op& x : moves)
            if (x.kind == m.kind && x.stream == m.stream && x.event == m.event && x.peer == m.peer) return;
        moves.push_back(m);
    };
    if (n_prefix == 0) {
        emit({DSPMV_OP_START, 0, 0, 0});
    } else {
        std::vector<DagVertex> present;
        for (int i = 0; i < n_offsets; ++i) {
            if (offsets[i] == 0) return fail(DSPMV_ERR_ARG, "offsets must be non-zero");
            present.push_back({DSPMV_OP_PACK, offsets[i]});
        }
        Dag g;
        std::string why;
        if (!build_dag(present, g, why)) return fail(DSPMV_ERR_ARG, why);
        // replay the prefix
        HB hb(g);
        std::vector<int> where(g.v.size(), -1);
        std::vector<int> ev_stream(DSPMV_MAX_EVENTS, -1), ev_pos(DSPMV_MAX_EVENTS, -1), ev_order;
        int used = 0, n_ev = 0;
        for (int t = 0; t < n_prefix; ++t) {
            const dspmv_op& o = prefix[t];
            if (is_dag_vertex(o.kind)) {
                const int id = g.find(o.kind, o.peer);
                if (id < 0 || where[id] >= 0) return fail(DSPMV_ERR_ARG, "prefix vertex not in the DAG or repeated");
                if (is_gpu_vertex(o.kind) && (o.stream < 0 || o.stream >= n_streams))
                    return fail(DSPMV_ERR_ARG, "prefix stream out of range");
                where[id] = t;
                hb.vertex(id, o.stream);
                if (is_gpu_vertex(o.kind)) used = std::max(used, o.stream + 1);
            } else if (o.kind == DSPMV_OP_EVENT_RECORD || o.kind == DSPMV_OP_EVENT_SYNC ||
                       o.kind == DSPMV_OP_STREAM_WAIT_EVENT) {
                if (o.event < 0 || o.event >= DSPMV_MAX_EVENTS) return fail(DSPMV_ERR_ARG, "prefix event out of range");
                if (o.kind != DSPMV_OP_EVENT_SYNC) {
                    if (o.stream < 0 || o.stream >= n_streams) return fail(DSPMV_ERR_ARG, "prefix stream out of range");
                    used = std::max(used, o.stream + 1);
                }
                if (o.kind == DSPMV_OP_EVENT_RECORD) {
                    ev_stream[o.event] = o.stream;
                    ev_pos[o.event] = t;
                    ev_order.push_back(o.event);
                    ++n_ev;
                }
                hb.sync(o);
            } else {
                return fail(DSPMV_ERR_ARG, "bad prefix op");
            }
        }
        // frontier vertices x stream choices (first-use pruning); the move is the
        // vertex if every in-edge is enforced, else the next sync step of the
        // first unmet predecessor (DESIGN.md R-N5)
        for (size_t v = 0; v < g.v.size(); ++v) {
            if (hb.done[v]) continue;
            bool ready = true;
            for (const auto& e : g.edges)
                if (e[1] == int(v) && !hb.done[e[0]]) ready = false;
            if (!ready) continue;
            const int k = g.v[v].kind;
            const int ns = is_gpu_vertex(k) ? std::min(used + 1, n_streams) : 1;
            for (int sv = 0; sv < ns; ++sv) {
                const int s_v = is_gpu_vertex(k) ? sv : -1;
                int unmet = -1;
                for (const auto& e : g.edges)
                    if (e[1] == int(v) && !hb.enforced(e[0], s_v)) {
                        unmet = e[0];
                        break;
                    }
                if (unmet < 0) {
                    emit({k, s_v < 0 ? 0 : s_v, 0, g.v[v].peer});
                    continue;
                }
                const int su = hb.stream_of[unmet];
                int ev = -1;  // latest event recorded on su after u
                for (int q = int(ev_order.size()) - 1; q >= 0 && ev < 0; --q) {
                    const int e = ev_order[q];
                    if (ev_stream[e] == su && ev_pos[e] > where[unmet]) ev = e;
                }
                if (ev < 0) emit({DSPMV_OP_EVENT_RECORD, su, n_ev, 0});
                else if (s_v < 0) emit({DSPMV_OP_EVENT_SYNC, 0, ev, 0});
                else emit({DSPMV_OP_STREAM_WAIT_EVENT, s_v, ev, 0});
            }
        }
    }
    *n_out = int(moves.size());
    if (int(moves.size()) > cap) return fail(DSPMV_ERR_ARG, "output capacity too small");
    std::copy(moves.begin(), moves.end(), out);
    return DSPMV_OK;
}

extern "C" dspmv_status dspmv_schedule_derive_peers(const int32_t* order, const int32_t* streams,
                                                    const int32_t* peers, int n_vertices, int n_streams,
                                                    dspmv_op* out, int cap, int* n_out) {
    if (!order || !out || !n_out) return fail(DSPMV_ERR_ARG, "null argument");
    if (n_streams < 1 || n_streams > DSPMV_MAX_STREAMS) return fail(DSPMV_ERR_ARG, "n_streams out of range");
    if (n_vertices < NV || n_vertices > DSPMV_MAX_OPS) return fail(DSPMV_ERR_ARG, "n_vertices out of range");
    std::vector<DagVertex> present(n_vertices);
    for (int i = 0; i < n_vertices; ++i) {
        present[i] = {order[i], peers ? peers[i] : 0};
        if (!is_dag_vertex(order[i])) return fail(DSPMV_ERR_ARG, "order holds a non-vertex kind");
    }
    Dag g;
    std::string why;
    if (!build_dag(present, g, why)) return fail(DSPMV_ERR_ARG, why);
    if (int(g.v.size()) != n_vertices) return fail(DSPMV_ERR_ARG, "order is not a permutation of the DAG vertices");
    std::vector<bool> seen(g.v.size(), false);
    std::vector<dspmv_op> ops;
    HB hb(g);
    int ev = 0;
    for (int i = 0; i < n_vertices; ++i) {
        const int id = g.find(present[i].kind, present[i].peer);
        if (id < 0 || seen[id]) return fail(DSPMV_ERR_ARG, "order is not a permutation of the DAG vertices");
        seen[id] = true;
        const int v = present[i].kind;
        const int sv = is_gpu_vertex(v) ? (streams ? streams[i] : 0) : -1;
        if (is_gpu_vertex(v) && (sv < 0 || sv >= n_streams)) return fail(DSPMV_ERR_ARG, "stream out of range");
        for (const auto& e : g.edges) {
            if (e[1] != id) continue;
            const int u = e[0];
            if (!hb.done[u])
                return fail(DSPMV_ERR_ARG, "order not topological at " + vertex_label(v, present[i].peer));
            if (hb.enforced(u, sv)) continue;
            if (ev >= DSPMV_MAX_EVENTS) return fail(DSPMV_ERR_SCHEDULE, "too many events");
            dspmv_op rec{DSPMV_OP_EVENT_RECORD, hb.stream_of[u], ev, 0};
            dspmv_op wait = sv < 0 ? dspmv_op{DSPMV_OP_EVENT_SYNC, 0, ev, 0}
                                   : dspmv_op{DSPMV_OP_STREAM_WAIT_EVENT, sv, ev, 0};
            ops.push_back(rec);
            hb.sync(rec);
            ops.push_back(wait);
            hb.sync(wait);
            ++ev;
        }
        ops.push_back(dspmv_op{v, sv < 0 ? 0 : sv, 0, present[i].peer});
        hb.vertex(id, sv < 0 ? 0 : sv);
    }
    *n_out = int(ops.size());
    if (int(ops.size()) > cap) return fail(DSPMV_ERR_ARG, "output capacity too small");
    std::copy(ops.begin(), ops.end(), out);
    return DSPMV_OK;
}

extern "C" dspmv_status dspmv_schedule_derive(const int32_t* order, const int32_t* streams,
                                              int n_streams, dspmv_op* out, int cap, int* n_out) {
    if (order)
        for (int i = 0; i < NV; ++i)
            if (!is_dag_vertex(order[i])) return fail(DSPMV_ERR_ARG, "order is not a permutation of the 10 vertices");
    return dspmv_schedule_derive_peers(order, streams, nullptr, NV, n_streams, out, cap, n_out);
}

extern "C" dspmv_status dspmv_schedule_parse(const char* text, dspmv_op* out, int cap, int* n_out,
                                             int* n_streams) {
    if (!text || !out || !n_out) return fail(DSPMV_ERR_ARG, "null argument");
    std::istringstream in(text);
    std::string line;
    int n = 0, smax = 0, lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        const size_t h = line.find('#');
        if (h != std::string::npos) line = line.substr(0, h);
        std::istringstream ls(line);
        std::string name, kind, tok;
        if (!(ls >> name)) continue;
        if (!(ls >> kind)) return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": missing kind");
        int stream = -1, event = -1, peer = 0;
        while (ls >> tok) {
            if (tok.rfind("stream=", 0) == 0) stream = std::atoi(tok.c_str() + 7);
            else if (tok.rfind("event=", 0) == 0) event = std::atoi(tok.c_str() + 6);
            else if (tok.rfind("peer=", 0) == 0) peer = std::atoi(tok.c_str() + 5);
            else return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": bad token " + tok);
        }
        dspmv_op op{-1, 0, 0, 0};
        if (kind == "EventRecord") op = {DSPMV_OP_EVENT_RECORD, stream, event, 0};
        else if (kind == "EventSync") op = {DSPMV_OP_EVENT_SYNC, 0, event, 0};
        else if (kind == "StreamWaitEvent") op = {DSPMV_OP_STREAM_WAIT_EVENT, stream, event, 0};
        else if (kind == "Cpu" || kind == "BoundGpu" || kind == "PostSend" || kind == "PostRecv" ||
                 kind == "WaitSend" || kind == "WaitRecv") {
            std::string vname = name;
            const size_t br = vname.find('[');  // "Pack[+1]" = Pack with peer=+1
            if (br != std::string::npos && vname.back() == ']') {
                peer = std::atoi(vname.substr(br + 1, vname.size() - br - 2).c_str());
                vname = vname.substr(0, br);
            }
            for (int v = 0; v < NV; ++v)
                if (vname == kNames[v]) op.kind = v;
            if (op.kind < 0) return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": unknown vertex " + name);
            op.peer = peer;
            if ((kind == "BoundGpu") != is_gpu_vertex(op.kind))
                return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": kind does not match vertex");
            op.stream = is_gpu_vertex(op.kind) ? stream : 0;
        } else {
            return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": unknown kind " + kind);
        }
        if ((op.kind == DSPMV_OP_EVENT_RECORD || op.kind == DSPMV_OP_EVENT_SYNC ||
             op.kind == DSPMV_OP_STREAM_WAIT_EVENT) && event < 0)
            return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": missing event=");
        if ((op.kind == DSPMV_OP_EVENT_RECORD || op.kind == DSPMV_OP_STREAM_WAIT_EVENT ||
             is_gpu_vertex(op.kind)) && stream < 0)
            return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": missing stream=");
        if (op.stream + 1 > smax) smax = op.stream + 1;
        if (n < cap) out[n] = op;
        ++n;
    }
    *n_out = n;
    if (n_streams) *n_streams = std::max(1, smax);
    if (n > cap) return fail(DSPMV_ERR_ARG, "output capacity too small");
    return DSPMV_OK;
}

extern "C" dspmv_status dspmv_schedule_format(const dspmv_op* ops, int n_ops, char* buf, size_t cap) {
    if (!ops || !buf) return fail(DSPMV_ERR_ARG, "null argument");
    std::ostringstream os;
    for (int t = 0; t < n_ops; ++t) {
        const dspmv_op& o = ops[t];
        if (is_dag_vertex(o.kind)) {
            const std::string nm = vertex_label(o.kind, o.peer);
            if (is_gpu_vertex(o.kind)) os << nm << " BoundGpu stream=" << o.stream << "\n";
            else os << nm << " Cpu\n";
        } else if (o.kind == DSPMV_OP_EVENT_RECORD) {
            const char* prev = "start";
            std::string prev_l = prev;
            for (int q = t - 1; q >= 0; --q)
                if (is_dag_vertex(ops[q].kind)) { prev_l = vertex_label(ops[q].kind, ops[q].peer); break; }
            os << "CER-after-" << prev_l << " EventRecord stream=" << o.stream << " event=" << o.event << "\n";
        } else {
            const char* next = "end";
            std::string next_l = next;
            for (int q = t + 1; q < n_ops; ++q)
                if (is_dag_vertex(ops[q].kind)) { next_l = vertex_label(ops[q].kind, ops[q].peer); break; }
            if (o.kind == DSPMV_OP_EVENT_SYNC) os << "CES-b4-" << next_l << " EventSync event=" << o.event << "\n";
            else os << "CSWE-b4-" << next_l << " StreamWaitEvent stream=" << o.stream << " event=" << o.event << "\n";
        }
    }
    const std::string s = os.str();
    if (s.size() + 1 > cap) return fail(DSPMV_ERR_ARG, "buffer too small (" + std::to_string(s.size() + 1) + ")");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return DSPMV_OK;
}
