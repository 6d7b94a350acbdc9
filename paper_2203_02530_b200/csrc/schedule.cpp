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
#include <algorithm>
#include <array>
#include <cstdio>
#include <sstream>

#include "internal.h"

namespace dspmv {

namespace {
constexpr int NV = 10;  // DAG vertices = op kinds 0..9
// SPEC.md S:125 edge list + DESIGN.md R-Q13 (deadlock-freedom edges last)
const int kEdges[][2] = {
    {DSPMV_OP_START, DSPMV_OP_PACK},          {DSPMV_OP_START, DSPMV_OP_SPMV_LOCAL},
    {DSPMV_OP_START, DSPMV_OP_POST_RECV},     {DSPMV_OP_PACK, DSPMV_OP_POST_SEND},
    {DSPMV_OP_POST_SEND, DSPMV_OP_WAIT_SEND}, {DSPMV_OP_POST_RECV, DSPMV_OP_WAIT_RECV},
    {DSPMV_OP_WAIT_RECV, DSPMV_OP_UNPACK},    {DSPMV_OP_UNPACK, DSPMV_OP_SPMV_REMOTE},
    {DSPMV_OP_SPMV_LOCAL, DSPMV_OP_END},      {DSPMV_OP_SPMV_REMOTE, DSPMV_OP_END},
    {DSPMV_OP_WAIT_SEND, DSPMV_OP_END},
    {DSPMV_OP_POST_SEND, DSPMV_OP_WAIT_RECV}, {DSPMV_OP_POST_RECV, DSPMV_OP_WAIT_SEND}};
constexpr int kNumEdges = sizeof(kEdges) / sizeof(kEdges[0]);
constexpr int kFirstDeadlockEdge = 11;

const char* kNames[NV] = {"start", "Pack", "y_L", "PostSend", "PostRecv",
                          "WaitSend", "WaitRecv", "Unpack", "y_R", "end"};

using Clock = std::array<int32_t, DSPMV_MAX_STREAMS>;

inline void merge(Clock& a, const Clock& b) {
    for (int i = 0; i < DSPMV_MAX_STREAMS; ++i) a[i] = std::max(a[i], b[i]);
}

// Incremental happens-before state over a prefix of a schedule.
struct HB {
    Clock host{};
    std::array<Clock, DSPMV_MAX_STREAMS> vc{};
    std::array<int32_t, DSPMV_MAX_STREAMS> len{};
    std::array<Clock, DSPMV_MAX_EVENTS> ev{};
    std::array<bool, DSPMV_MAX_EVENTS> recorded{};
    std::array<int, NV> stream_of{};  // GPU vertex -> stream
    std::array<int32_t, NV> pos{};    // GPU vertex -> position in its stream
    std::array<bool, NV> done{};

    void enqueue(int s) { merge(vc[s], host); }
    // would a DAG edge u->v be enforced if v (on stream sv, or CPU if sv<0) ran now?
    bool enforced(int u, int sv) const {
        if (!is_gpu_vertex(u)) return true;
        const int su = stream_of[u];
        if (sv < 0) return host[su] >= pos[u];
        if (sv == su) return true;
        Clock c = vc[sv];
        merge(c, host);
        return c[su] >= pos[u];
    }
    void apply(const dspmv_op& op) {
        const int k = op.kind;
        if (k >= 0 && k < NV) {
            if (is_gpu_vertex(k)) {
                enqueue(op.stream);
                pos[k] = ++len[op.stream];
                stream_of[k] = op.stream;
            }
            done[k] = true;
        } else if (k == DSPMV_OP_EVENT_RECORD) {
            enqueue(op.stream);
            Clock c = vc[op.stream];
            c[op.stream] = len[op.stream];
            ev[op.event] = c;
            recorded[op.event] = true;
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
const char* vertex_name(int kind) { return is_dag_vertex(kind) ? kNames[kind] : "?"; }

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
    std::array<int, NV> where;
    where.fill(-1);
    std::array<bool, DSPMV_MAX_EVENTS> rec{};
    for (int t = 0; t < n_ops; ++t) {
        const dspmv_op& o = ops[t];
        const std::string at = "op " + std::to_string(t) + ": ";
        if (is_dag_vertex(o.kind)) {
            if (where[o.kind] >= 0) return bad(DSPMV_ERR_SCHEDULE, at + "duplicate " + kNames[o.kind]);
            where[o.kind] = t;
            if (is_gpu_vertex(o.kind) && (o.stream < 0 || o.stream >= n_streams))
                return bad(DSPMV_ERR_SCHEDULE, at + "stream out of range");
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
    for (int v = 0; v < NV; ++v)
        if (where[v] < 0) return bad(DSPMV_ERR_SCHEDULE, std::string("missing vertex ") + kNames[v]);
    if (where[DSPMV_OP_START] != 0) return bad(DSPMV_ERR_SCHEDULE, "start is not the first op");
    if (where[DSPMV_OP_END] != n_ops - 1) return bad(DSPMV_ERR_SCHEDULE, "end is not the last op");
    for (int e = 0; e < kNumEdges; ++e) {
        const int u = kEdges[e][0], v = kEdges[e][1];
        if (where[u] > where[v])
            return bad(e >= kFirstDeadlockEdge ? DSPMV_ERR_DEADLOCK : DSPMV_ERR_SCHEDULE,
                       std::string(kNames[v]) + " before " + kNames[u]);
    }
    HB hb;
    for (int t = 0; t < n_ops; ++t) {
        const dspmv_op& o = ops[t];
        if (is_dag_vertex(o.kind)) {
            const int sv = is_gpu_vertex(o.kind) ? o.stream : -1;
            for (int e = 0; e < kNumEdges; ++e) {
                if (kEdges[e][1] != o.kind) continue;
                if (!hb.enforced(kEdges[e][0], sv))
                    return bad(DSPMV_ERR_SCHEDULE, std::string("edge ") + kNames[kEdges[e][0]] + "->" +
                                                       kNames[o.kind] + " not synchronised (tab:sync)");
            }
        }
        hb.apply(o);
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

extern "C" dspmv_status dspmv_schedule_derive(const int32_t* order, const int32_t* streams,
                                              int n_streams, dspmv_op* out, int cap, int* n_out) {
    if (!order || !out || !n_out) return fail(DSPMV_ERR_ARG, "null argument");
    if (n_streams < 1 || n_streams > DSPMV_MAX_STREAMS) return fail(DSPMV_ERR_ARG, "n_streams out of range");
    std::vector<dspmv_op> ops;
    HB hb;
    int ev = 0;
    bool seen[NV] = {};
    for (int i = 0; i < NV; ++i) {
        const int v = order[i];
        if (!is_dag_vertex(v) || seen[v]) return fail(DSPMV_ERR_ARG, "order is not a permutation of the 10 vertices");
        seen[v] = true;
        const int sv = is_gpu_vertex(v) ? (streams ? streams[i] : 0) : -1;
        if (is_gpu_vertex(v) && (sv < 0 || sv >= n_streams)) return fail(DSPMV_ERR_ARG, "stream out of range");
        for (int e = 0; e < kNumEdges; ++e) {
            if (kEdges[e][1] != v) continue;
            const int u = kEdges[e][0];
            if (!hb.done[u]) return fail(DSPMV_ERR_ARG, std::string("order not topological at ") + kNames[v]);
            if (hb.enforced(u, sv)) continue;
            if (ev >= DSPMV_MAX_EVENTS) return fail(DSPMV_ERR_SCHEDULE, "too many events");
            dspmv_op rec{DSPMV_OP_EVENT_RECORD, hb.stream_of[u], ev, 0};
            dspmv_op wait = sv < 0 ? dspmv_op{DSPMV_OP_EVENT_SYNC, 0, ev, 0}
                                   : dspmv_op{DSPMV_OP_STREAM_WAIT_EVENT, sv, ev, 0};
            ops.push_back(rec);
            hb.apply(rec);
            ops.push_back(wait);
            hb.apply(wait);
            ++ev;
        }
        dspmv_op vop{v, sv < 0 ? 0 : sv, 0, 0};
        ops.push_back(vop);
        hb.apply(vop);
    }
    *n_out = int(ops.size());
    if (int(ops.size()) > cap) return fail(DSPMV_ERR_ARG, "output capacity too small");
    std::copy(ops.begin(), ops.end(), out);
    return DSPMV_OK;
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
        int stream = -1, event = -1;
        while (ls >> tok) {
            if (tok.rfind("stream=", 0) == 0) stream = std::atoi(tok.c_str() + 7);
            else if (tok.rfind("event=", 0) == 0) event = std::atoi(tok.c_str() + 6);
            else return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": bad token " + tok);
        }
        dspmv_op op{-1, 0, 0, 0};
        if (kind == "EventRecord") op = {DSPMV_OP_EVENT_RECORD, stream, event, 0};
        else if (kind == "EventSync") op = {DSPMV_OP_EVENT_SYNC, 0, event, 0};
        else if (kind == "StreamWaitEvent") op = {DSPMV_OP_STREAM_WAIT_EVENT, stream, event, 0};
        else if (kind == "Cpu" || kind == "BoundGpu" || kind == "PostSend" || kind == "PostRecv" ||
                 kind == "WaitSend" || kind == "WaitRecv") {
            for (int v = 0; v < NV; ++v)
                if (name == kNames[v]) op.kind = v;
            if (op.kind < 0) return fail(DSPMV_ERR_ARG, "line " + std::to_string(lineno) + ": unknown vertex " + name);
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
            if (is_gpu_vertex(o.kind)) os << kNames[o.kind] << " BoundGpu stream=" << o.stream << "\n";
            else os << kNames[o.kind] << " Cpu\n";
        } else if (o.kind == DSPMV_OP_EVENT_RECORD) {
            const char* prev = "start";
            for (int q = t - 1; q >= 0; --q)
                if (is_dag_vertex(ops[q].kind)) { prev = kNames[ops[q].kind]; break; }
            os << "CER-after-" << prev << " EventRecord stream=" << o.stream << " event=" << o.event << "\n";
        } else {
            const char* next = "end";
            for (int q = t + 1; q < n_ops; ++q)
                if (is_dag_vertex(ops[q].kind)) { next = kNames[ops[q].kind]; break; }
            if (o.kind == DSPMV_OP_EVENT_SYNC) os << "CES-b4-" << next << " EventSync event=" << o.event << "\n";
            else os << "CSWE-b4-" << next << " StreamWaitEvent stream=" << o.stream << " event=" << o.event << "\n";
        }
    }
    const std::string s = os.str();
    if (s.size() + 1 > cap) return fail(DSPMV_ERR_ARG, "buffer too small (" + std::to_string(s.size() + 1) + ")");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return DSPMV_OK;
}
