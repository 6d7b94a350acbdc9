// api.cpp -- the C ABI (include/dspmv.h): communicators, plans, schedules,
// the schedule executor and the NCCL / in-process halo exchange.
//
// Executor semantics (§III-A/§III-C): a schedule is walked op by op
// on the host.  GPU vertices are asynchronous launches on their
// bound stream; CPU vertices run synchronously; CER/CES/CSWE are
// cudaEventRecord / cudaEventSynchronize / cudaStreamWaitEvent (tab:sync,
// P:444-448).  PostSend / PostRecv set host flags; the later of the two
// issues ONE NCCL group (ncclRecv from every owner, ncclSend to every
// requester) on the high-priority comm stream -- NCCL requires sends and
// receives that must progress together to be in one group (DESIGN.md R-Q16).
// WaitSend / WaitRecv synchronise on the group's completion event while
// polling ncclCommGetAsyncError.  END returns (all GPU work was
// already host-synchronised by the schedule's own CES ops, R-Q17).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <thread>

#include "runtime.h"

namespace dspmv {

static thread_local std::string t_err;

void set_error(const std::string& msg) { t_err = msg; }
dspmv_status fail(dspmv_status st, const std::string& msg) {
    t_err = msg;
    return st;
}

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return fail(DSPMV_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)
// inside ncclGroupStart/End: record the first error, keep going, end the group
#define NCCL_GROUP_CALL(res, expr)                          \
    do {                                                    \
        ncclResult_t _r = (expr);                           \
        if (_r != ncclSuccess && (res) == ncclSuccess) (res) = _r; \
    } while (0)
#define NCCL_TRY(expr)                                                                         \
    do {                                                                                       \
        ncclResult_t _r = (expr);                                                              \
        if (_r != ncclSuccess)                                                                 \
            return fail(DSPMV_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));   \
    } while (0)

int device_sm_count();
int prof_read(unsigned long long* out, int n, bool reset);

namespace {

#define ST_TRY(expr)                       \
    do {                                   \
        dspmv_status _s = (expr);          \
        if (_s != DSPMV_OK) return _s;     \
    } while (0)

ncclDataType_t nccl_type(int dtype) { return dtype == DSPMV_F32 ? ncclFloat32 : ncclFloat64; }

// Device memory of a plan: the caller's allocator (opts.alloc, e.g. torch's
// caching allocator) unless `ipc` (buffers peers map through CUDA IPC need
// their own cudaMalloc allocation) or no allocator was given.
dspmv_status raw_alloc(Plan& p, void** dst, size_t bytes, bool ipc) {
    *dst = nullptr;
    const bool cb = !ipc && p.opts.alloc && p.opts.free;
    if (cb) {
        *dst = p.opts.alloc(bytes, p.device, p.opts.alloc_ctx);
        if (!*dst) return fail(DSPMV_ERR_OOM, "allocator callback returned NULL for " + std::to_string(bytes) + " bytes");
    } else if (cudaMalloc(dst, bytes) != cudaSuccess) {
        cudaGetLastError();
        *dst = nullptr;
        return fail(DSPMV_ERR_OOM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    }
    p.allocs.push_back({*dst, bytes, cb});
    p.device_bytes += int64_t(bytes);
    return DSPMV_OK;
}

template <typename T>
dspmv_status dev_upload(Plan& p, T** dst, const T* src, size_t n) {
    *dst = nullptr;
    if (n == 0) return DSPMV_OK;
    void* d = nullptr;
    ST_TRY(raw_alloc(p, &d, n * sizeof(T), false));
    if (src) CUDA_TRY(cudaMemcpy(d, src, n * sizeof(T), cudaMemcpyHostToDevice));
    *dst = static_cast<T*>(d);
    return DSPMV_OK;
}

dspmv_status dev_alloc(Plan& p, void** dst, size_t bytes, bool zero, bool ipc = false) {
    *dst = nullptr;
    if (bytes == 0) return DSPMV_OK;
    ST_TRY(raw_alloc(p, dst, bytes, ipc));
    if (zero) {
        // cudaMemset runs on the legacy stream, which does not order the
        // library's non-blocking streams (nor peers writing over IPC): wait
        // for it, or a flag written later could be zeroed after the fact
        CUDA_TRY(cudaMemset(*dst, 0, bytes));
        CUDA_TRY(cudaDeviceSynchronize());
    }
    return DSPMV_OK;
}

// Scratch device buffer freed on every exit path.
struct DevScratch {
    void* p = nullptr;
    ~DevScratch() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};


static bool stream_tma_default();

dspmv_status upload_layout(Plan& p, const Layout& L, int cfg, DevLayout& D) {
    D = DevLayout();
    D.nS = L.nS;
    D.nb = L.nb;
    D.nV = L.nV;
    const int sms = device_sm_count();
    if (L.nb > 0) {
        if (!L.sell) {   // the sliced form keeps its own copy of the S entries
            ST_TRY(dev_upload(p, &D.s_rowptr, L.s_rowptr.data(), L.s_rowptr.size()));
            ST_TRY(dev_upload(p, &D.s_col, L.s_col.data(), L.s_col.size()));
            ST_TRY(dev_upload(p, reinterpret_cast<uint8_t**>(&D.s_val), L.s_val.data(), L.s_val.size()));
            ST_TRY(dev_upload(p, &D.s_desc, L.s_desc.data(), L.s_desc.size()));
        }
        if (L.s_has_slot) ST_TRY(dev_upload(p, &D.s_slot, L.s_slot.data(), L.s_slot.size()));
        if (!L.s_identity) ST_TRY(dev_upload(p, &D.s_out, L.s_out.data(), L.s_out.size()));
        D.cfg = cfg;
        if (const char* ev = std::getenv("DSPMV_L2PF")) D.l2pf = std::atoi(ev);   // sweeps (< 0: evict_first hint)
        if (const char* ev = std::getenv("DSPMV_ST_L2PF")) D.st_l2pf = std::atoi(ev);   // sweeps (< 0: col only)
        const int per_sm = block_kernel_ctas_per_sm(p.dtype, cfg);
        // optionally leave SMs free for concurrent NCCL / pack kernels
        const int reserve = p.opts.reserve_sms >= 0 ? p.opts.reserve_sms : (p.comm->nranks > 1 ? kAutoReserveSms : 0);
        const int usable = std::max(1, sms - reserve);
        D.grid_s = std::max(1, std::min(L.nb, per_sm * usable));
        if (L.sell) {
            D.stream = true;
            D.sell = true;
            D.nslices = int32_t(L.sl_base.size()) - 1;
            D.nchunks = int32_t(L.sl_chunk.size()) - 1;
            ST_TRY(dev_upload(p, &D.sl_chunk, L.sl_chunk.data(), L.sl_chunk.size()));
            ST_TRY(dev_upload(p, &D.sl_base, L.sl_base.data(), L.sl_base.size()));
            ST_TRY(dev_upload(p, &D.sl_srow, L.sl_srow.data(), L.sl_srow.size()));
            ST_TRY(dev_upload(p, &D.sl_len, L.sl_len.data(), L.sl_len.size()));
            ST_TRY(dev_upload(p, &D.sl_col, L.sl_col.data(), L.sl_col.size()));
            ST_TRY(dev_upload(p, reinterpret_cast<uint8_t**>(&D.sl_val), L.sl_val.data(), L.sl_val.size()));
            D.sell_unroll = sell_unroll();
            D.st_dynamic = kStreamDynamic;
            if (const char* ev = std::getenv("DSPMV_ST_DYNAMIC")) D.st_dynamic = std::atoi(ev) != 0;   // A/B
            if (D.st_dynamic) ST_TRY(dev_alloc(p, reinterpret_cast<void**>(&D.d_work), 2 * sizeof(unsigned), true));
            if (const char* ev = std::getenv("DSPMV_SELL_L1")) D.sell_l1 = std::atoi(ev) != 0;
            set_x_persist_limit();
            int spsm = sell_kernel_ctas_per_sm(p.dtype, D.sell_unroll);
            if (const char* ev = std::getenv("DSPMV_SELL_CTAS")) spsm = std::max(1, std::min(spsm, std::atoi(ev)));  // sweeps
            D.grid_sl = std::max(1, std::min((D.nchunks + kSellCtaWarps - 1) / kSellCtaWarps, spsm * usable));
        } else if (L.stream) {
            D.stream = true;
            set_x_persist_limit();
            D.ntiles = int32_t(L.s_tiles.size() / 2);
            ST_TRY(dev_upload(p, &D.s_tiles, L.s_tiles.data(), L.s_tiles.size()));
            D.st_dynamic = kStreamDynamic;
            if (const char* ev = std::getenv("DSPMV_ST_DYNAMIC")) D.st_dynamic = std::atoi(ev) != 0;   // A/B
            if (const char* ev = std::getenv("DSPMV_ST_GRAB")) D.st_grab = std::max(1, std::atoi(ev));   // sweeps
            if (D.st_dynamic) ST_TRY(dev_alloc(p, reinterpret_cast<void**>(&D.d_work), 2 * sizeof(unsigned), true));
            int tpsm = stream_kernel_ctas_per_sm(p.dtype);
            if (const char* ev = std::getenv("DSPMV_STREAM_CTAS")) tpsm = std::max(1, std::min(tpsm, std::atoi(ev)));  // sweeps
            D.grid_t = std::max(1, std::min((D.ntiles + kStreamCtaWarps - 1) / kStreamCtaWarps, tpsm * usable));
            if (p.opts.s_kernel == DSPMV_SKERNEL_STREAM_TMA ||
                (p.opts.s_kernel == DSPMV_SKERNEL_AUTO && stream_tma_default())) {
                D.stream_tma = true;
                D.ntblocks = int32_t(L.s_tdesc.size() / kDescInts);
                ST_TRY(dev_upload(p, &D.s_tdesc, L.s_tdesc.data(), L.s_tdesc.size()));
                D.st_variant = stream_tma_variant();
                const int bpsm = stream_tma_kernel_ctas_per_sm(p.dtype, D.st_variant);
                D.grid_tt = std::max(1, std::min(D.ntblocks, bpsm * usable));
            }
        }
    }
    if (L.nV > 0) {
        ST_TRY(dev_upload(p, &D.v_rowptr, L.v_rowptr.data(), L.v_rowptr.size()));
        ST_TRY(dev_upload(p, &D.v_col, L.v_col.data(), L.v_col.size()));
        ST_TRY(dev_upload(p, reinterpret_cast<uint8_t**>(&D.v_val), L.v_val.data(), L.v_val.size()));
        ST_TRY(dev_upload(p, &D.v_out, L.v_out.data(), L.v_out.size()));
        if (L.v_has_slot) ST_TRY(dev_upload(p, &D.v_slot, L.v_slot.data(), L.v_slot.size()));
        D.grid_v = int(std::min<int64_t>((int64_t(L.nV) + 7) / 8, int64_t(sms) * 8));
        D.v_ordered = p.opts.long_row_sum == DSPMV_LONG_ROW_STORED;
    }
    D.combine = L.s_has_slot || L.v_has_slot;
    return DSPMV_OK;
}

// Irregular matrices: the TMA-producer CSR-stream variant by default
// (DSPMV_STREAM_TMA=0/1 overrides, for sweeps)
static bool stream_tma_default() {
    static const int v = [] {
        const char* ev = std::getenv("DSPMV_STREAM_TMA");
        return ev ? std::atoi(ev) : 0;
    }();
    return v != 0;
}

// S-group kernel of a matrix: forced by opts.s_kernel, else the row-block
// kernel when a block configuration is forced, else chosen by row lengths.
bool use_stream(const dspmv_plan_opts& o, const int32_t* rowptr, int32_t nrows, int vthr) {
    if (o.s_kernel == DSPMV_SKERNEL_STREAM || o.s_kernel == DSPMV_SKERNEL_STREAM_TMA ||
        o.s_kernel == DSPMV_SKERNEL_SELL)
        return true;
    if (o.s_kernel == DSPMV_SKERNEL_BLOCK || o.block_cfg >= 0) return false;
    if (const char* ev = std::getenv("DSPMV_SKERNEL")) return std::atoi(ev) == DSPMV_SKERNEL_STREAM;  // sweeps
    return auto_stream(rowptr, nrows, vthr);
}

// The sliced form for a CSR-stream S group: forced by opts.s_kernel, else
// DSPMV_SELL (sweeps), else the default for irregular matrices.
bool use_sell(const dspmv_plan_opts& o, bool stream) {
    if (!stream || o.s_kernel == DSPMV_SKERNEL_STREAM || o.s_kernel == DSPMV_SKERNEL_STREAM_TMA) return false;
    if (o.s_kernel == DSPMV_SKERNEL_SELL) return true;
    static const int v = [] {
        const char* ev = std::getenv("DSPMV_SELL");
        return ev ? std::atoi(ev) : 0;
    }();
    return v != 0;
}

// Streamed host input of dspmv_apply_host (plan time, host only).  x is cut
// into K chunks; y_L's row blocks are grouped so that group k reads x chunks
// <= k only (prefix max of each block's highest column chunk).
void build_host_pipe(Plan& p, Layout& L) {
    auto& H = p.pipe;
    H.K = 0;
    const int64_t n = p.host.n_local();
    const int64_t bytes = n * p.esize;
    if (L.nb < 2 || bytes < (int64_t(2) << 20)) return;   // small: one transfer is as good
    // ~4 MiB chunks, at most 16: measured best on C2 (16.8 MB of x: K = 1 / 2 / 4 / 8
    // / 12 -> 0.647 / 0.527 / 0.487 / 0.510 / 0.560 ms per apply_host) and on C3
    // (134 MB: K = 4 / 8 / 16 / 32 -> 3.98 / 3.67 / 3.60 / 3.72 ms,
    // profiles/r2_e2e_chunks_c3.txt): each chunk boundary costs a copy-engine
    // drain, the last chunk's rows trail the copy
    int K = int(std::max<int64_t>(2, std::min<int64_t>(16, bytes / (int64_t(4) << 20))));
    if (const char* ev = std::getenv("DSPMV_HOST_CHUNKS"))   // tuning
        K = int(std::min<int64_t>(std::max(1, std::min(64, std::atoi(ev))), bytes / (int64_t(1) << 20)));
    std::vector<double> frac;   // chunk end fractions (uniform by default)
    for (int k = 1; k < K; ++k) frac.push_back(double(k) / K);
    if (const char* ev = std::getenv("DSPMV_HOST_SPLIT")) {  // tuning: "0.4,0.7,0.9"
        frac.clear();
        for (const char* q = ev; *q;) {
            char* e = nullptr;
            const double f = std::strtod(q, &e);
            if (e == q) break;
            if (f > 0 && f < 1 && (frac.empty() || f > frac.back())) frac.push_back(f);
            q = *e == ',' ? e + 1 : e;
        }
        K = int(frac.size()) + 1;
    }
    H.x_chunk.assign(K + 1, 0);
    for (int k = 1; k < K; ++k)
        H.x_chunk[k] = std::min<int64_t>(n, (int64_t(frac[k - 1] * double(n)) + 255) / 256 * 256);
    H.x_chunk[K] = n;
    auto chunk_of = [&](int64_t c) {
        return int(std::upper_bound(H.x_chunk.begin(), H.x_chunk.end(), c) - H.x_chunk.begin()) - 1;
    };
    H.grp.assign(K + 1, L.nb);
    H.grp[0] = 0;
    int pm = 0;
    for (int32_t b = 0; b < L.nb; ++b) {
        const int32_t* d = L.s_desc.data() + size_t(b) * kDescInts;
        int32_t cmax = 0;
        for (int32_t q = d[2]; q < d[3]; ++q) cmax = std::max(cmax, L.s_col[q]);
        pm = std::max(pm, d[3] > d[2] ? chunk_of(cmax) : 0);
        for (int k = 0; k < pm; ++k) H.grp[k + 1] = std::min(H.grp[k + 1], b);
        L.s_desc[size_t(b) * kDescInts + 15] = pm;
    }
    H.K = K;
    // y by copy engine: only where each group's blocks cover a contiguous,
    // increasing run of rows that no other kernel writes (one rank, S rows in
    // matrix order, no warp-per-row rows, no combined rows)
    H.ycopy = false;
    if (p.host.nranks == 1 && L.nV == 0 && L.s_identity && !L.stream && !L.s_has_slot) {
        H.yrow.assign(size_t(K) + 1, 0);
        H.nblk.assign(size_t(K), 0);
        bool ok = true;
        int32_t prev = -1;
        for (int32_t b = 0; b < L.nb && ok; ++b) {
            const int32_t* d = L.s_desc.data() + size_t(b) * kDescInts;
            const int g = d[15];
            ok = g >= prev;   // groups in block order
            if (g != prev) {
                for (int k = prev + 1; k <= g; ++k) H.yrow[k] = d[0];
                prev = g;
            }
            H.nblk[g]++;
        }
        for (int k = prev + 1; k <= K; ++k) H.yrow[k] = L.nS;
        // measured (profiles/r2_e2e_ycopy.txt): C3 (134 MB of y) 3.46-3.79 ms vs
        // 3.77-3.85 ms zero-copy; C2 (16.8 MB) 0.60 vs 0.54 ms -- copy engine
        // for large y only
        H.ycopy = ok && L.nS == n && bytes >= (int64_t(64) << 20);
        if (const char* ev = std::getenv("DSPMV_HOST_YCOPY")) H.ycopy = H.ycopy && std::atoi(ev) != 0;  // A/B
    }
}

// Phase 2 on the device side: pack map + send buffer.
dspmv_status finalize_send(Plan& p) {
    p.has_peers = false;
    for (int q = 0; q < p.host.nranks; ++q)
        p.has_peers |= (p.host.recv_count[q] > 0 || p.host.send_count[q] > 0);
    const size_t s = p.host.pack_map.size();
    // DSPMV_PACK_ALIAS_IF_CONTIGUOUS: every destination's
    // send list a run of consecutive local rows -> send from x, no Pack kernel
    p.pack_alias = p.opts.pack_mode == DSPMV_PACK_ALIAS_IF_CONTIGUOUS && !p.put_mode && s > 0 &&
                   pack_alias_offsets(p.host, p.alias_off);
    ST_TRY(dev_upload(p, &p.d_pack_map, p.host.pack_map.data(), s));
    if (!p.pack_alias) ST_TRY(dev_alloc(p, &p.d_sendbuf, s * p.esize, true));
    p.ready = true;
    return DSPMV_OK;
}

// ------------------------------------------------- DSPMV_EXCHANGE_PUT setup
struct PutSeg {
    int64_t begin;
    char* dst0;        // peer receive buffer + its displacement for us (parity 0)
    char* dst1;        // same, parity 1
    unsigned* flag;    // peer flag slot for us
};

dspmv_status upload_put(Plan& p, const std::vector<PutSeg>& segs) {
    const int n = int(segs.size());
    p.put_nseg = n;
    if (n == 0) return DSPMV_OK;
    std::vector<int64_t> begin(n + 1);
    std::vector<void*> dst(2 * n);
    std::vector<unsigned*> flag(n);
    for (int j = 0; j < n; ++j) {
        begin[j] = segs[j].begin;
        dst[j] = segs[j].dst0;
        dst[n + j] = segs[j].dst1;
        flag[j] = segs[j].flag;
    }
    begin[n] = int64_t(p.host.pack_map.size());
    ST_TRY(dev_upload(p, &p.d_seg_begin, begin.data(), begin.size()));
    ST_TRY(dev_upload(p, &p.d_seg_dst, dst.data(), dst.size()));
    ST_TRY(dev_upload(p, &p.d_seg_flag, flag.data(), flag.size()));
    return DSPMV_OK;
}

// PUT: a rank publishes its epoch to, and waits for the epoch of, every rank
// it exchanges anything with in either direction (empty segments carry only
// the flag).  Otherwise a rank that only sends could run two applies ahead
// and overwrite the receive buffer its peer is still unpacking.
bool flag_peer(const RankPlan& h, int q) {
    return q != h.rank && (h.send_count[q] > 0 || h.recv_count[q] > 0);
}

// In-process group: peers' buffers are plain device pointers.
dspmv_status setup_put_local(LocalGroup& g) {
    for (int r = 0; r < g.nranks; ++r) {
        Plan& p = *g.plans[r];
        std::vector<PutSeg> segs;
        for (int d = 0; d < g.nranks; ++d) {
            if (!flag_peer(p.host, d)) continue;
            Plan& q = *g.plans[d];
            char* base = static_cast<char*>(q.d_recvbuf) + size_t(q.host.recv_displ[r]) * q.esize;
            segs.push_back({p.host.send_displ[d], base, base + q.recv_stride * q.esize, q.d_flags + r});
        }
        ST_TRY(upload_put(p, segs));
    }
    return DSPMV_OK;
}

// Plan-time all-gather over the comm's transport (NCCL or the HOST callback).
dspmv_status comm_allgather(Plan& p, const void* send, void* recv, size_t bytes) {
    Comm& c = *p.comm;
    if (c.kind == DSPMV_COMM_HOST) {
        if (c.allgather(send, recv, bytes, c.allgather_ctx) != 0) return fail(DSPMV_ERR_ARG, "allgather callback failed");
        return DSPMV_OK;
    }
    DevScratch d_in, d_out;
    CUDA_TRY(cudaMalloc(&d_in.p, bytes));
    CUDA_TRY(cudaMalloc(&d_out.p, bytes * c.nranks));
    CUDA_TRY(cudaMemcpy(d_in.p, send, bytes, cudaMemcpyHostToDevice));
    NCCL_TRY(ncclAllGather(d_in.p, d_out.p, bytes, ncclUint8, c.nccl, p.comm_stream));
    CUDA_TRY(cudaStreamSynchronize(p.comm_stream));
    CUDA_TRY(cudaMemcpy(recv, d_out.p, bytes * c.nranks, cudaMemcpyDeviceToHost));
    return DSPMV_OK;
}

// The request-list protocol of plan_create over all-gathers (HOST comms):
// counts matrix first, then every rank's halo (padded to the longest).
dspmv_status exchange_requests_allgather(Plan& p) {
    RankPlan& h = p.host;
    const int P = h.nranks, me = h.rank;
    std::vector<int32_t> counts(size_t(P) * P);
    ST_TRY(comm_allgather(p, h.recv_count.data(), counts.data(), size_t(P) * 4));
    int64_t hmax = 0;
    for (int r = 0; r < P; ++r) {
        int64_t t = 0;
        for (int q = 0; q < P; ++q) t += counts[size_t(r) * P + q];
        hmax = std::max(hmax, t);
    }
    std::vector<int32_t> mine(size_t(std::max<int64_t>(hmax, 1)), -1), all(size_t(std::max<int64_t>(hmax, 1)) * P);
    std::copy(h.halo_gid.begin(), h.halo_gid.end(), mine.begin());
    ST_TRY(comm_allgather(p, mine.data(), all.data(), mine.size() * 4));
    std::vector<std::vector<int32_t>> req(P);
    for (int r = 0; r < P; ++r) {
        int64_t off = 0;
        for (int q = 0; q < me; ++q) off += counts[size_t(r) * P + q];
        const int32_t c = counts[size_t(r) * P + me];
        const int32_t* src = all.data() + size_t(r) * mine.size() + off;
        req[r].assign(src, src + c);
    }
    plan_phase2_from_requests(h, req);
    return DSPMV_OK;
}

// Separate processes (NCCL or HOST comm): all-gather every rank's IPC handles
// (receive buffer, flags), parity stride and receive displacements; map the
// destinations' buffers (NVLink P2P between GPUs, or the same device).
dspmv_status setup_put_nccl(Plan& p) {
    const int P = p.host.nranks, me = p.host.rank;
    struct Rec {
        cudaIpcMemHandle_t recv, flags;
        int64_t h;
    };
    const size_t rec_bytes = (sizeof(Rec) + size_t(P) * 4 + 15) & ~size_t(15);
    std::vector<unsigned char> mine(rec_bytes, 0), all(rec_bytes * P, 0);
    Rec r{};
    if (p.d_recvbuf) CUDA_TRY(cudaIpcGetMemHandle(&r.recv, p.d_recvbuf));
    CUDA_TRY(cudaIpcGetMemHandle(&r.flags, p.d_flags));
    r.h = int64_t(p.recv_stride);  // parity stride of the receive buffer
    std::memcpy(mine.data(), &r, sizeof(Rec));
    std::memcpy(mine.data() + sizeof(Rec), p.host.recv_displ.data(), size_t(P) * 4);
    ST_TRY(comm_allgather(p, mine.data(), all.data(), rec_bytes));
    std::vector<PutSeg> segs;
    for (int d = 0; d < P; ++d) {
        if (!flag_peer(p.host, d)) continue;
        Rec rd;
        std::memcpy(&rd, all.data() + rec_bytes * d, sizeof(Rec));
        int32_t displ_me = 0;
        std::memcpy(&displ_me, all.data() + rec_bytes * d + sizeof(Rec) + size_t(me) * 4, 4);
        void *rb = nullptr, *fl = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&rb, rd.recv, cudaIpcMemLazyEnablePeerAccess));
        p.ipc_opened.push_back(rb);
        CUDA_TRY(cudaIpcOpenMemHandle(&fl, rd.flags, cudaIpcMemLazyEnablePeerAccess));
        p.ipc_opened.push_back(fl);
        char* base = static_cast<char*>(rb) + size_t(displ_me) * p.esize;
        segs.push_back({p.host.send_displ[d], base, base + size_t(rd.h) * p.esize, static_cast<unsigned*>(fl) + me});
    }
    return upload_put(p, segs);
}

dspmv_status finalize_local_group(LocalGroup& g) {
    const int P = g.nranks;
    for (int p = 0; p < P; ++p) {
        std::vector<std::vector<int32_t>> req(P);
        for (int r = 0; r < P; ++r) req[r] = halo_segment_for(g.plans[r]->host, p);
        plan_phase2_from_requests(g.plans[p]->host, req);
    }
    for (int p = 0; p < P; ++p) {
        CUDA_TRY(cudaSetDevice(g.plans[p]->device));
        ST_TRY(finalize_send(*g.plans[p]));
    }
    for (int p = 1; p < P; ++p)
        if (g.plans[p]->put_mode != g.plans[0]->put_mode)
            return fail(DSPMV_ERR_ARG, "every rank of a group must use the same exchange mode");
    if (g.plans[0]->put_mode) ST_TRY(setup_put_local(g));
    return DSPMV_OK;
}

dspmv_status exchange_requests_nccl(Plan& p) {
    RankPlan& h = p.host;
    const int P = h.nranks, me = h.rank;
    if (P == 1) {
        std::vector<std::vector<int32_t>> req(1);
        plan_phase2_from_requests(h, req);
        return DSPMV_OK;
    }
    ncclComm_t comm = p.comm->nccl;
    cudaStream_t s = p.comm_stream;
    DevScratch s_cnt, s_scnt, s_halo, s_req;
    CUDA_TRY(cudaMalloc(&s_cnt.p, sizeof(int32_t) * P));
    CUDA_TRY(cudaMalloc(&s_scnt.p, sizeof(int32_t) * P));
    int32_t* d_cnt = s_cnt.as<int32_t>();
    int32_t* d_scnt = s_scnt.as<int32_t>();
    CUDA_TRY(cudaMemcpy(d_cnt, h.recv_count.data(), sizeof(int32_t) * P, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemset(d_scnt, 0, sizeof(int32_t) * P));
    ncclResult_t gr = ncclSuccess;
    NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        NCCL_GROUP_CALL(gr, ncclSend(d_cnt + q, 1, ncclInt32, q, comm, s));
        NCCL_GROUP_CALL(gr, ncclRecv(d_scnt + q, 1, ncclInt32, q, comm, s));
    }
    NCCL_TRY(ncclGroupEnd());
    NCCL_TRY(gr);
    CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<int32_t> scnt(P);
    CUDA_TRY(cudaMemcpy(scnt.data(), d_scnt, sizeof(int32_t) * P, cudaMemcpyDeviceToHost));
    int64_t tot = 0;
    std::vector<int64_t> sdis(P, 0);
    for (int q = 0; q < P; ++q) {
        sdis[q] = tot;
        tot += scnt[q];
    }
    if (!h.halo_gid.empty()) {
        CUDA_TRY(cudaMalloc(&s_halo.p, sizeof(int32_t) * h.halo_gid.size()));
        CUDA_TRY(cudaMemcpy(s_halo.p, h.halo_gid.data(), sizeof(int32_t) * h.halo_gid.size(), cudaMemcpyHostToDevice));
    }
    if (tot) CUDA_TRY(cudaMalloc(&s_req.p, sizeof(int32_t) * tot));
    int32_t* d_halo = s_halo.as<int32_t>();
    int32_t* d_req = s_req.as<int32_t>();
    NCCL_TRY(ncclGroupStart());
    for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        if (h.recv_count[q] > 0)
            NCCL_GROUP_CALL(gr, ncclSend(d_halo + h.recv_displ[q], h.recv_count[q], ncclInt32, q, comm, s));
        if (scnt[q] > 0) NCCL_GROUP_CALL(gr, ncclRecv(d_req + sdis[q], scnt[q], ncclInt32, q, comm, s));
    }
    NCCL_TRY(ncclGroupEnd());
    NCCL_TRY(gr);
    CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<int32_t> all(tot);
    if (tot) CUDA_TRY(cudaMemcpy(all.data(), d_req, sizeof(int32_t) * tot, cudaMemcpyDeviceToHost));
    std::vector<std::vector<int32_t>> req(P);
    for (int q = 0; q < P; ++q) req[q].assign(all.begin() + sdis[q], all.begin() + sdis[q] + scnt[q]);
    plan_phase2_from_requests(h, req);
    return DSPMV_OK;
}

// ------------------------------------------------------------- executor
// CES: spin on cudaEventQuery (lower wake-up latency than the runtime's
// cudaEventSynchronize); DSPMV_BLOCKING_SYNC=1 falls back to the latter.
cudaError_t host_wait(cudaEvent_t ev) {
    static const bool blocking = [] {
        const char* v = std::getenv("DSPMV_BLOCKING_SYNC");
        return v && std::atoi(v) != 0;
    }();
    if (blocking) return cudaEventSynchronize(ev);
    for (;;) {
        const cudaError_t q = cudaEventQuery(ev);
        if (q != cudaErrorNotReady) return q;
    }
}

dspmv_status wait_group(Plan& p, const ExGroup& g) {
    if (g.empty()) return DSPMV_OK;  // nothing sent or received in this group
    if (p.comm->kind != DSPMV_COMM_NCCL || p.host.nranks == 1) {
        if (!p.put_mode || p.comm->kind == DSPMV_COMM_LOCAL) {
            CUDA_TRY(host_wait(g.ev));
            return DSPMV_OK;
        }
        // PUT across processes: a peer that never publishes must not hang us
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            const cudaError_t q = cudaEventQuery(g.ev);
            if (q == cudaSuccess) return DSPMV_OK;
            if (q != cudaErrorNotReady) return fail(DSPMV_ERR_CUDA, std::string("exchange: ") + cudaGetErrorString(q));
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) {
                p.poisoned = true;
                return fail(DSPMV_ERR_STATE, "PUT exchange: peer flags not published within 60 s");
            }
        }
    }
    const auto t_start = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t q = cudaEventQuery(g.ev);
        if (q == cudaSuccess) return DSPMV_OK;
        if (q != cudaErrorNotReady) return fail(DSPMV_ERR_CUDA, std::string("exchange: ") + cudaGetErrorString(q));
        ncclResult_t ar = ncclSuccess;
        ncclCommGetAsyncError(p.comm->nccl, &ar);
        if (ar != ncclSuccess && ar != ncclInProgress) {
            ncclCommAbort(p.comm->nccl);
            p.comm->nccl = nullptr;
            p.comm->poisoned = true;
            p.poisoned = true;
            return fail(DSPMV_ERR_NCCL, std::string("NCCL async error at Wait: ") + ncclGetErrorString(ar));
        }
        if (std::chrono::steady_clock::now() - t_start > std::chrono::seconds(120)) {
            p.poisoned = true;
            return fail(DSPMV_ERR_NCCL, "exchange did not complete within 120 s");
        }
    }
}

// COPY over NCCL: the group's receives and sends as one NCCL group.
dspmv_status issue_group_nccl(Plan& p, ExGroup& g) {
    g.issued = true;
    if (g.empty()) return DSPMV_OK;
    if (p.skip_exchange) {  // DSPMV_EXCHANGE_NONE: timing baseline, no data moves
        CUDA_TRY(cudaEventRecord(g.ev, p.comm_stream));
        return DSPMV_OK;
    }
    const RankPlan& h = p.host;
    const ncclDataType_t ty = nccl_type(p.dtype);
    char* rb = static_cast<char*>(p.d_recvbuf);
    char* sb = static_cast<char*>(p.d_sendbuf);
    if (p.pack_alias && p.streaming && p.pipe.pack_chunk >= 0 && !g.send_to.empty())
        CUDA_TRY(cudaStreamWaitEvent(p.comm_stream, p.pipe.ev_x[p.pipe.pack_chunk], 0));
    ncclResult_t gr = ncclSuccess;
    NCCL_TRY(ncclGroupStart());
    for (int q : g.recv_from)
        NCCL_GROUP_CALL(gr, ncclRecv(rb + size_t(h.recv_displ[q]) * p.esize, h.recv_count[q], ty, q, p.comm->nccl,
                                     p.comm_stream));
    for (int q : g.send_to) {
        const char* src = p.pack_alias ? static_cast<const char*>(p.cur_x) + size_t(p.alias_off[q]) * p.esize
                                       : sb + size_t(h.send_displ[q]) * p.esize;
        NCCL_GROUP_CALL(gr, ncclSend(src, h.send_count[q], ty, q, p.comm->nccl, p.comm_stream));
    }
    NCCL_TRY(ncclGroupEnd());
    NCCL_TRY(gr);
    CUDA_TRY(cudaEventRecord(g.ev, p.comm_stream));
    return DSPMV_OK;
}

PFN_cuStreamWaitValue32_v11070 wait_value32() {
    static PFN_cuStreamWaitValue32_v11070 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(f);
    }();
    return fn;
}

PFN_cuStreamWriteValue32_v11070 write_value32() {
    static PFN_cuStreamWriteValue32_v11070 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(f);
    }();
    return fn;
}

// PUT mode: the data moves inside the fused Pack kernels; the exchange is the
// comm stream waiting until every source of the group has published this epoch.
dspmv_status issue_group_put(Plan& p, ExGroup& g) {
    g.issued = true;
    if (g.empty()) return DSPMV_OK;
    if (p.comm->kind == DSPMV_COMM_HOST) {
        // peers may be other processes on this same GPU: their contexts
        // time-slice the device, and a context parked on a stream semaphore
        // wait is not switched out for the context that would release it --
        // so the wait is a (preemptible) spin kernel instead
        if (g.recv_from.size() > size_t(kMaxWaitPeers)) return fail(DSPMV_ERR_ARG, "too many peers for the flag wait");
        CUDA_TRY(launch_wait_flags(p.d_flags, g.recv_from.data(), int(g.recv_from.size()), nullptr, p.comm_stream,
                                   p.epoch));
        CUDA_TRY(cudaEventRecord(g.ev, p.comm_stream));
        return DSPMV_OK;
    }
    auto wv = wait_value32();
    if (!wv) return fail(DSPMV_ERR_CUDA, "cuStreamWaitValue32 unavailable");
    for (int q : g.recv_from) {
        const CUresult r = wv(reinterpret_cast<CUstream>(p.comm_stream), reinterpret_cast<CUdeviceptr>(p.d_flags + q),
                              p.epoch, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) return fail(DSPMV_ERR_CUDA, "cuStreamWaitValue32 failed (" + std::to_string(int(r)) + ")");
    }
    CUDA_TRY(cudaEventRecord(g.ev, p.comm_stream));
    return DSPMV_OK;
}

// PUT inside a captured graph: the wait on the sources' flags is a kernel
// comparing against the device epoch (a stream memory operation would freeze
// the epoch of the apply that was captured).
dspmv_status issue_group_put_graph(Plan& p, ExGroup& g) {
    g.issued = true;
    if (g.empty()) return DSPMV_OK;
    if (g.recv_from.size() > size_t(kMaxWaitPeers)) return fail(DSPMV_ERR_ARG, "too many peers for the graph wait");
    CUDA_TRY(launch_wait_flags(p.d_flags, g.recv_from.data(), int(g.recv_from.size()), p.d_epoch, p.comm_stream));
    CUDA_TRY(cudaEventRecord(g.ev, p.comm_stream));
    return DSPMV_OK;
}

// LOCAL group: group gi of every rank (lock-step, so all ranks have posted it).
dspmv_status issue_group_local(const std::vector<Schedule*>& ss, int gi) {
    if (!ss.empty() && ss[0]->plan->put_mode) {
        for (Schedule* s : ss) ST_TRY(issue_group_put(*s->plan, s->groups[gi]));
        return DSPMV_OK;
    }
    for (Schedule* s : ss) {
        Plan& pr = *s->plan;
        ExGroup& g = s->groups[gi];
        g.issued = true;
        const RankPlan& h = pr.host;
        for (int q : g.recv_from) {
            if (pr.skip_exchange) break;
            const Plan* src = ss[q]->plan;
            const char* from = src->pack_alias
                                   ? static_cast<const char*>(src->cur_x) + size_t(src->alias_off[h.rank]) * pr.esize
                                   : static_cast<const char*>(src->d_sendbuf) +
                                         size_t(src->host.send_displ[h.rank]) * pr.esize;
            CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(pr.d_recvbuf) + size_t(h.recv_displ[q]) * pr.esize,
                                     from,
                                     size_t(h.recv_count[q]) * pr.esize, cudaMemcpyDeviceToDevice, pr.comm_stream));
        }
        if (!g.empty()) CUDA_TRY(cudaEventRecord(g.ev, pr.comm_stream));
    }
    return DSPMV_OK;
}

// Resolve a schedule's exchange vertices against its plan (once the plan is
// ready): groups, peers, PUT segments, and the per-destination coverage check.
dspmv_status compile_exchange(Schedule& s) {
    Plan& p = *s.plan;
    const RankPlan& h = p.host;
    const int P = h.nranks, me = h.rank;
    auto data_send = [&](int q) { return q != me && h.send_count[q] > 0; };
    auto data_recv = [&](int q) { return q != me && h.recv_count[q] > 0; };
    auto sends = [&](int q) { return p.put_mode ? flag_peer(h, q) : data_send(q); };
    auto recvs = [&](int q) { return p.put_mode ? flag_peer(h, q) : data_recv(q); };
    std::vector<int> seg_of(P, -1);  // PUT segment index per destination
    for (int q = 0, j = 0; q < P; ++q)
        if (p.put_mode && flag_peer(h, q)) seg_of[q] = j++;
    const std::vector<int>& S = s.dag.offsets;
    auto has = [&](int d) { return std::binary_search(S.begin(), S.end(), d); };
    std::vector<ExGroup> groups;
    if (!s.dag.fine) {
        ExGroup g;
        for (int q = 0; q < P; ++q) {
            if (sends(q)) g.send_to.push_back(q);
            if (recvs(q)) g.recv_from.push_back(q);
        }
        groups.push_back(g);
    } else {
        for (int q = 0; q < P; ++q) {
            if ((sends(q) && !has(q - me)) || (recvs(q) && !has(me - q)))
                return fail(DSPMV_ERR_SCHEDULE, "per-destination schedule names no exchange with rank offset " +
                                                    std::to_string(q - me) + " (rank " + std::to_string(me) +
                                                    " exchanges with rank " + std::to_string(q) + ")");
        }
        for (int d : S) {
            ExGroup g;
            g.d = d;
            const int to = me + d, from = me - d;
            if (to >= 0 && to < P && sends(to)) g.send_to.push_back(to);
            if (from >= 0 && from < P && recvs(from)) g.recv_from.push_back(from);
            groups.push_back(g);
        }
    }
    auto group_of = [&](int d) {
        for (size_t i = 0; i < groups.size(); ++i)
            if (groups[i].d == d) return int(i);
        return -1;
    };
    const int n = int(s.ops.size());
    s.op_group.assign(n, -1);
    s.op_peer.assign(n, -2);
    s.op_seg.assign(n, -1);
    for (int t = 0; t < n; ++t) {
        const dspmv_op& o = s.ops[t];
        switch (o.kind) {
            case DSPMV_OP_POST_SEND:
            case DSPMV_OP_WAIT_SEND: s.op_group[t] = group_of(o.peer); break;
            case DSPMV_OP_POST_RECV:
            case DSPMV_OP_WAIT_RECV: s.op_group[t] = group_of(-o.peer); break;
            case DSPMV_OP_PACK:
                if (o.peer) {
                    const int q = me + o.peer;
                    const bool ok = q >= 0 && q < P && (p.put_mode ? flag_peer(h, q) : data_send(q));
                    s.op_peer[t] = ok ? q : -1;
                    s.op_seg[t] = ok && p.put_mode ? seg_of[q] : -1;
                }
                break;
            case DSPMV_OP_UNPACK:
                if (o.peer) {
                    const int q = me + o.peer;
                    s.op_peer[t] = (q >= 0 && q < P && data_recv(q)) ? q : -1;
                }
                break;
            default: break;
        }
    }
    for (ExGroup& g : groups)
        if (!g.ev) CUDA_TRY(cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming));
    s.groups.swap(groups);
    s.compiled = true;
    return DSPMV_OK;
}

dspmv_status begin_apply(Schedule& s, cudaStream_t caller) {
    Plan& p = *s.plan;
    if (p.poisoned) return fail(DSPMV_ERR_STATE, "plan is poisoned by an earlier error");
    if (!p.ready) return fail(DSPMV_ERR_STATE, "plan not ready (LOCAL group: not every rank has called plan_create)");
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != p.device) CUDA_TRY(cudaSetDevice(p.device));
    if (!s.compiled) ST_TRY(compile_exchange(s));
    if (s.step0) CUDA_TRY(cudaEventRecord(s.step0, caller));
    // timestamp aliasing (runtime.h): nothing on the caller stream yet; END is
    // recorded after the host's last wait, so it is never aliased here
    s.origin = caller;
    s.origin_dirty = p.streaming || !s.step0;
    s.origin_tail = -1;
    s.end_alias = -1;
    std::fill(s.t0_alias.begin(), s.t0_alias.end(), 0);
    ++p.epoch;
    if (p.d_epoch) {   // PUT: the kernels read the epoch from device memory
        auto wv = write_value32();
        if (!wv) return fail(DSPMV_ERR_CUDA, "cuStreamWriteValue32 unavailable");
        const CUresult r = wv(reinterpret_cast<CUstream>(caller), reinterpret_cast<CUdeviceptr>(p.d_epoch), p.epoch,
                              CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) return fail(DSPMV_ERR_CUDA, "cuStreamWriteValue32 failed (" + std::to_string(int(r)) + ")");
    }
    CUDA_TRY(cudaEventRecord(p.ev_start, caller));
    // schedule stream 0 may be the caller's stream itself (no cross-stream
    // wait for its work); the others wait on the caller's START point
    const bool cs0 = s.caller_stream0 >= 0 ? s.caller_stream0 != 0 : p.opts.caller_stream0 != 0;
    p.cur_stream0 = cs0 ? caller : p.streams[0];
    for (int i = cs0 ? 1 : 0; i < s.n_streams; ++i)
        CUDA_TRY(cudaStreamWaitEvent(p.streams[i], p.ev_start, 0));
    for (ExGroup& g : s.groups) g.ps = g.pr = g.issued = false;
    return DSPMV_OK;
}

// apply_host, y by copy engine: queue each group's wait-for-count + copy on
// the D2H stream.  Called right AFTER the y_L launch: streams can share a
// hardware queue (CUDA_DEVICE_MAX_CONNECTIONS), and a stream wait queued
// before the kernel that satisfies it could then block that kernel.
cudaError_t enqueue_ycopy(Plan& p) {
    auto& H = p.pipe;
    auto wait = wait_value32();
    if (!wait) return cudaErrorNotSupported;
    for (int k = 0; k < H.K; ++k) {
        if (H.yrow[k + 1] <= H.yrow[k]) continue;
        if (wait(reinterpret_cast<CUstream>(H.d2h), reinterpret_cast<CUdeviceptr>(H.d_ydone + k), H.nblk[k],
                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return cudaErrorUnknown;
        const size_t off = size_t(H.yrow[k]) * p.esize, len = size_t(H.yrow[k + 1] - H.yrow[k]) * p.esize;
        const cudaError_t e = cudaMemcpyAsync(static_cast<char*>(H.y_host) + off,
                                              static_cast<const char*>(p.d_yout) + off, len,
                                              cudaMemcpyDeviceToHost, H.d2h);
        if (e != cudaSuccess) return e;
    }
    H.y_queued = true;
    return cudaEventRecord(H.ev_out, H.d2h);
}

// The kernel(s) of GPU vertex op t on stream st (shared by the host-driven
// executor and graph capture).
cudaError_t launch_gpu_vertex(Schedule& s, int t, const void* x, void* y, cudaStream_t st) {
    Plan& p = *s.plan;
    cudaError_t e = cudaSuccess;
    switch (s.ops[t].kind) {
        case DSPMV_OP_PACK: {
            const int q = s.op_peer[t];  // -2: every destination; -1: nothing to send
            if (q == -1 || p.pack_alias) break;
            if (p.streaming && p.pipe.pack_chunk >= 0) {  // x still arriving (apply_host)
                e = cudaStreamWaitEvent(st, p.pipe.ev_x[p.pipe.pack_chunk], 0);
                if (e != cudaSuccess) break;
            }
            if (p.put_mode) {
                if (q == -2) {
                    PutArgs a{x, p.d_pack_map, 0, int64_t(p.host.pack_map.size()), p.d_seg_begin, p.d_seg_dst,
                              p.d_seg_flag, p.put_nseg, p.put_nseg, p.d_epoch, p.d_put_counter + p.put_nseg};
                    e = launch_pack_put(p.dtype, a, st);
                } else {
                    const int j = s.op_seg[t];
                    const int64_t k0 = p.host.send_displ[q];
                    PutArgs a{x, p.d_pack_map, k0, k0 + p.host.send_count[q], p.d_seg_begin + j, p.d_seg_dst + j,
                              p.d_seg_flag + j, 1, p.put_nseg, p.d_epoch, p.d_put_counter + j};
                    e = launch_pack_put(p.dtype, a, st);
                }
            } else if (q == -2) {
                e = launch_pack(p.dtype, x, p.d_pack_map, p.d_sendbuf, int64_t(p.host.pack_map.size()), st);
            } else {
                const int64_t k0 = p.host.send_displ[q];
                e = launch_pack(p.dtype, x, p.d_pack_map + k0, static_cast<char*>(p.d_sendbuf) + k0 * p.esize,
                                p.host.send_count[q], st);
            }
            break;
        }
        case DSPMV_OP_SPMV_LOCAL: {
            SpmvOperands op{x, y, p.d_partL, p.explicit_acc, p.d_partR, p.d_ticket};
            if (!p.streaming) {
                e = launch_spmv(p.L, p.dtype, op, st);
                break;
            }
            // apply_host pipeline: one launch; the producer warp of each CTA
            // waits for the x chunk flag of a block before staging it
            auto& H = p.pipe;
            if (p.L.stream) {  // CSR-stream tiles have no per-block x chunk: wait for all of x
                e = cudaStreamWaitEvent(st, H.ev_x[H.K - 1], 0);
                if (e == cudaSuccess) e = launch_spmv(p.L, p.dtype, op, st);
                break;
            }
            op.xflag = H.d_xflag;
            op.epoch = p.epoch;
            op.ydone = H.ycopy ? H.d_ydone : nullptr;
            e = launch_spmv_part(p.L, p.dtype, op, st, 0, p.L.nb, false);
            op.xflag = nullptr;
            op.ydone = nullptr;
            if (e == cudaSuccess && H.ycopy) e = enqueue_ycopy(p);
            if (e == cudaSuccess && p.L.nV > 0) {
                e = cudaStreamWaitEvent(st, H.ev_x[H.K - 1], 0);
                if (e == cudaSuccess) e = launch_spmv_part(p.L, p.dtype, op, st, p.L.nb, p.L.nb, true);
            }
            break;
        }
        case DSPMV_OP_UNPACK: {
            const int q = s.op_peer[t];
            if (q == -1 || p.unpack_fused) break;   // fused: y_R reads the receive buffer
            if (p.put_mode) {   // receive-buffer parity of this apply, from the device epoch
                const size_t off = q == -2 ? 0 : size_t(p.host.recv_displ[q]) * p.esize;
                const int64_t cnt = q == -2 ? int64_t(p.host.halo_gid.size()) : p.host.recv_count[q];
                e = launch_copy_parity(p.dtype, static_cast<const char*>(p.d_recvbuf) + off,
                                       p.recv_stride * size_t(p.esize), p.d_epoch,
                                       static_cast<char*>(p.d_xhalo) + off, cnt, st);
                break;
            }
            const char* src = static_cast<const char*>(p.d_recvbuf);
            if (q == -2) {
                e = launch_copy(p.dtype, src, p.d_xhalo, int64_t(p.host.halo_gid.size()), st);
            } else {
                const size_t off = size_t(p.host.recv_displ[q]) * p.esize;
                e = launch_copy(p.dtype, src + off, static_cast<char*>(p.d_xhalo) + off, p.host.recv_count[q], st);
            }
            break;
        }
        case DSPMV_OP_SPMV_REMOTE: {
            SpmvOperands op{p.d_xhalo, y, p.d_partR, p.explicit_acc, p.d_partL, p.d_ticket};
            if (p.unpack_fused) {   // R-Q8 fused: the halo is read where it was received
                op.x = p.d_recvbuf;
                if (p.put_mode) {
                    op.x_epoch = p.d_epoch;
                    op.x_parity_elems = int64_t(p.recv_stride);
                }
            }
            e = launch_spmv(p.R, p.dtype, op, st);
            break;
        }
        default:
            break;
    }
    return e;
}

// Execute op t of schedule s. `defer` = LOCAL group (exchange issued by caller).
// NVTX ranges (DSPMV_NVTX=1): one host range per executed schedule op and
// per apply, named after the paper's vertices and sync ops (SURVEY §5 tracing),
// so an nsys/ncu timeline shows the traversal.  Header-only NVTX3: free when no
// tool is attached, skipped entirely when the variable is unset.
bool nvtx_on() {
    static const bool on = [] {
        const char* ev = std::getenv("DSPMV_NVTX");
        return ev && std::atoi(ev) != 0;
    }();
    return on;
}
struct NvtxScope {
    bool on;
    explicit NvtxScope(bool enable, const std::string& name) : on(enable) {
        if (on) nvtxRangePushA(name.c_str());
    }
    ~NvtxScope() {
        if (on) nvtxRangePop();
    }
};
std::string op_label(const dspmv_op& o) {
    static const char* sync_names[] = {"CER", "CES", "CSWE"};
    std::string nm = is_dag_vertex(o.kind) ? vertex_label(o.kind, o.peer)
                                           : std::string(sync_names[(o.kind - DSPMV_OP_EVENT_RECORD) % 3]);
    if (is_gpu_vertex(o.kind) || o.kind == DSPMV_OP_EVENT_RECORD || o.kind == DSPMV_OP_STREAM_WAIT_EVENT)
        nm += "@s" + std::to_string(o.stream);
    return nm;
}

dspmv_status exec_op(Schedule& s, int t, const void* x, void* y, bool defer) {
    Plan& p = *s.plan;
    const dspmv_op& o = s.ops[t];
    NvtxScope nvtx_scope(nvtx_on(), nvtx_on() ? op_label(o) : std::string());
    const bool gpu = is_gpu_vertex(o.kind);
    const bool on_stream = gpu || o.kind == DSPMV_OP_EVENT_RECORD || o.kind == DSPMV_OP_STREAM_WAIT_EVENT;
    cudaStream_t st = on_stream ? (o.stream == 0 ? p.cur_stream0 : p.streams[o.stream]) : nullptr;
    const bool timed = gpu && s.timing && s.t0[t];
    if (timed) {
        if (st == s.origin && !s.origin_dirty) s.t0_alias[t] = 1;  // same position as START
        else CUDA_TRY(cudaEventRecord(s.t0[t], st));
    }
    const bool timed_x = !gpu && s.timing && s.t0[t];  // a Post: time the exchange it issues
    const uint64_t launches0 = g_launches.load(std::memory_order_relaxed);
    cudaError_t e = cudaSuccess;
    switch (o.kind) {
        case DSPMV_OP_START:
        case DSPMV_OP_END:
            break;
        case DSPMV_OP_PACK:
        case DSPMV_OP_SPMV_LOCAL:
        case DSPMV_OP_UNPACK:
        case DSPMV_OP_SPMV_REMOTE:
            e = launch_gpu_vertex(s, t, x, y, st);
            break;
        case DSPMV_OP_POST_SEND:
        case DSPMV_OP_POST_RECV: {
            ExGroup& g = s.groups[s.op_group[t]];
            if (o.kind == DSPMV_OP_POST_SEND) g.ps = true; else g.pr = true;
            if (!defer && g.ps && g.pr && !g.issued) {
                // exchange time on the comm stream (0 in op_times unless this op issued it)
                if (timed_x) CUDA_TRY(cudaEventRecord(s.t0[t], p.comm_stream));
                dspmv_status r = p.put_mode ? issue_group_put(p, g) : issue_group_nccl(p, g);
                if (r != DSPMV_OK) {
                    p.poisoned = true;
                    return r;
                }
                if (timed_x) CUDA_TRY(cudaEventRecord(s.t1[t], p.comm_stream));
            } else if (timed_x) {
                CUDA_TRY(cudaEventRecord(s.t0[t], p.comm_stream));
                CUDA_TRY(cudaEventRecord(s.t1[t], p.comm_stream));
            }
            break;
        }
        case DSPMV_OP_WAIT_SEND:
        case DSPMV_OP_WAIT_RECV: {
            const ExGroup& g = s.groups[s.op_group[t]];
            if (!g.issued) return fail(DSPMV_ERR_STATE, "Wait before the exchange was issued");
            dspmv_status r = wait_group(p, g);
            if (r != DSPMV_OK) return r;
            break;
        }
        case DSPMV_OP_EVENT_RECORD:
            e = cudaEventRecord(s.ev[o.event], st);
            break;
        case DSPMV_OP_EVENT_SYNC:
            e = host_wait(s.ev[o.event]);
            s.origin_dirty = true;  // later work is enqueued after a host wait
            break;
        case DSPMV_OP_STREAM_WAIT_EVENT:
            e = cudaStreamWaitEvent(st, s.ev[o.event], 0);
            if (st == s.origin) s.origin_dirty = true;
            break;
        default:
            return fail(DSPMV_ERR_SCHEDULE, "bad op");
    }
    if (o.kind == DSPMV_OP_WAIT_SEND || o.kind == DSPMV_OP_WAIT_RECV) s.origin_dirty = true;
    if (st == s.origin && g_launches.load(std::memory_order_relaxed) != launches0) s.origin_dirty = true;
    if (e != cudaSuccess) {
        p.poisoned = true;
        const char* sync_names[] = {"CER", "CES", "CSWE"};
        const std::string nm = is_dag_vertex(o.kind) ? vertex_label(o.kind, o.peer)
                                                     : std::string(sync_names[(o.kind - DSPMV_OP_EVENT_RECORD) % 3]);
        return fail(DSPMV_ERR_CUDA, "op " + std::to_string(t) + " (" + nm + "): " + cudaGetErrorString(e));
    }
    if (timed) {
        CUDA_TRY(cudaEventRecord(s.t1[t], st));
        if (st == s.origin) s.origin_dirty = true;
    }
    return DSPMV_OK;
}

// DSPMV_ACC_EXPLICIT_IN_END: after END every GPU vertex has completed,
// so one kernel on the caller's stream adds the deposited partials.
dspmv_status end_combine(Schedule& s, void* y, cudaStream_t st) {
    Plan& p = *s.plan;
    if (!p.explicit_acc || p.host.ar_rows.empty()) return DSPMV_OK;
    CUDA_TRY(launch_combine_end(p.dtype, p.d_partL, p.d_partR, p.d_ar_rows, y, int64_t(p.host.ar_rows.size()), st));
    if (s.origin == st) s.origin_dirty = true;
    return DSPMV_OK;
}

// FNV-1a over bytes
uint64_t fnv1a(const void* data, size_t n, uint64_t h = 1469598103934665603ull) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

// opts.debug_checks: does every rank hold the same value?  NCCL: all-reduce
// MIN of (h, ~h) -- equal everywhere iff min(h) == ~min(~h) = max(h); HOST:
// the caller's allgather; LOCAL: compared over the group's plans.
dspmv_status ranks_agree(Plan& p, uint64_t h, bool* same) {
    *same = true;
    Comm& c = *p.comm;
    if (c.nranks == 1) return DSPMV_OK;
    if (c.kind == DSPMV_COMM_NCCL) {
        DevScratch d;
        CUDA_TRY(cudaMalloc(&d.p, 16));
        const uint64_t hv[2] = {h, ~h};
        CUDA_TRY(cudaMemcpyAsync(d.p, hv, 16, cudaMemcpyHostToDevice, p.comm_stream));
        NCCL_TRY(ncclAllReduce(d.p, d.p, 2, ncclUint64, ncclMin, c.nccl, p.comm_stream));
        uint64_t r[2];
        CUDA_TRY(cudaMemcpyAsync(r, d.p, 16, cudaMemcpyDeviceToHost, p.comm_stream));
        CUDA_TRY(cudaStreamSynchronize(p.comm_stream));
        *same = r[0] == ~r[1];
    } else if (c.kind == DSPMV_COMM_HOST) {
        std::vector<uint64_t> all(size_t(c.nranks));
        if (c.allgather(&h, all.data(), 8, c.allgather_ctx) != 0) return fail(DSPMV_ERR_ARG, "allgather failed");
        for (uint64_t v : all) *same &= v == h;
    }
    return DSPMV_OK;
}

dspmv_status check_schedule_hash(Schedule& s) {
    Plan& p = *s.plan;
    if (!p.opts.debug_checks || s.hash_checked || p.comm->kind == DSPMV_COMM_LOCAL) return DSPMV_OK;
    bool same = true;
    ST_TRY(ranks_agree(p, fnv1a(s.ops.data(), s.ops.size() * sizeof(dspmv_op), fnv1a(&s.n_streams, 4)), &same));
    if (!same) return fail(DSPMV_ERR_SCHEDULE, "debug check: the ranks apply different schedules (P:460)");
    s.hash_checked = true;
    return DSPMV_OK;
}

// ------------------------------------------------ GPU-resident schedules
// Capture the schedule into a CUDA graph (NEXT-3 (iii)): GPU vertices,
// CER and CSWE are captured as they are; a host synchronisation point (CES,
// WaitSend, WaitRecv) -- after which the host would enqueue every later op --
// becomes "every stream waits on that event", which orders all later work
// after it exactly as the host sync did; the exchange (NCCL group) is
// captured on the comm stream; START/END are the fork from / join into the
// caller's stream.  Timed ops record external events, so op times and the
// timeline work unchanged.
// One capture serves a single rank (dspmv_apply_graph) or every rank of a
// LOCAL group in lock-step (dspmv_apply_graph_group: one graph, each rank's
// ops on that rank's own streams, so the ranks' branches run concurrently).
// The graph and the pointers it was captured for are stored on ss[0].
dspmv_status capture_graph(const std::vector<Schedule*>& ss, const std::vector<const void*>& xs,
                           const std::vector<void*>& ys, cudaStream_t origin) {
    const int R = int(ss.size());
    const bool group = R > 1;
    Schedule& s0 = *ss[0];
    for (Schedule* sp : ss) {
        if (!sp->compiled) ST_TRY(compile_exchange(*sp));
        for (auto& e : sp->gev)
            if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // per rank: schedule streams (stream 0 may be the origin for one rank
    // only), all streams incl. the comm stream, Pack-done events (COPY groups)
    struct RankCap {
        std::vector<cudaStream_t> st, all;
        bool ev_trivial[DSPMV_MAX_EVENTS] = {};
        std::vector<cudaEvent_t> pack_ev;   // by destination rank, recorded after its Pack
    };
    std::vector<RankCap> rc(R);
    for (int r = 0; r < R; ++r) {
        Plan& p = *ss[r]->plan;
        const int ns = ss[r]->n_streams;
        rc[r].st.resize(ns);
        const bool cs0 = ss[r]->caller_stream0 >= 0 ? ss[r]->caller_stream0 != 0 : p.opts.caller_stream0 != 0;
        for (int i = 0; i < ns; ++i) rc[r].st[i] = (i == 0 && cs0 && !group) ? origin : p.streams[i];
        rc[r].all = rc[r].st;
        if (p.has_peers) rc[r].all.push_back(p.comm_stream);
        if (group && !p.put_mode) {
            if (p.g_pack_ev.empty()) {
                p.g_pack_ev.assign(size_t(p.host.nranks), nullptr);
                for (auto& e : p.g_pack_ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            }
            rc[r].pack_ev.assign(size_t(p.host.nranks), nullptr);
        }
    }
    auto is_origin = [&](cudaStream_t q) { return q == origin; };
    const uint64_t launches0 = g_launches.load();
    CUDA_TRY(cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal));
    auto abort_capture = [&](dspmv_status stt) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(origin, &g);
        if (g) cudaGraphDestroy(g);
        return stt;
    };
#define CAP_TRY(expr)                                                                          \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return abort_capture(fail(DSPMV_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e))); \
    } while (0)
    for (Schedule* sp : ss)
        if (sp->step0) CAP_TRY(cudaEventRecordWithFlags(sp->step0, origin, cudaEventRecordExternal));
    // PUT: the first node advances the device epoch (the host executor writes
    // it at START instead); every Pack / Unpack / flag wait of this graph
    // reads it, so one captured graph serves every apply
    bool any_epoch = false;
    for (Schedule* sp : ss)
        if (sp->plan->d_epoch) {
            CAP_TRY(launch_epoch_bump(sp->plan->d_epoch, origin));
            any_epoch = true;
        }
    CAP_TRY(cudaEventRecord(s0.gev[0], origin));
    // timestamp aliasing (runtime.h), single rank only: track what lands on
    // the origin stream
    bool odirty = !s0.step0 || any_epoch || group, others = false;
    int otail = -1;
    std::vector<std::vector<char>> a0(R);
    for (int r = 0; r < R; ++r) {
        a0[r].assign(ss[r]->ops.size(), 0);
        for (int& v : ss[r]->ev_on) v = 0;
        for (cudaStream_t q : rc[r].all)
            if (!is_origin(q)) CAP_TRY(cudaStreamWaitEvent(q, s0.gev[0], 0));
        for (ExGroup& g : ss[r]->groups) g.ps = g.pr = g.issued = false;
        ss[r]->plan->cur_x = xs[r];
    }
    // every stream of rank r waits on ev; the stream ev was recorded on
    // (from, if known) needs no wait on itself
    auto all_wait = [&](int r, cudaEvent_t ev, cudaStream_t from, bool trivial) -> cudaError_t {
        for (cudaStream_t q : rc[r].all) {
            if (q == from) continue;
            cudaError_t e = cudaStreamWaitEvent(q, ev, 0);
            if (e != cudaSuccess) return e;
            if (is_origin(q) && !trivial) odirty = true, otail = -1;
        }
        return cudaSuccess;
    };
    const int n_ops = int(s0.ops.size());
    for (int t = 0; t < n_ops; ++t) {
        for (int r = 0; r < R; ++r) {
            Schedule& s = *ss[r];
            Plan& p = *s.plan;
            const dspmv_op& o = s.ops[t];
            const bool gpu = is_gpu_vertex(o.kind);
            cudaStream_t q = (gpu || o.kind == DSPMV_OP_EVENT_RECORD || o.kind == DSPMV_OP_STREAM_WAIT_EVENT)
                                 ? rc[r].st[o.stream] : nullptr;
            const bool timed = gpu && s.timing && s.t0[t];
            if (timed) {
                if (is_origin(q) && !odirty) a0[r][t] = 1;  // same position as START
                else CAP_TRY(cudaEventRecordWithFlags(s.t0[t], q, cudaEventRecordExternal));
                if (!is_origin(q)) others = true;
            }
            switch (o.kind) {
                case DSPMV_OP_PACK:
                case DSPMV_OP_SPMV_LOCAL:
                case DSPMV_OP_UNPACK:
                case DSPMV_OP_SPMV_REMOTE: {
                    const uint64_t l0 = g_launches.load();
                    CAP_TRY(launch_gpu_vertex(s, t, xs[r], ys[r], q));
                    if (g_launches.load() != l0) {
                        if (is_origin(q)) odirty = true, otail = -1;
                        else others = true;
                    }
                    // LOCAL COPY group: the receivers' copies wait for this Pack
                    if (o.kind == DSPMV_OP_PACK && !rc[r].pack_ev.empty() && s.op_peer[t] != -1) {
                        const int qd = s.op_peer[t];
                        cudaEvent_t ev = p.g_pack_ev[qd == -2 ? 0 : qd];
                        CAP_TRY(cudaEventRecord(ev, q));
                        for (int d = 0; d < p.host.nranks; ++d)
                            if (qd == -2 || d == qd) rc[r].pack_ev[d] = ev;
                    }
                    break;
                }
                case DSPMV_OP_POST_SEND:
                case DSPMV_OP_POST_RECV: {
                    ExGroup& g = s.groups[s.op_group[t]];
                    (o.kind == DSPMV_OP_POST_SEND ? g.ps : g.pr) = true;
                    const bool tx = s.timing && s.t0[t];
                    cudaStream_t xs_ = p.has_peers ? p.comm_stream : origin;  // comm joins only with peers
                    if (tx) CAP_TRY(cudaEventRecordWithFlags(s.t0[t], xs_, cudaEventRecordExternal));
                    if (g.ps && g.pr && !g.issued && (!group || p.put_mode)) {
                        // captured on the comm stream: the NCCL group, or (PUT) a
                        // kernel waiting for the sources' epoch flags
                        dspmv_status st_ = p.put_mode ? issue_group_put_graph(p, g) : issue_group_nccl(p, g);
                        if (st_ != DSPMV_OK) return abort_capture(st_);
                    }
                    if (tx && !group) CAP_TRY(cudaEventRecordWithFlags(s.t1[t], xs_, cudaEventRecordExternal));
                    if (tx || p.has_peers) {
                        if (is_origin(xs_)) odirty = true, otail = -1;
                        else others = true;
                    }
                    break;
                }
                case DSPMV_OP_WAIT_SEND:
                case DSPMV_OP_WAIT_RECV: {
                    const ExGroup& g = s.groups[s.op_group[t]];
                    if (!g.empty()) CAP_TRY(all_wait(r, g.ev, nullptr, false));
                    break;
                }
                case DSPMV_OP_EVENT_RECORD:
                    CAP_TRY(cudaEventRecord(s.ev[o.event], q));
                    s.ev_on[o.event] = o.stream + 1;
                    rc[r].ev_trivial[o.event] = !is_origin(q) && !others;
                    break;
                case DSPMV_OP_EVENT_SYNC:
                    CAP_TRY(all_wait(r, s.ev[o.event], s.ev_on[o.event] ? rc[r].st[s.ev_on[o.event] - 1] : nullptr,
                                     rc[r].ev_trivial[o.event]));
                    break;
                case DSPMV_OP_STREAM_WAIT_EVENT:
                    CAP_TRY(cudaStreamWaitEvent(q, s.ev[o.event], 0));
                    if (is_origin(q) && !rc[r].ev_trivial[o.event]) odirty = true, otail = -1;
                    break;
                default:
                    break;
            }
            if (timed) {
                CAP_TRY(cudaEventRecordWithFlags(s.t1[t], q, cudaEventRecordExternal));
                if (is_origin(q)) odirty = true, otail = t;
            }
        }
        // LOCAL COPY group, lock-step: group gi is posted on every rank at op t
        if (group && !s0.plan->put_mode) {
            const int gi = s0.op_group[t];
            if (gi >= 0 && s0.groups[gi].ps && s0.groups[gi].pr && !s0.groups[gi].issued) {
                for (int r = 0; r < R; ++r) {
                    Plan& pr = *ss[r]->plan;
                    ExGroup& g = ss[r]->groups[gi];
                    g.issued = true;
                    const RankPlan& h = pr.host;
                    for (int q : g.recv_from) {
                        if (pr.skip_exchange) break;
                        if (cudaEvent_t ev = rc[q].pack_ev.empty() ? nullptr : rc[q].pack_ev[h.rank])
                            CAP_TRY(cudaStreamWaitEvent(pr.comm_stream, ev, 0));
                        const Plan* src = ss[q]->plan;
                        const char* from = src->pack_alias
                                               ? static_cast<const char*>(xs[q]) + size_t(src->alias_off[h.rank]) * pr.esize
                                               : static_cast<const char*>(src->d_sendbuf) +
                                                     size_t(src->host.send_displ[h.rank]) * pr.esize;
                        CAP_TRY(cudaMemcpyAsync(static_cast<char*>(pr.d_recvbuf) + size_t(h.recv_displ[q]) * pr.esize,
                                                from, size_t(h.recv_count[q]) * pr.esize, cudaMemcpyDeviceToDevice,
                                                pr.comm_stream));
                    }
                    if (!g.empty()) CAP_TRY(cudaEventRecord(g.ev, pr.comm_stream));
                }
            }
        }
        if (group) {   // timed Posts of a group: the exchange interval on each comm stream
            for (int r = 0; r < R; ++r) {
                Schedule& s = *ss[r];
                const int k = s.ops[t].kind;
                if ((k == DSPMV_OP_POST_SEND || k == DSPMV_OP_POST_RECV) && s.timing && s.t0[t])
                    CAP_TRY(cudaEventRecordWithFlags(s.t1[t], s.plan->has_peers ? s.plan->comm_stream : origin,
                                                     cudaEventRecordExternal));
            }
        }
    }
    bool any_explicit = false;
    for (Schedule* sp : ss) any_explicit |= sp->plan->explicit_acc;
    // END directly behind an op's end event on origin, with no node on any
    // other stream: that event is END (no second record)
    const int ealias = (!group && s0.step1 && otail >= 0 && !others && !any_explicit) ? otail : -1;
    // join every stream back into the origin
    int k = 1;
    for (int r = 0; r < R; ++r) {
        Schedule& s = *ss[r];
        for (cudaStream_t q : rc[r].all) {
            if (is_origin(q)) continue;
            cudaEvent_t ev = s.gev[k];   // k <= DSPMV_MAX_STREAMS + 1
            CAP_TRY(cudaEventRecord(ev, q));
            CAP_TRY(cudaStreamWaitEvent(origin, ev, 0));
            ++k;
        }
        k = 1;
    }
    for (int r = 0; r < R; ++r) {
        if (ss[r]->plan->explicit_acc) {
            const dspmv_status cst = end_combine(*ss[r], ys[r], origin);
            if (cst != DSPMV_OK) return abort_capture(cst);
        }
    }
    for (Schedule* sp : ss)
        if (sp->step1 && ealias < 0) CAP_TRY(cudaEventRecordWithFlags(sp->step1, origin, cudaEventRecordExternal));
#undef CAP_TRY
    cudaGraph_t g = nullptr;
    CUDA_TRY(cudaStreamEndCapture(origin, &g));
    // captured launches run with each graph launch, not now
    s0.graph_kernels = g_launches.load() - launches0;
    g_launches.fetch_sub(s0.graph_kernels);
    if (s0.gexec) cudaGraphExecDestroy(s0.gexec), s0.gexec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&s0.gexec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail(DSPMV_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
    s0.gx = xs[0];
    s0.gy = ys[0];
    for (Schedule* m : s0.g_group)
        if (m != &s0) m->g_leader = nullptr;
    s0.g_group.clear();
    if (group)
        for (int r = 0; r < R; ++r) {
            if (r > 0) ss[r]->g_leader = &s0;
            s0.g_group.push_back(ss[r]);
            s0.g_group_ptrs.push_back(xs[r]);
            s0.g_group_ptrs.push_back(ys[r]);
        }
    for (int r = 0; r < R; ++r) {
        Schedule& s = *ss[r];
        s.g_timing = s.timing;
        if (s.timing) {
            s.g_t0_alias = a0[r];
            s.g_end_alias = ealias;
        }
    }
    return DSPMV_OK;
}

dspmv_status capture_graph(Schedule& s, const void* x, void* y, cudaStream_t origin) {
    Plan& p = *s.plan;
    if (p.comm->kind == DSPMV_COMM_LOCAL && p.host.nranks > 1)
        return fail(DSPMV_ERR_ARG, "apply_graph: LOCAL groups with > 1 rank run with dspmv_apply_graph_group");
    s.g_group_ptrs.clear();
    return capture_graph(std::vector<Schedule*>{&s}, std::vector<const void*>{x}, std::vector<void*>{y}, origin);
}

std::mutex g_flush_mu;
void* g_flush_buf[64] = {};
size_t g_flush_bytes[64] = {};

}  // namespace
}  // namespace dspmv

using namespace dspmv;

struct dspmv_comm_s : dspmv::Comm {};
struct dspmv_plan_s : dspmv::Plan {};
struct dspmv_schedule_s : dspmv::Schedule {};
struct dspmv_host_plan_s {
    std::vector<dspmv::RankPlan> ranks;
    int esize = 8;
    bool has_val = false;
};

extern "C" {

const char* dspmv_last_error(void) { return t_err.c_str(); }
int dspmv_version(void) { return DSPMV_VERSION; }

dspmv_status dspmv_partition(int64_t n_global, int nranks, int64_t* row_begin) {
    if (nranks < 1 || n_global < 0 || !row_begin) return fail(DSPMV_ERR_ARG, "bad partition arguments");
    const auto rb = partition(n_global, nranks);
    std::copy(rb.begin(), rb.end(), row_begin);
    return DSPMV_OK;
}

// ---------------------------------------------------------------- comms
dspmv_status dspmv_comm_unique_id(unsigned char id[128]) {
    if (!id) return fail(DSPMV_ERR_ARG, "null id");
    ncclUniqueId u;
    NCCL_TRY(ncclGetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(id, &u, 128);
    return DSPMV_OK;
}

dspmv_status dspmv_comm_create(const unsigned char id[128], int nranks, int rank, int cuda_device,
                               dspmv_comm_t* out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(DSPMV_ERR_ARG, "bad comm arguments");
    CUDA_TRY(cudaSetDevice(cuda_device));
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    auto* c = new dspmv_comm_s();
    c->kind = DSPMV_COMM_NCCL;
    c->nranks = nranks;
    c->rank = rank;
    c->device = cuda_device;
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(DSPMV_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    *out = c;
    return DSPMV_OK;
}

dspmv_status dspmv_comm_create_local(int nranks, int cuda_device, dspmv_comm_t* out) {
    if (!out || nranks < 1) return fail(DSPMV_ERR_ARG, "bad local comm arguments");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (cuda_device < 0 || cuda_device >= ndev) return fail(DSPMV_ERR_ARG, "no such device");
    auto g = std::make_shared<LocalGroup>();
    g->nranks = nranks;
    g->device = cuda_device;
    g->plans.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
        auto* c = new dspmv_comm_s();
        c->kind = DSPMV_COMM_LOCAL;
        c->nranks = nranks;
        c->rank = r;
        c->device = cuda_device;
        c->group = g;
        out[r] = c;
    }
    return DSPMV_OK;
}

dspmv_status dspmv_comm_create_host(int nranks, int rank, int cuda_device, dspmv_allgather_fn allgather, void* ctx,
                                    dspmv_comm_t* out) {
    if (!out || !allgather || nranks < 1 || rank < 0 || rank >= nranks) return fail(DSPMV_ERR_ARG, "bad host comm arguments");
    CUDA_TRY(cudaSetDevice(cuda_device));
    auto* c = new dspmv_comm_s();
    c->kind = DSPMV_COMM_HOST;
    c->nranks = nranks;
    c->rank = rank;
    c->device = cuda_device;
    c->allgather = allgather;
    c->allgather_ctx = ctx;
    *out = c;
    return DSPMV_OK;
}

dspmv_status dspmv_comm_destroy(dspmv_comm_t comm) {
    if (!comm) return fail(DSPMV_ERR_ARG, "null comm");
    if (comm->live_plans > 0) return fail(DSPMV_ERR_STATE, "comm still has live plans");
    if (comm->nccl) ncclCommDestroy(comm->nccl);
    delete comm;
    return DSPMV_OK;
}

dspmv_status dspmv_comm_info(dspmv_comm_t comm, int* nranks, int* rank, int* kind) {
    if (!comm) return fail(DSPMV_ERR_ARG, "null comm");
    if (nranks) *nranks = comm->nranks;
    if (rank) *rank = comm->rank;
    if (kind) *kind = comm->kind;
    return DSPMV_OK;
}

// ----------------------------------------------------------------- plans
void dspmv_plan_opts_default(dspmv_plan_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->dtype = DSPMV_F64;
    o->vector_threshold = -1;
    o->keep_host = 0;
    o->comm_priority = 1;
    o->block_cfg = -1;
    o->caller_stream0 = 0;
    o->reserve_sms = -1;
    o->exchange = DSPMV_EXCHANGE_COPY;
    if (const char* ev = std::getenv("DSPMV_CALLER_STREAM0")) o->caller_stream0 = std::atoi(ev);
    if (const char* ev = std::getenv("DSPMV_RESERVE_SMS")) o->reserve_sms = std::atoi(ev);
    if (const char* ev = std::getenv("DSPMV_DEBUG_CHECKS")) o->debug_checks = std::atoi(ev);
}

static void free_plan_device(Plan& p) {
    for (void* a : p.ipc_opened) cudaIpcCloseMemHandle(a);
    p.ipc_opened.clear();
    if (!p.allocs.empty()) cudaDeviceSynchronize();   // nothing of the plan in flight
    for (const auto& a : p.allocs) {
        if (a.cb) p.opts.free(a.ptr, a.bytes, p.device, p.opts.alloc_ctx);
        else cudaFree(a.ptr);
    }
    p.allocs.clear();
    for (auto& s : p.streams)
        if (s) cudaStreamDestroy(s), s = nullptr;
    if (p.comm_stream) cudaStreamDestroy(p.comm_stream), p.comm_stream = nullptr;
    if (p.pipe.h2d) cudaStreamDestroy(p.pipe.h2d), p.pipe.h2d = nullptr;
    for (auto& e : p.pipe.ev_x)
        if (e) cudaEventDestroy(e), e = nullptr;
    if (p.pipe.ev_in) cudaEventDestroy(p.pipe.ev_in), p.pipe.ev_in = nullptr;
    if (p.pipe.d2h) cudaStreamDestroy(p.pipe.d2h), p.pipe.d2h = nullptr;
    if (p.pipe.ev_zero) cudaEventDestroy(p.pipe.ev_zero), p.pipe.ev_zero = nullptr;
    if (p.pipe.ev_out) cudaEventDestroy(p.pipe.ev_out), p.pipe.ev_out = nullptr;
    for (auto& e : p.g_pack_ev)
        if (e) cudaEventDestroy(e);
    p.g_pack_ev.clear();
    if (p.ev_start) cudaEventDestroy(p.ev_start), p.ev_start = nullptr;
}

dspmv_status dspmv_plan_create(dspmv_comm_t comm, int64_t n_global, int64_t n_local, const int64_t* rowptr,
                               const int32_t* col_global, const void* val, const dspmv_plan_opts* opts_in,
                               dspmv_plan_t* out) {
    if (!comm || !out) return fail(DSPMV_ERR_ARG, "null comm/out");
    if (comm->poisoned) return fail(DSPMV_ERR_STATE, "comm poisoned");
    dspmv_plan_opts opts;
    dspmv_plan_opts_default(&opts);
    if (opts_in) opts = *opts_in;
    if (opts.dtype != DSPMV_F64 && opts.dtype != DSPMV_F32) return fail(DSPMV_ERR_ARG, "bad dtype");
    if (opts.long_row_sum != DSPMV_LONG_ROW_TREE && opts.long_row_sum != DSPMV_LONG_ROW_STORED)
        return fail(DSPMV_ERR_ARG, "bad long_row_sum");
    int vthr = opts.vector_threshold < 0 ? kDefaultVectorThreshold : opts.vector_threshold;
    int cfg = opts.block_cfg;  // -1: chosen per layout (auto_block_cfg)
    if (const char* ev = std::getenv("DSPMV_BLOCK_CFG")) cfg = std::atoi(ev);  // tuning sweeps
    if (cfg < -1 || cfg >= kNumBlockCfgs) return fail(DSPMV_ERR_ARG, "block_cfg out of range");
    if (vthr > (cfg < 0 ? kTileMin : kBlockCfgs[cfg].tile))
        return fail(DSPMV_ERR_ARG, "vector_threshold > tile of block_cfg");
    if (n_local > 0 && !val) return fail(DSPMV_ERR_ARG, "null val");
    if (comm->kind == DSPMV_COMM_LOCAL && comm->group->plans[comm->rank])
        return fail(DSPMV_ERR_STATE, "this LOCAL rank already has a plan");
    CUDA_TRY(cudaSetDevice(comm->device));

    auto* p = new dspmv_plan_s();
    p->comm = comm;
    p->device = comm->device;
    p->dtype = opts.dtype;
    p->esize = opts.dtype == DSPMV_F32 ? 4 : 8;
    p->opts = opts;
    auto bail = [&](dspmv_status st) {
        std::string keep = t_err;
        free_plan_device(*p);
        delete p;
        t_err = keep;
        return st;
    };
    dspmv_status st = plan_phase1(n_global, comm->nranks, comm->rank, n_local, rowptr, col_global, val, p->esize,
                                  p->host);
    if (st != DSPMV_OK) return bail(st);
    RankPlan& h = p->host;
    p->nnz_L = int64_t(h.al_col.size());
    p->nnz_R = int64_t(h.ar_col.size());

    // streams: schedule streams + comm stream (highest priority if requested).
    // Every schedule stream gets the same priority: the design space treats
    // the streams as interchangeable (stream-bijection pruning), so
    // no schedule stream may be privileged.
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    for (int i = 0; i < DSPMV_MAX_STREAMS; ++i) {
        if (cudaStreamCreateWithPriority(&p->streams[i], cudaStreamNonBlocking, lo) != cudaSuccess)
            return bail(fail(DSPMV_ERR_CUDA, "cudaStreamCreateWithPriority failed"));
    }
    if (cudaStreamCreateWithPriority(&p->comm_stream, cudaStreamNonBlocking, opts.comm_priority ? hi : lo) !=
            cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(DSPMV_ERR_CUDA, "stream/event creation failed"));

    // device layouts of A_L (slots = position of the row in ar_rows) and A_R
    const int32_t nR = int32_t(h.ar_rows.size());
    std::vector<int32_t> slotL;
    if (nR > 0) {
        slotL.assign(size_t(h.n_local()), -1);
        for (int32_t k = 0; k < nR; ++k) slotL[h.ar_rows[k]] = k;
    }
    {
        Layout L;
        const int c = cfg >= 0 ? cfg : auto_block_cfg(h.al_rowptr.data(), int32_t(h.n_local()), vthr, p->esize);
        const bool sl = use_stream(opts, h.al_rowptr.data(), int32_t(h.n_local()), vthr);
        build_layout(h.al_rowptr.data(), int32_t(h.n_local()), h.al_col.data(), h.al_val.data(), p->esize, nullptr,
                     nR > 0 ? slotL.data() : nullptr, vthr, kBlockCfgs[c], L, sl, use_sell(opts, sl));
        build_host_pipe(*p, L);   // also stores each block's x chunk in desc[15]
        if ((st = upload_layout(*p, L, c, p->L)) != DSPMV_OK) return bail(st);
        p->L.x_bytes = h.n_local() * p->esize;
    }
    {
        std::vector<int32_t> slotR(nR);
        for (int32_t k = 0; k < nR; ++k) slotR[k] = k;
        Layout R;
        const int c = cfg >= 0 ? cfg : auto_block_cfg(h.ar_rowptr.data(), nR, vthr, p->esize);
        const bool sr = use_stream(opts, h.ar_rowptr.data(), nR, vthr);
        build_layout(h.ar_rowptr.data(), nR, h.ar_col.data(), h.ar_val.data(), p->esize, h.ar_rows.data(),
                     slotR.data(), vthr, kBlockCfgs[c], R, sr, use_sell(opts, sr));
        if ((st = upload_layout(*p, R, c, p->R)) != DSPMV_OK) return bail(st);
        p->R.x_bytes = int64_t(h.halo_gid.size()) * p->esize;
    }
    const size_t hsz = h.halo_gid.size();
    p->put_mode = opts.exchange == DSPMV_EXCHANGE_PUT;
    p->skip_exchange = opts.exchange == DSPMV_EXCHANGE_NONE;
    if (opts.exchange != DSPMV_EXCHANGE_COPY && opts.exchange != DSPMV_EXCHANGE_PUT &&
        opts.exchange != DSPMV_EXCHANGE_NONE)
        return bail(fail(DSPMV_ERR_ARG, "bad exchange mode"));
    // PUT: two receive buffers (apply parity) -- a rank may run one apply ahead
    // parity stride padded to 256 B so both halves stay 16-B aligned for Unpack
    p->recv_stride = ((hsz * p->esize + 255) / 256 * 256) / p->esize;
    if ((st = dev_alloc(*p, &p->d_recvbuf,
                        p->put_mode ? std::max<size_t>(2 * p->recv_stride * p->esize, 256) : hsz * p->esize, true,
                        p->put_mode)) != DSPMV_OK)
        return bail(st);
    if (p->put_mode) {
        // own allocation (IPC-exportable); at least one word so every rank has a handle
        if ((st = dev_alloc(*p, reinterpret_cast<void**>(&p->d_flags), size_t(comm->nranks) * 4, true, true)) !=
            DSPMV_OK)
            return bail(st);
        if ((st = dev_alloc(*p, reinterpret_cast<void**>(&p->d_epoch), 4, true)) != DSPMV_OK) return bail(st);
        // last-CTA counters: one per destination segment (per-destination Pack) + one
        if ((st = dev_alloc(*p, reinterpret_cast<void**>(&p->d_put_counter), size_t(comm->nranks + 1) * 4, true)) !=
            DSPMV_OK)
            return bail(st);
    }
    if ((st = dev_alloc(*p, &p->d_xhalo, hsz * p->esize, true)) != DSPMV_OK) return bail(st);
    if ((st = dev_alloc(*p, &p->d_partL, size_t(nR) * p->esize, true)) != DSPMV_OK) return bail(st);
    if ((st = dev_alloc(*p, &p->d_partR, size_t(nR) * p->esize, true)) != DSPMV_OK) return bail(st);
    if ((st = dev_alloc(*p, reinterpret_cast<void**>(&p->d_ticket), size_t(nR) * 4, true)) != DSPMV_OK)
        return bail(st);
    p->explicit_acc = opts.accumulate_mode == DSPMV_ACC_EXPLICIT_IN_END;
    p->unpack_fused = opts.unpack_mode == DSPMV_UNPACK_FUSED;
    if (opts.unpack_mode != DSPMV_UNPACK_COPY && !p->unpack_fused)
        return bail(fail(DSPMV_ERR_ARG, "bad unpack_mode"));
    if (opts.accumulate_mode != DSPMV_ACC_TICKET && !p->explicit_acc)
        return bail(fail(DSPMV_ERR_ARG, "bad accumulate_mode"));
    if (opts.pack_mode != DSPMV_PACK_GATHER && opts.pack_mode != DSPMV_PACK_ALIAS_IF_CONTIGUOUS)
        return bail(fail(DSPMV_ERR_ARG, "bad pack_mode"));
    if (p->explicit_acc && nR > 0 &&
        (st = dev_upload(*p, &p->d_ar_rows, h.ar_rows.data(), h.ar_rows.size())) != DSPMV_OK)
        return bail(st);
    if (!opts.keep_host) {
        std::vector<int32_t>().swap(h.al_rowptr);
        std::vector<int32_t>().swap(h.al_col);
        std::vector<uint8_t>().swap(h.al_val);
        std::vector<int32_t>().swap(h.ar_rowptr);
        std::vector<int32_t>().swap(h.ar_col);
        std::vector<uint8_t>().swap(h.ar_val);
    }

    // phase 2: request lists -> send counts + pack maps
    if (comm->kind == DSPMV_COMM_NCCL || comm->kind == DSPMV_COMM_HOST) {
        if (comm->kind == DSPMV_COMM_HOST && !p->put_mode && !p->skip_exchange)
            return bail(fail(DSPMV_ERR_ARG, "plans on a HOST comm need exchange = DSPMV_EXCHANGE_PUT"));
        st = comm->kind == DSPMV_COMM_NCCL ? exchange_requests_nccl(*p) : exchange_requests_allgather(*p);
        if (st != DSPMV_OK) return bail(st);
        if ((st = finalize_send(*p)) != DSPMV_OK) return bail(st);
        if (opts.debug_checks) {   // COLLECTIVE arguments agree across ranks
            const int64_t key[6] = {n_global, comm->nranks, opts.dtype, opts.exchange, opts.pack_mode,
                                    opts.accumulate_mode};
            bool same = true;
            if ((st = ranks_agree(*p, fnv1a(key, sizeof(key)), &same)) != DSPMV_OK) return bail(st);
            if (!same) return bail(fail(DSPMV_ERR_ARG, "debug check: plan_create arguments differ across ranks"));
        }
        if (p->put_mode && comm->nranks > 1 && (st = setup_put_nccl(*p)) != DSPMV_OK) return bail(st);
    } else {
        LocalGroup& g = *comm->group;
        g.plans[comm->rank] = p;
        g.registered++;
        if (g.registered == g.nranks) {
            if ((st = finalize_local_group(g)) != DSPMV_OK) {
                g.plans[comm->rank] = nullptr;
                g.registered--;
                return bail(st);
            }
        }
    }
    CUDA_TRY(cudaDeviceSynchronize());
    comm->live_plans++;
    *out = p;
    return DSPMV_OK;
}

dspmv_status dspmv_plan_destroy(dspmv_plan_t plan) {
    if (!plan) return fail(DSPMV_ERR_ARG, "null plan");
    if (plan->live_scheds > 0) return fail(DSPMV_ERR_STATE, "plan still has live schedules");
    cudaSetDevice(plan->device);
    cudaDeviceSynchronize();
    free_plan_device(*plan);
    if (plan->comm->kind == DSPMV_COMM_LOCAL) {
        LocalGroup& g = *plan->comm->group;
        if (g.plans[plan->comm->rank] == plan) {
            g.plans[plan->comm->rank] = nullptr;
            g.registered--;
        }
    }
    plan->comm->live_plans--;
    delete plan;
    return DSPMV_OK;
}

static void fill_info(const RankPlan& h, dspmv_plan_info* o) {
    std::memset(o, 0, sizeof(*o));
    o->n_global = h.n_global;
    o->row_begin = h.row_begin;
    o->row_end = h.row_end;
    o->n_remote_rows = int64_t(h.ar_rows.size());
    o->n_halo = int64_t(h.halo_gid.size());
    o->n_send = int64_t(h.pack_map.size());
    for (int q = 0; q < h.nranks; ++q) {
        o->n_recv_peers += h.recv_count[q] > 0;
        if (!h.send_count.empty()) o->n_send_peers += h.send_count[q] > 0;
    }
    o->rank = h.rank;
    o->nranks = h.nranks;
    o->dtype = h.esize == 4 ? DSPMV_F32 : DSPMV_F64;
}

dspmv_status dspmv_plan_info_get(dspmv_plan_t plan, dspmv_plan_info* out) {
    if (!plan || !out) return fail(DSPMV_ERR_ARG, "null argument");
    fill_info(plan->host, out);
    out->nnz_local = plan->nnz_L;
    out->nnz_remote = plan->nnz_R;
    out->n_blocks_local = plan->L.nb;
    out->n_vrows_local = plan->L.nV;
    out->n_blocks_remote = plan->R.nb;
    out->n_vrows_remote = plan->R.nV;
    out->grid_local = plan->L.grid_s;
    out->grid_remote = plan->R.grid_s;
    out->ready = plan->ready;
    out->device_bytes = plan->device_bytes;
    auto skern = [](const DevLayout& D) {
        return D.sell ? DSPMV_SKERNEL_SELL
                      : D.stream ? (D.stream_tma ? DSPMV_SKERNEL_STREAM_TMA : DSPMV_SKERNEL_STREAM) : DSPMV_SKERNEL_BLOCK;
    };
    out->s_kernel_local = skern(plan->L);
    out->s_kernel_remote = skern(plan->R);
    out->pack_alias = plan->pack_alias ? 1 : 0;
    out->unpack_fused = plan->unpack_fused ? 1 : 0;
    out->accumulate_mode = plan->explicit_acc ? DSPMV_ACC_EXPLICIT_IN_END : DSPMV_ACC_TICKET;
    return DSPMV_OK;
}

static dspmv_status export_array(const RankPlan& h, int what, void* dst, size_t bytes, size_t* needed,
                                 bool have_split) {
    const void* src = nullptr;
    size_t n = 0;
    auto pick = [&](const auto& v) {
        src = v.data();
        n = v.size() * sizeof(v[0]);
    };
    switch (what) {
        case DSPMV_HALO_GID: pick(h.halo_gid); break;
        case DSPMV_RECV_COUNTS: pick(h.recv_count); break;
        case DSPMV_RECV_DISPL: pick(h.recv_displ); break;
        case DSPMV_SEND_COUNTS: pick(h.send_count); break;
        case DSPMV_SEND_DISPL: pick(h.send_displ); break;
        case DSPMV_PACK_MAP: pick(h.pack_map); break;
        case DSPMV_AR_ROWS: pick(h.ar_rows); break;
        case DSPMV_AL_ROWPTR: case DSPMV_AL_COL: case DSPMV_AR_ROWPTR: case DSPMV_AR_COL:
        case DSPMV_AL_VAL: case DSPMV_AR_VAL:
            if (!have_split) return fail(DSPMV_ERR_STATE, "split arrays not kept (opts.keep_host = 0)");
            if (what == DSPMV_AL_ROWPTR) pick(h.al_rowptr);
            else if (what == DSPMV_AL_COL) pick(h.al_col);
            else if (what == DSPMV_AR_ROWPTR) pick(h.ar_rowptr);
            else if (what == DSPMV_AR_COL) pick(h.ar_col);
            else if (what == DSPMV_AL_VAL) pick(h.al_val);
            else pick(h.ar_val);
            break;
        default:
            return fail(DSPMV_ERR_ARG, "unknown export id");
    }
    if (needed) *needed = n;
    if (!dst) return DSPMV_OK;
    if (bytes < n) return fail(DSPMV_ERR_ARG, "destination too small");
    if (n) std::memcpy(dst, src, n);
    return DSPMV_OK;
}

dspmv_status dspmv_plan_export(dspmv_plan_t plan, int what, void* host_dst, size_t bytes, size_t* needed) {
    if (!plan) return fail(DSPMV_ERR_ARG, "null plan");
    if (!plan->ready && (what == DSPMV_SEND_COUNTS || what == DSPMV_SEND_DISPL || what == DSPMV_PACK_MAP))
        return fail(DSPMV_ERR_STATE, "plan not ready");
    return export_array(plan->host, what, host_dst, bytes, needed, plan->opts.keep_host != 0);
}

dspmv_status dspmv_plan_build_host(int nranks, int64_t n_global, const int64_t* rowptr_global,
                                   const int32_t* col_global, const void* val_global, int dtype,
                                   dspmv_host_plan_t* out) {
    if (!out || nranks < 1 || n_global < 0 || (n_global > 0 && !rowptr_global))
        return fail(DSPMV_ERR_ARG, "bad arguments");
    if (dtype != DSPMV_F64 && dtype != DSPMV_F32) return fail(DSPMV_ERR_ARG, "bad dtype");
    auto* hp = new dspmv_host_plan_s();
    hp->esize = dtype == DSPMV_F32 ? 4 : 8;
    hp->has_val = val_global != nullptr;
    hp->ranks.resize(nranks);
    const auto rb = partition(n_global, nranks);
    for (int r = 0; r < nranks; ++r) {
        const uint8_t* v = val_global ? static_cast<const uint8_t*>(val_global) : nullptr;
        // the rank's rows: rowptr slice; col/val are addressed relative to rowptr[0]
        const int64_t b = rb[r], nl = rb[r + 1] - rb[r];
        const int64_t off = n_global > 0 ? rowptr_global[b] : 0;
        dspmv_status st = plan_phase1(n_global, nranks, r, nl, n_global > 0 ? rowptr_global + b : nullptr,
                                      col_global ? col_global + off : nullptr,
                                      v ? v + size_t(off) * hp->esize : nullptr, hp->esize, hp->ranks[r]);
        if (st != DSPMV_OK) {
            delete hp;
            return st;
        }
    }
    for (int p = 0; p < nranks; ++p) {
        std::vector<std::vector<int32_t>> req(nranks);
        for (int r = 0; r < nranks; ++r) req[r] = halo_segment_for(hp->ranks[r], p);
        plan_phase2_from_requests(hp->ranks[p], req);
    }
    *out = hp;
    return DSPMV_OK;
}

dspmv_status dspmv_host_plan_info(dspmv_host_plan_t hp, int rank, dspmv_plan_info* out) {
    if (!hp || !out || rank < 0 || rank >= int(hp->ranks.size())) return fail(DSPMV_ERR_ARG, "bad arguments");
    const RankPlan& h = hp->ranks[rank];
    fill_info(h, out);
    out->nnz_local = int64_t(h.al_col.size());
    out->nnz_remote = int64_t(h.ar_col.size());
    out->ready = 1;
    std::vector<int64_t> off;
    out->pack_alias = pack_alias_offsets(h, off) ? 1 : 0;   // would ALIAS_IF_CONTIGUOUS alias?
    return DSPMV_OK;
}

dspmv_status dspmv_host_plan_export(dspmv_host_plan_t hp, int rank, int what, void* dst, size_t bytes,
                                    size_t* needed) {
    if (!hp || rank < 0 || rank >= int(hp->ranks.size())) return fail(DSPMV_ERR_ARG, "bad arguments");
    if ((what == DSPMV_AL_VAL || what == DSPMV_AR_VAL) && !hp->has_val)
        return fail(DSPMV_ERR_STATE, "host plan built without values");
    return export_array(hp->ranks[rank], what, dst, bytes, needed, true);
}

dspmv_status dspmv_rank_plan_build_host(int nranks, int rank, int64_t n_global, int64_t n_local,
                                        const int64_t* rowptr, const int32_t* col_global, const void* val,
                                        int dtype, dspmv_host_plan_t* out) {
    if (!out) return fail(DSPMV_ERR_ARG, "null out");
    if (dtype != DSPMV_F64 && dtype != DSPMV_F32) return fail(DSPMV_ERR_ARG, "bad dtype");
    auto* hp = new dspmv_host_plan_s();
    hp->esize = dtype == DSPMV_F32 ? 4 : 8;
    hp->has_val = val != nullptr;
    hp->ranks.resize(1);
    dspmv_status st = plan_phase1(n_global, nranks, rank, n_local, rowptr, col_global, val, hp->esize, hp->ranks[0]);
    if (st != DSPMV_OK) {
        delete hp;
        return st;
    }
    *out = hp;
    return DSPMV_OK;
}

dspmv_status dspmv_host_plan_requests(dspmv_host_plan_t hp, int owner, int32_t* dst, size_t cap, size_t* count) {
    if (!hp || hp->ranks.size() != 1) return fail(DSPMV_ERR_ARG, "need a one-rank host plan");
    const RankPlan& h = hp->ranks[0];
    if (owner < 0 || owner >= h.nranks) return fail(DSPMV_ERR_ARG, "bad owner");
    const size_t n = size_t(h.recv_count[owner]);
    if (count) *count = n;
    if (!dst) return DSPMV_OK;
    if (cap < n) return fail(DSPMV_ERR_ARG, "destination too small");
    std::memcpy(dst, h.halo_gid.data() + h.recv_displ[owner], n * 4);
    return DSPMV_OK;
}

dspmv_status dspmv_host_plan_set_requests(dspmv_host_plan_t hp, const int32_t* const* lists, const int32_t* counts) {
    if (!hp || hp->ranks.size() != 1 || !counts) return fail(DSPMV_ERR_ARG, "need a one-rank host plan");
    RankPlan& h = hp->ranks[0];
    std::vector<std::vector<int32_t>> req(h.nranks);
    for (int r = 0; r < h.nranks; ++r) {
        if (counts[r] < 0 || (counts[r] > 0 && (!lists || !lists[r]))) return fail(DSPMV_ERR_ARG, "bad request list");
        req[r].assign(lists ? lists[r] : nullptr, lists ? lists[r] + counts[r] : nullptr);
        for (int32_t g : req[r])
            if (g < h.row_begin || g >= h.row_end)
                return fail(DSPMV_ERR_ARG, "rank " + std::to_string(r) + " requested id " + std::to_string(g) +
                                               " not owned by this rank");
    }
    plan_phase2_from_requests(h, req);
    return DSPMV_OK;
}

dspmv_status dspmv_layout_host(const int64_t* rowptr, int32_t nrows, int dtype, int cfg, int vthr, int32_t* s_rows,
                               int32_t* n_s, int32_t* desc, int32_t* n_blocks, int32_t* v_rows, int32_t* n_v,
                               int32_t* cfg_used) {
    if (!rowptr || nrows < 0 || !n_s || !n_blocks || !n_v) return fail(DSPMV_ERR_ARG, "null argument");
    const int esize = dtype == DSPMV_F32 ? 4 : 8;
    if (vthr < 0) vthr = kDefaultVectorThreshold;
    std::vector<int32_t> rp(static_cast<size_t>(nrows) + 1);
    for (int32_t i = 0; i <= nrows; ++i) {
        const int64_t v = rowptr[i] - rowptr[0];
        if (v >= (int64_t(1) << 31)) return fail(DSPMV_ERR_RANGE, "nnz >= 2^31");
        rp[i] = int32_t(v);
    }
    const int c = cfg >= 0 ? cfg : auto_block_cfg(rp.data(), nrows, vthr, esize);
    if (c < 0 || c >= kNumBlockCfgs || vthr > kBlockCfgs[c].tile) return fail(DSPMV_ERR_ARG, "bad cfg / vthr");
    std::vector<int32_t> col(size_t(rp[nrows]), 0);
    std::vector<int32_t> ident(static_cast<size_t>(nrows));
    for (int32_t i = 0; i < nrows; ++i) ident[i] = i;
    Layout L;
    build_layout(rp.data(), nrows, col.data(), nullptr, esize, ident.data(), nullptr, vthr, kBlockCfgs[c], L);
    const bool fit = (!s_rows || *n_s >= L.nS) && (!desc || *n_blocks >= L.nb) && (!v_rows || *n_v >= L.nV);
    if (s_rows && fit) std::copy(L.s_out.begin(), L.s_out.end(), s_rows);
    if (desc && fit) std::copy(L.s_desc.begin(), L.s_desc.end(), desc);
    if (v_rows && fit) std::copy(L.v_out.begin(), L.v_out.end(), v_rows);
    *n_s = L.nS;
    *n_blocks = L.nb;
    *n_v = L.nV;
    if (cfg_used) *cfg_used = c;
    if (!fit) return fail(DSPMV_ERR_ARG, "output arrays too small");
    return DSPMV_OK;
}

dspmv_status dspmv_sell_layout_host(const int64_t* rowptr, int32_t nrows, int vthr, int window,
                                    int32_t* slice_base, int32_t* lane_row, int32_t* lane_len,
                                    int32_t* entry_src, int32_t* chunks, int32_t* n_slices,
                                    int64_t* n_entries, int32_t* n_chunks) {
    if (!rowptr || nrows < 0 || !n_slices || !n_entries || !n_chunks) return fail(DSPMV_ERR_ARG, "null argument");
    if (vthr < 0) vthr = kDefaultVectorThreshold;
    if (window == 0 || window < -1) return fail(DSPMV_ERR_ARG, "window must be -1 or > 0");
    std::vector<int32_t> rp(static_cast<size_t>(nrows) + 1);
    for (int32_t i = 0; i <= nrows; ++i) {
        const int64_t v = rowptr[i] - rowptr[0];
        if (v >= (int64_t(1) << 31)) return fail(DSPMV_ERR_RANGE, "nnz >= 2^31");
        rp[i] = int32_t(v);
    }
    // col[q] = q: the stored col array then is each entry's CSR position
    std::vector<int32_t> col(size_t(rp[nrows])), ident(static_cast<size_t>(nrows));
    for (size_t q = 0; q < col.size(); ++q) col[q] = int32_t(q);
    for (int32_t i = 0; i < nrows; ++i) ident[i] = i;
    Layout L;
    build_layout(rp.data(), nrows, col.data(), nullptr, 8, ident.data(), nullptr, vthr,
                 kBlockCfgs[kDefaultBlockCfg], L, true, true, window > 0 ? window : 0);
    const int32_t ns = int32_t(L.sl_base.size()) - 1, nc = int32_t(L.sl_chunk.size()) - 1;
    const int64_t ne = L.sl_base.back();
    const bool fit = !slice_base || (*n_slices >= ns && *n_entries >= ne && *n_chunks >= nc);
    if (slice_base && fit) {
        std::copy(L.sl_base.begin(), L.sl_base.end(), slice_base);
        if (lane_row) std::copy(L.sl_srow.begin(), L.sl_srow.end(), lane_row);
        if (lane_len) std::copy(L.sl_len.begin(), L.sl_len.end(), lane_len);
        // S-group CSR position of each stored entry: the S rows' entries back to back
        if (entry_src) {
            std::vector<int32_t> spos(col.size(), -1);
            for (int64_t q = 0; q < int64_t(L.s_rowptr[L.nS]); ++q) spos[size_t(L.s_col[size_t(q)])] = int32_t(q);
            for (int64_t q = 0; q < ne; ++q) entry_src[q] = spos[size_t(L.sl_col[size_t(q)])];
        }
        if (chunks) std::copy(L.sl_chunk.begin(), L.sl_chunk.end(), chunks);
    }
    *n_slices = ns;
    *n_entries = ne;
    *n_chunks = nc;
    if (!fit) return fail(DSPMV_ERR_ARG, "output arrays too small");
    return DSPMV_OK;
}

dspmv_status dspmv_stream_layout_host(const int64_t* rowptr, int32_t nrows, int vthr, int s_kernel,
                                      int32_t* tiles, int32_t* n_tiles, int32_t* v_rows, int32_t* n_v,
                                      int32_t* stream_used) {
    if (!rowptr || nrows < 0 || !n_tiles || !n_v) return fail(DSPMV_ERR_ARG, "null argument");
    if (vthr < 0) vthr = kDefaultVectorThreshold;
    std::vector<int32_t> rp(static_cast<size_t>(nrows) + 1);
    for (int32_t i = 0; i <= nrows; ++i) {
        const int64_t v = rowptr[i] - rowptr[0];
        if (v >= (int64_t(1) << 31)) return fail(DSPMV_ERR_RANGE, "nnz >= 2^31");
        rp[i] = int32_t(v);
    }
    dspmv_plan_opts o;
    dspmv_plan_opts_default(&o);
    o.s_kernel = s_kernel;
    std::vector<int32_t> col(size_t(rp[nrows]), 0), ident(static_cast<size_t>(nrows));
    for (int32_t i = 0; i < nrows; ++i) ident[i] = i;
    Layout L;
    build_layout(rp.data(), nrows, col.data(), nullptr, 8, ident.data(), nullptr, vthr,
                 kBlockCfgs[kDefaultBlockCfg], L, true);
    const int32_t nt = int32_t(L.s_tiles.size() / 2);
    const bool fit = (!tiles || *n_tiles >= nt) && (!v_rows || *n_v >= L.nV);
    if (tiles && fit) std::copy(L.s_tiles.begin(), L.s_tiles.end(), tiles);
    if (v_rows && fit) std::copy(L.v_out.begin(), L.v_out.end(), v_rows);
    *n_tiles = nt;
    *n_v = L.nV;
    if (stream_used) *stream_used = use_stream(o, rp.data(), nrows, vthr) ? 1 : 0;
    if (!fit) return fail(DSPMV_ERR_ARG, "output arrays too small");
    return DSPMV_OK;
}

dspmv_status dspmv_host_plan_destroy(dspmv_host_plan_t hp) {
    if (!hp) return fail(DSPMV_ERR_ARG, "null host plan");
    delete hp;
    return DSPMV_OK;
}

// ------------------------------------------------------------- schedules
dspmv_status dspmv_schedule_create(dspmv_plan_t plan, const dspmv_op* ops, int n_ops, int n_streams,
                                   dspmv_schedule_t* out) {
    if (!plan || !out) return fail(DSPMV_ERR_ARG, "null plan/out");
    SchedCheck c = validate_schedule(ops, n_ops, n_streams);
    if (c.st != DSPMV_OK) return fail(c.st, c.why);
    CUDA_TRY(cudaSetDevice(plan->device));
    auto* s = new dspmv_schedule_s();
    s->plan = plan;
    s->ops.assign(ops, ops + n_ops);
    s->n_streams = n_streams;
    s->dag = std::move(c.dag);
    for (const dspmv_op& o : s->ops) {
        if (o.kind == DSPMV_OP_EVENT_RECORD && !s->ev[o.event]) {
            if (cudaEventCreateWithFlags(&s->ev[o.event], cudaEventDisableTiming) != cudaSuccess) {
                for (auto& e : s->ev)
                    if (e) cudaEventDestroy(e);
                delete s;
                return fail(DSPMV_ERR_CUDA, "cudaEventCreate failed");
            }
        }
    }
    // per-destination coverage is checked here when the plan is ready (a LOCAL
    // rank's plan becomes ready when the whole group has planned: then at the
    // first apply)
    if (plan->ready) {
        const dspmv_status cs = compile_exchange(*s);
        if (cs != DSPMV_OK) {
            std::string keep = t_err;
            for (auto& e : s->ev)
                if (e) cudaEventDestroy(e);
            for (auto& g : s->groups)
                if (g.ev) cudaEventDestroy(g.ev);
            delete s;
            t_err = keep;
            return cs;
        }
    }
    plan->live_scheds++;
    *out = s;
    return DSPMV_OK;
}

static void destroy_timing(Schedule& s) {
    if (s.step0) cudaEventDestroy(s.step0), s.step0 = nullptr;
    if (s.step1) cudaEventDestroy(s.step1), s.step1 = nullptr;
    for (auto e : s.t0)
        if (e) cudaEventDestroy(e);
    for (auto e : s.t1)
        if (e) cudaEventDestroy(e);
    s.t0.clear();
    s.t1.clear();
}

dspmv_status dspmv_schedule_destroy(dspmv_schedule_t s) {
    if (!s) return fail(DSPMV_ERR_ARG, "null schedule");
    cudaSetDevice(s->plan->device);
    // a group graph references every member's events: a member going away
    // drops the leader's graph (re-captured on the next group apply), a
    // leader going away releases its members
    if (Schedule* L = s->g_leader) {
        if (L->gexec) cudaGraphExecDestroy(L->gexec), L->gexec = nullptr;
        for (Schedule* m : L->g_group)
            if (m != L) m->g_leader = nullptr;
        L->g_group.clear();
        L->g_group_ptrs.clear();
    }
    for (Schedule* m : s->g_group)
        if (m != s) m->g_leader = nullptr;
    if (s->gexec) cudaGraphExecDestroy(s->gexec);
    for (auto& e : s->gev)
        if (e) cudaEventDestroy(e);
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    for (auto& g : s->groups)
        if (g.ev) cudaEventDestroy(g.ev);
    destroy_timing(*s);
    s->plan->live_scheds--;
    delete s;
    return DSPMV_OK;
}

dspmv_status dspmv_schedule_set_caller_stream0(dspmv_schedule_t s, int mode) {
    if (!s) return fail(DSPMV_ERR_ARG, "null schedule");
    if (mode < -1 || mode > 1) return fail(DSPMV_ERR_ARG, "mode must be -1, 0 or 1");
    if (s->caller_stream0 != mode && s->gexec) {
        CUDA_TRY(cudaSetDevice(s->plan->device));
        cudaGraphExecDestroy(s->gexec);   // captured with the other stream binding
        s->gexec = nullptr;
    }
    s->caller_stream0 = mode;
    return DSPMV_OK;
}

dspmv_status dspmv_schedule_set_timing(dspmv_schedule_t s, int enable) {
    if (!s) return fail(DSPMV_ERR_ARG, "null schedule");
    CUDA_TRY(cudaSetDevice(s->plan->device));
    destroy_timing(*s);
    if (s->gexec) cudaGraphExecDestroy(s->gexec), s->gexec = nullptr;  // captured the old events
    s->timing = enable != 0;
    s->timed_valid = false;
    if (s->timing) {
        s->t0.assign(s->ops.size(), nullptr);
        s->t1.assign(s->ops.size(), nullptr);
        s->t0_alias.assign(s->ops.size(), 0);
        s->g_t0_alias.assign(s->ops.size(), 0);
        s->end_alias = s->g_end_alias = -1;
        // enable == 1: every GPU vertex; otherwise a bit mask (1 << kind)
        const unsigned mask = enable == 1 ? ~0u : unsigned(enable);
        if (mask & 1u) {  // bit of START: whole apply, START..END on the caller stream
            CUDA_TRY(cudaEventCreate(&s->step0));
            CUDA_TRY(cudaEventCreate(&s->step1));
        }
        for (size_t t = 0; t < s->ops.size(); ++t) {
            const int k = s->ops[t].kind;
            const bool post = k == DSPMV_OP_POST_SEND || k == DSPMV_OP_POST_RECV;
            if (!(is_gpu_vertex(k) || post) || !(mask & (1u << k))) continue;
            CUDA_TRY(cudaEventCreate(&s->t0[t]));
            CUDA_TRY(cudaEventCreate(&s->t1[t]));
        }
    }
    return DSPMV_OK;
}

dspmv_status dspmv_schedule_op_times(dspmv_schedule_t s, float* ms, int n) {
    if (!s || !ms) return fail(DSPMV_ERR_ARG, "null argument");
    if (!s->timing || !s->timed_valid) return fail(DSPMV_ERR_STATE, "timing not enabled or no apply yet");
    if (s->step1) CUDA_TRY(cudaEventSynchronize(s->end_event()));  // recorded at END, may still be queued
    for (int t = 0; t < n && t < int(s->ops.size()); ++t) {
        ms[t] = 0.f;
        if (s->t0[t]) CUDA_TRY(cudaEventElapsedTime(&ms[t], s->begin_event(t), s->t1[t]));
    }
    if (s->step0 && n > 0) CUDA_TRY(cudaEventElapsedTime(&ms[0], s->step0, s->end_event()));
    return DSPMV_OK;
}

dspmv_status dspmv_schedule_op_timeline(dspmv_schedule_t s, float* begin_ms, float* end_ms, int n) {
    if (!s || !begin_ms || !end_ms) return fail(DSPMV_ERR_ARG, "null argument");
    if (!s->timing || !s->timed_valid || !s->step0)
        return fail(DSPMV_ERR_STATE, "timeline needs timing with the START bit and an apply");
    CUDA_TRY(cudaEventSynchronize(s->end_event()));
    for (int t = 0; t < n && t < int(s->ops.size()); ++t) {
        begin_ms[t] = end_ms[t] = -1.f;
        if (s->t0[t]) {
            if (s->t0_alias[t]) begin_ms[t] = 0.f;
            else CUDA_TRY(cudaEventElapsedTime(&begin_ms[t], s->step0, s->t0[t]));
            CUDA_TRY(cudaEventElapsedTime(&end_ms[t], s->step0, s->t1[t]));
        }
    }
    if (n > 0) {
        begin_ms[0] = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&end_ms[0], s->step0, s->end_event()));
    }
    return DSPMV_OK;
}

// ----------------------------------------------------------------- apply
dspmv_status dspmv_apply(dspmv_schedule_t s, const void* x, void* y, dspmv_stream_t stream) {
    if (!s) return fail(DSPMV_ERR_ARG, "null schedule");
    Plan& p = *s->plan;
    if (p.comm->kind == DSPMV_COMM_LOCAL && p.host.nranks > 1)
        return fail(DSPMV_ERR_ARG, "LOCAL groups with >1 rank use dspmv_apply_group");
    if (p.host.n_local() > 0 && (!x || !y)) return fail(DSPMV_ERR_ARG, "null x/y");
    ST_TRY(check_schedule_hash(*s));
    NvtxScope nvtx_scope(nvtx_on(), "dspmv_apply rank " + std::to_string(p.host.rank));
    ST_TRY(begin_apply(*s, static_cast<cudaStream_t>(stream)));
    p.cur_x = x;
    const bool local = p.comm->kind == DSPMV_COMM_LOCAL;
    for (int t = 0; t < int(s->ops.size()); ++t) {
        ST_TRY(exec_op(*s, t, x, y, local));
        const int gi = s->op_group[t];
        if (local && gi >= 0 && s->groups[gi].ps && s->groups[gi].pr && !s->groups[gi].issued)
            ST_TRY(issue_group_local({s}, gi));
    }
    ST_TRY(end_combine(*s, y, static_cast<cudaStream_t>(stream)));
    if (s->step1) CUDA_TRY(cudaEventRecord(s->step1, static_cast<cudaStream_t>(stream)));
    s->timed_valid = s->timing;
    return DSPMV_OK;
}

dspmv_status dspmv_apply_graph(dspmv_schedule_t s, const void* x, void* y, dspmv_stream_t stream) {
    if (!s) return fail(DSPMV_ERR_ARG, "null schedule");
    Plan& p = *s->plan;
    if (p.poisoned) return fail(DSPMV_ERR_STATE, "plan is poisoned by an earlier error");
    if (!p.ready) return fail(DSPMV_ERR_STATE, "plan not ready");
    if (p.host.n_local() > 0 && (!x || !y)) return fail(DSPMV_ERR_ARG, "null x/y");
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != p.device) CUDA_TRY(cudaSetDevice(p.device));
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (!cs) return fail(DSPMV_ERR_ARG, "apply_graph needs a non-default stream");
    ST_TRY(check_schedule_hash(*s));
    NvtxScope nvtx_scope(nvtx_on(), "dspmv_apply_graph rank " + std::to_string(p.host.rank));
    if (!s->gexec || !s->g_group.empty() || s->gx != x || s->gy != y || s->g_timing != s->timing)
        ST_TRY(capture_graph(*s, x, y, cs));
    const cudaError_t e = cudaGraphLaunch(s->gexec, cs);
    if (e != cudaSuccess) {
        p.poisoned = true;
        return fail(DSPMV_ERR_CUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
    }
    if (p.d_epoch) ++p.epoch;   // the graph bumped the device copy (keeps host-mode applies in step)
    g_launches.fetch_add(s->graph_kernels, std::memory_order_relaxed);
    if (s->timing) {
        s->t0_alias = s->g_t0_alias;
        s->end_alias = s->g_end_alias;
    }
    s->timed_valid = s->timing;
    return DSPMV_OK;
}

dspmv_status dspmv_apply_graph_group(const dspmv_schedule_t* scheds, int nranks, const void* const* x,
                                     void* const* y, dspmv_stream_t stream) {
    if (!scheds || nranks < 1 || !x || !y) return fail(DSPMV_ERR_ARG, "null argument");
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (!cs) return fail(DSPMV_ERR_ARG, "apply_graph_group needs a non-default stream");
    std::vector<Schedule*> ss(nranks);
    std::vector<const void*> xs(x, x + nranks);
    std::vector<void*> ys(y, y + nranks);
    for (int r = 0; r < nranks; ++r) {
        if (!scheds[r]) return fail(DSPMV_ERR_ARG, "null schedule");
        Plan* p = scheds[r]->plan;
        if (p->comm->kind != DSPMV_COMM_LOCAL || p->comm->nranks != nranks || p->comm->rank != r)
            return fail(DSPMV_ERR_ARG, "schedules must be ranks 0..n-1 of one LOCAL group");
        if (r > 0 && p->comm->group != scheds[0]->plan->comm->group) return fail(DSPMV_ERR_ARG, "mixed groups");
        if (scheds[r]->ops.size() != scheds[0]->ops.size() ||
            std::memcmp(scheds[r]->ops.data(), scheds[0]->ops.data(), sizeof(dspmv_op) * scheds[0]->ops.size()))
            return fail(DSPMV_ERR_ARG, "every rank must run the same schedule (P:460)");
        if (p->poisoned) return fail(DSPMV_ERR_STATE, "plan is poisoned by an earlier error");
        if (!p->ready) return fail(DSPMV_ERR_STATE, "plan not ready");
        if (p->host.n_local() > 0 && (!x[r] || !y[r])) return fail(DSPMV_ERR_ARG, "null x/y");
        ss[r] = scheds[r];
    }
    Schedule& s0 = *ss[0];
    CUDA_TRY(cudaSetDevice(s0.plan->device));
    bool fresh = s0.gexec && s0.g_group.size() == size_t(nranks);
    for (int r = 0; fresh && r < nranks; ++r)
        fresh = s0.g_group[r] == ss[r] && s0.g_group_ptrs[2 * r] == x[r] && s0.g_group_ptrs[2 * r + 1] == y[r] &&
                ss[r]->g_timing == ss[r]->timing;
    if (!fresh) {
        s0.g_group_ptrs.clear();
        ST_TRY(capture_graph(ss, xs, ys, cs));
    }
    const cudaError_t e = cudaGraphLaunch(s0.gexec, cs);
    if (e != cudaSuccess) {
        for (Schedule* sp : ss) sp->plan->poisoned = true;
        return fail(DSPMV_ERR_CUDA, std::string("cudaGraphLaunch: ") + cudaGetErrorString(e));
    }
    g_launches.fetch_add(s0.graph_kernels, std::memory_order_relaxed);
    for (Schedule* sp : ss) {
        ++sp->plan->epoch;
        if (sp->timing) {
            sp->t0_alias = sp->g_t0_alias;
            sp->end_alias = sp->g_end_alias;
        }
        sp->timed_valid = sp->timing;
    }
    return DSPMV_OK;
}

dspmv_status dspmv_apply_graph_prepare(dspmv_schedule_t s, const void* x, void* y, dspmv_stream_t stream) {
    if (!s) return fail(DSPMV_ERR_ARG, "null schedule");
    Plan& p = *s->plan;
    if (p.poisoned) return fail(DSPMV_ERR_STATE, "plan is poisoned by an earlier error");
    if (!p.ready) return fail(DSPMV_ERR_STATE, "plan not ready");
    if (p.host.n_local() > 0 && (!x || !y)) return fail(DSPMV_ERR_ARG, "null x/y");
    CUDA_TRY(cudaSetDevice(p.device));
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (!cs) return fail(DSPMV_ERR_ARG, "apply_graph needs a non-default stream");
    if (!s->gexec || !s->g_group.empty() || s->gx != x || s->gy != y || s->g_timing != s->timing)
        ST_TRY(capture_graph(*s, x, y, cs));
    return DSPMV_OK;
}

static bool pinned_host(const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

dspmv_status dspmv_apply_host(dspmv_schedule_t s, const void* x_host, void* y_host, dspmv_stream_t stream) {
    if (!s) return fail(DSPMV_ERR_ARG, "null schedule");
    Plan& p = *s->plan;
    const size_t bytes = size_t(p.host.n_local()) * p.esize;
    if (bytes && (!x_host || !y_host)) return fail(DSPMV_ERR_ARG, "null x/y");
    CUDA_TRY(cudaSetDevice(p.device));
    if (bytes && !p.d_xin) {
        ST_TRY(dev_alloc(p, &p.d_xin, bytes, false));
        ST_TRY(dev_alloc(p, &p.d_yout, bytes, false));
    }
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    auto& H = p.pipe;
    if (!bytes || H.K == 0 || !pinned_host(x_host) || !pinned_host(y_host)) {
        // one transfer each way around the apply
        if (bytes) CUDA_TRY(cudaMemcpyAsync(p.d_xin, x_host, bytes, cudaMemcpyHostToDevice, cs));
        ST_TRY(dspmv_apply(s, p.d_xin, p.d_yout, stream));
        if (bytes) CUDA_TRY(cudaMemcpyAsync(y_host, p.d_yout, bytes, cudaMemcpyDeviceToHost, cs));
        CUDA_TRY(cudaStreamSynchronize(cs));
        return DSPMV_OK;
    }
    // pinned x/y: x goes over in K chunks on a copy stream and y_L runs group
    // by group right behind it; the kernels store y straight into the mapped
    // host buffer (zero-copy), so no device-to-host copy follows and the one
    // copy engine in use never shares PCIe with a second transfer direction
    void* y_map = nullptr;
    if (cudaHostGetDevicePointer(&y_map, y_host, 0) != cudaSuccess || !y_map) {
        cudaGetLastError();
        if (bytes) CUDA_TRY(cudaMemcpyAsync(p.d_xin, x_host, bytes, cudaMemcpyHostToDevice, cs));
        ST_TRY(dspmv_apply(s, p.d_xin, p.d_yout, stream));
        if (bytes) CUDA_TRY(cudaMemcpyAsync(y_host, p.d_yout, bytes, cudaMemcpyDeviceToHost, cs));
        CUDA_TRY(cudaStreamSynchronize(cs));
        return DSPMV_OK;
    }
    auto wv = write_value32();
    if (!wv) return fail(DSPMV_ERR_CUDA, "cuStreamWriteValue32 unavailable");
    if (!H.h2d) {
        ST_TRY(dev_alloc(p, reinterpret_cast<void**>(&H.d_xflag), size_t(H.K) * 4, true));
        CUDA_TRY(cudaStreamCreateWithFlags(&H.h2d, cudaStreamNonBlocking));
        H.ev_x.assign(H.K, nullptr);
        for (auto& e : H.ev_x) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&H.ev_in, cudaEventDisableTiming));
    }
    if (H.pack_chunk == -1) {
        H.pack_chunk = -2;                               // no Pack reads of x
        if (!p.host.pack_map.empty()) {
            const int32_t mx = *std::max_element(p.host.pack_map.begin(), p.host.pack_map.end());
            H.pack_chunk = int(std::upper_bound(H.x_chunk.begin(), H.x_chunk.end(), int64_t(mx)) - H.x_chunk.begin()) - 1;
        }
    }
    CUDA_TRY(cudaEventRecord(H.ev_in, cs));              // after prior work on the caller stream
    CUDA_TRY(cudaStreamWaitEvent(H.h2d, H.ev_in, 0));
    const unsigned epoch = p.epoch + 1;                  // begin_apply's epoch of this apply
    for (int k = 0; k < H.K; ++k) {
        const size_t off = size_t(H.x_chunk[k]) * p.esize, len = size_t(H.x_chunk[k + 1] - H.x_chunk[k]) * p.esize;
        cudaStream_t q = H.h2d;
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(p.d_xin) + off, static_cast<const char*>(x_host) + off, len,
                                 cudaMemcpyHostToDevice, q));
        const CUresult r =
            wv(reinterpret_cast<CUstream>(q), reinterpret_cast<CUdeviceptr>(H.d_xflag + k), epoch, CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) return fail(DSPMV_ERR_CUDA, "cuStreamWriteValue32 failed (" + std::to_string(int(r)) + ")");
        CUDA_TRY(cudaEventRecord(H.ev_x[k], q));
    }
    if (H.ycopy) {
        // y leaves on the second copy engine, group by group, as the row
        // blocks of each x chunk finish (SM stores into host memory share
        // PCIe less well: profiles/r2_ubench_zerocopy.txt).  The counters are
        // cleared on the caller stream before the apply's kernels; the waits
        // and copies follow the y_L launch (enqueue_ycopy).
        auto wait = wait_value32();
        if (!wait) return fail(DSPMV_ERR_CUDA, "cuStreamWaitValue32 unavailable");
        if (!H.d2h) {
            ST_TRY(dev_alloc(p, reinterpret_cast<void**>(&H.d_ydone), size_t(H.K) * 4, true));
            CUDA_TRY(cudaStreamCreateWithFlags(&H.d2h, cudaStreamNonBlocking));
            CUDA_TRY(cudaEventCreateWithFlags(&H.ev_zero, cudaEventDisableTiming));
            CUDA_TRY(cudaEventCreateWithFlags(&H.ev_out, cudaEventDisableTiming));
        }
        CUDA_TRY(cudaMemsetAsync(H.d_ydone, 0, size_t(H.K) * 4, cs));   // before this apply's kernels
        CUDA_TRY(cudaEventRecord(H.ev_zero, cs));
        CUDA_TRY(cudaStreamWaitEvent(H.d2h, H.ev_zero, 0));
        H.y_host = y_host;   // the waits and copies are queued right after the y_L launch (enqueue_ycopy)
    }
    p.streaming = true;
    const dspmv_status st = dspmv_apply(s, p.d_xin, H.ycopy ? p.d_yout : y_map, stream);
    p.streaming = false;
    if (st != DSPMV_OK) {
        cudaStreamSynchronize(H.h2d);
        return st;
    }
    CUDA_TRY(cudaStreamWaitEvent(cs, H.ev_x[H.K - 1], 0));   // every H2D done before d_xin is reused
    if (H.ycopy) {
        if (!H.y_queued) return fail(DSPMV_ERR_STATE, "apply_host: the schedule launched no y_L");
        H.y_queued = false;
        // the last y copies; bounded wait (a kernel that died would leave the
        // copy stream parked on its counter)
        const auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            const cudaError_t q = cudaEventQuery(H.ev_out);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) return fail(DSPMV_ERR_CUDA, std::string("apply_host y copy: ") + cudaGetErrorString(q));
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60)) {
                p.poisoned = true;
                return fail(DSPMV_ERR_STATE, "apply_host: y copies did not complete within 60 s");
            }
        }
    }
    CUDA_TRY(cudaStreamSynchronize(cs));
    return DSPMV_OK;
}

dspmv_status dspmv_apply_group(const dspmv_schedule_t* scheds, int nranks, const void* const* x, void* const* y,
                               dspmv_stream_t stream) {
    if (!scheds || nranks < 1 || !x || !y) return fail(DSPMV_ERR_ARG, "null argument");
    std::vector<Plan*> plans(nranks);
    for (int r = 0; r < nranks; ++r) {
        if (!scheds[r]) return fail(DSPMV_ERR_ARG, "null schedule");
        Plan* p = scheds[r]->plan;
        if (p->comm->kind != DSPMV_COMM_LOCAL || p->comm->nranks != nranks || p->comm->rank != r)
            return fail(DSPMV_ERR_ARG, "schedules must be ranks 0..n-1 of one LOCAL group");
        if (r > 0 && p->comm->group != plans[0]->comm->group) return fail(DSPMV_ERR_ARG, "mixed groups");
        if (scheds[r]->ops.size() != scheds[0]->ops.size() ||
            std::memcmp(scheds[r]->ops.data(), scheds[0]->ops.data(), sizeof(dspmv_op) * scheds[0]->ops.size()))
            return fail(DSPMV_ERR_ARG, "every rank must run the same schedule (P:460)");
        plans[r] = p;
    }
    for (int r = 0; r < nranks; ++r) {
        ST_TRY(begin_apply(*scheds[r], static_cast<cudaStream_t>(stream)));
        scheds[r]->origin_dirty = true;  // the ranks share the caller stream: no timestamp aliasing
        plans[r]->cur_x = x[r];
    }
    std::vector<Schedule*> ss(scheds, scheds + nranks);
    const int n_ops = int(scheds[0]->ops.size());
    for (int t = 0; t < n_ops; ++t) {
        for (int r = 0; r < nranks; ++r) ST_TRY(exec_op(*scheds[r], t, x[r], y[r], true));
        // lock-step and SPMD: a group is posted on every rank at the same op
        const int gi = scheds[0]->op_group[t];
        if (gi >= 0 && scheds[0]->groups[gi].ps && scheds[0]->groups[gi].pr && !scheds[0]->groups[gi].issued)
            ST_TRY(issue_group_local(ss, gi));
    }
    for (int r = 0; r < nranks; ++r) {
        ST_TRY(end_combine(*scheds[r], y[r], static_cast<cudaStream_t>(stream)));
        if (scheds[r]->step1) CUDA_TRY(cudaEventRecord(scheds[r]->step1, static_cast<cudaStream_t>(stream)));
        scheds[r]->timed_valid = scheds[r]->timing;
    }
    return DSPMV_OK;
}

// -------------------------------------------------------------- utilities
dspmv_status dspmv_l2_flush(int dev, dspmv_stream_t stream) {
    if (dev < 0 || dev >= 64) return fail(DSPMV_ERR_ARG, "bad device");
    std::lock_guard<std::mutex> lk(g_flush_mu);
    CUDA_TRY(cudaSetDevice(dev));
    if (!g_flush_buf[dev]) {
        int l2 = 0;
        CUDA_TRY(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
        size_t bytes = size_t(std::max(l2, 64 << 20)) * 2;
        bytes = (bytes + 4095) & ~size_t(4095);
        if (cudaMalloc(&g_flush_buf[dev], bytes) != cudaSuccess) {
            cudaGetLastError();
            g_flush_buf[dev] = nullptr;
            return fail(DSPMV_ERR_OOM, "flush buffer allocation failed");
        }
        CUDA_TRY(cudaMemset(g_flush_buf[dev], 0, bytes));
        g_flush_bytes[dev] = bytes;
    }
    CUDA_TRY(launch_flush(g_flush_buf[dev], g_flush_bytes[dev], static_cast<cudaStream_t>(stream)));
    return DSPMV_OK;
}

dspmv_status dspmv_profile_counters(unsigned long long* out, int n, int reset, int* n_out) {
    if (!out || !n_out) return fail(DSPMV_ERR_ARG, "null argument");
    const int r = prof_read(out, n, reset != 0);
    if (r < 0) return fail(DSPMV_ERR_CUDA, "reading profile counters failed");
    *n_out = r;
    return DSPMV_OK;
}

dspmv_status dspmv_launch_count(uint64_t* count) {
    if (!count) return fail(DSPMV_ERR_ARG, "null count");
    *count = g_launches.load();
    return DSPMV_OK;
}

}  // extern "C"
