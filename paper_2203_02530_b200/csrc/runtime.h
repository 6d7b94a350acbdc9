// runtime.h -- device-side objects of libdspmv (plans, schedules, comms) and
// the kernel launchers of kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <memory>
#include <vector>

#include "internal.h"

typedef struct ncclComm* ncclComm_t;

namespace dspmv {

// ---------------------------------------------------------- launch counter
extern std::atomic<uint64_t> g_launches;

// Device copy of one Layout (A_L or A_R), see planner.cpp / kernels.cu.
struct DevLayout {
    int32_t nS = 0, nb = 0, nV = 0;
    int grid_s = 0, grid_v = 0;
    int cfg = 0;                       // kBlockCfgs index of the row-block kernel
    int l2pf = kBlockL2Prefetch;       // row-block producer's L2 prefetch distance (blocks of this CTA)
    int st_l2pf = 0;                   // CSR-stream / sliced kernels: L2 prefetch distance (tiles / chunks)
    bool st_dynamic = false;           // CSR-stream: tile batches from an atomic counter (d_work)
    int st_grab = kStreamGrab;         // CSR-stream: tiles per batch
    unsigned* d_work = nullptr;        // [2] zeroed; reset by the last warp of each launch
    bool combine = false;              // any row of this matrix needs the ticket combine
    int32_t* s_rowptr = nullptr;
    int32_t* s_col = nullptr;
    void* s_val = nullptr;
    int32_t* s_desc = nullptr;         // kDescInts per block
    int32_t* s_out = nullptr;          // null when identity
    int32_t* s_slot = nullptr;         // null when no combine
    int32_t* v_rowptr = nullptr;
    int32_t* v_col = nullptr;
    void* v_val = nullptr;
    int32_t* v_out = nullptr;
    int32_t* v_slot = nullptr;
    int32_t v_ordered = 0;             // V rows summed in stored order (long_row_sum STORED: bitwise O1)
    // CSR-stream S group (Layout::stream): tiles instead of TMA row blocks
    bool stream = false;
    int32_t ntiles = 0;
    int grid_t = 0;
    int32_t* s_tiles = nullptr;
    // TMA-producer variant of the CSR-stream kernel (Layout::s_tdesc)
    bool stream_tma = false;
    int st_variant = 0;                // kStVariants index (kernels.cu)
    int32_t ntblocks = 0;
    int grid_tt = 0;
    int32_t* s_tdesc = nullptr;
    // sliced form of the S group (Layout::sell, spmv_sell_kernel)
    bool sell = false;
    int32_t nslices = 0;
    int grid_sl = 0;
    int sell_unroll = 8;
    bool sell_l1 = false;              // x gathers allocate in L1 (DSPMV_SELL_L1, sweeps)
    int32_t nchunks = 0;
    int32_t* sl_chunk = nullptr;
    int32_t* sl_base = nullptr;
    int32_t* sl_srow = nullptr;
    uint16_t* sl_len = nullptr;
    int32_t* sl_col = nullptr;
    void* sl_val = nullptr;
    int64_t x_bytes = 0;               // bytes of the x operand (L2 access-policy window)
};

// Operands of one SpMV op (y_L or y_R) for the kernels.
struct SpmvOperands {
    const void* x = nullptr;           // x_L (caller) or x_halo
    void* y = nullptr;                 // caller's y
    void* my_part = nullptr;           // this op's partial for combined rows
    bool explicit_acc = false;         // deposit only; END combines (DSPMV_ACC_EXPLICIT_IN_END)
    const void* other_part = nullptr;  // the other op's partial
    unsigned* ticket = nullptr;        // per combined row, epoch counter
    // streamed x (dspmv_apply_host): row block b waits until
    // xflag[desc[15] of b] >= epoch, i.e. its x chunks have landed
    const unsigned* xflag = nullptr;
    unsigned epoch = 0;
    // fused Unpack on a PUT plan: y_R reads the receive buffer of this apply's
    // parity, x + ((*x_epoch) & 1) * x_parity_elems (device epoch, graphs)
    const unsigned* x_epoch = nullptr;
    int64_t x_parity_elems = 0;
    // apply_host with y leaving by copy engine: the producer of each row-block
    // CTA adds 1 to ydone[desc[15]] once a staged block's rows are stored
    unsigned* ydone = nullptr;
};

// kernels.cu
int block_kernel_smem_bytes(int dtype, int cfg);
int block_kernel_ctas_per_sm(int dtype, int cfg);
int stream_kernel_ctas_per_sm(int dtype);
int sell_kernel_ctas_per_sm(int dtype, int unroll);
int sell_unroll();   // gathers in flight per lane of spmv_sell_kernel (4 / 8 / 16)
int stream_tma_kernel_ctas_per_sm(int dtype, int variant);
int stream_tma_variant();   // kStVariants index in use (DSPMV_STMA_VARIANT)
void set_x_persist_limit();   // experiment DSPMV_X_PERSIST (plan time)
cudaError_t launch_spmv(const DevLayout& L, int dtype, const SpmvOperands& o, cudaStream_t s);
// row blocks [b0, b1) of the S group, plus the V group (long rows) if vec
cudaError_t launch_spmv_part(const DevLayout& L, int dtype, const SpmvOperands& o, cudaStream_t s, int32_t b0,
                             int32_t b1, bool vec);
cudaError_t launch_pack(int dtype, const void* x, const int32_t* map, void* out, int64_t n,
                        cudaStream_t s);
// DSPMV_ACC_EXPLICIT_IN_END: y[rows[k]] = partL[k] + partR[k], k < n
cudaError_t launch_combine_end(int dtype, const void* partL, const void* partR, const int32_t* rows, void* y,
                               int64_t n, cudaStream_t s);
cudaError_t launch_copy(int dtype, const void* src, void* dst, int64_t n, cudaStream_t s);
cudaError_t launch_flush(void* buf, size_t bytes, cudaStream_t s);
// fused Pack + put (DSPMV_EXCHANGE_PUT): entries [seg_begin[j], seg_begin[j+1])
// go to seg_dst[j] (peer receive buffer, this apply's parity); the last CTA
// publishes `epoch` to every seg_flag[j] with a system-scope release.
// The apply's epoch lives in device memory (*epoch, written by the host
// executor at START or bumped by the first node of a captured graph), so one
// captured graph serves every apply: the kernel picks the receive-buffer
// parity (epoch & 1) and publishes the epoch itself.
struct PutArgs {
    const void* x;
    const int32_t* pack_map;
    int64_t k0, n;              // send-list entries [k0, n)
    const int64_t* seg_begin;   // [nseg + 1]
    void* const* seg_dst;       // [2][seg_stride]: parity 0 / parity 1 destinations
    unsigned* const* seg_flag;  // [nseg]
    int nseg, seg_stride;
    const unsigned* epoch;
    unsigned* counter;          // last-CTA detection, self-resetting
};
cudaError_t launch_pack_put(int dtype, const PutArgs& a, cudaStream_t s);
// PUT Unpack: dst = (recvbuf + (epoch & 1) * parity_bytes)[0, n)
cudaError_t launch_copy_parity(int dtype, const void* recv, size_t parity_bytes, const unsigned* epoch, void* dst,
                               int64_t n, cudaStream_t s);
// PUT exchange inside a graph: wait until flags[peers[i]] >= *epoch for all i
// (system-scope acquire); traps after ~30 s so a dead peer cannot hang the GPU
// (epoch == nullptr: compare against epoch_val, the host executor's epoch)
cudaError_t launch_wait_flags(const unsigned* flags, const int* peers, int n, const unsigned* epoch,
                              cudaStream_t s, unsigned epoch_val = 0);
cudaError_t launch_epoch_bump(unsigned* epoch, cudaStream_t s);
constexpr int kMaxWaitPeers = 64;

struct Plan;

struct LocalGroup {
    int nranks = 0;
    int device = 0;
    std::vector<Plan*> plans;          // by rank, once registered
    int registered = 0;
};

struct Comm {
    int kind = DSPMV_COMM_NCCL;
    int nranks = 1, rank = 0, device = 0;
    ncclComm_t nccl = nullptr;
    std::shared_ptr<LocalGroup> group;
    dspmv_allgather_fn allgather = nullptr;  // HOST comms
    void* allgather_ctx = nullptr;
    int live_plans = 0;
    bool poisoned = false;
};

struct Plan {
    Comm* comm = nullptr;
    int device = 0, dtype = DSPMV_F64, esize = 8;
    dspmv_plan_opts opts{};
    RankPlan host;                     // split arrays (AL/AR freed unless keep_host)
    int64_t nnz_L = 0, nnz_R = 0;
    DevLayout L, R;
    int32_t* d_pack_map = nullptr;
    void* d_sendbuf = nullptr;
    void* d_recvbuf = nullptr;
    void* d_xhalo = nullptr;
    void* d_partL = nullptr;
    void* d_partR = nullptr;
    unsigned* d_ticket = nullptr;
    void* d_xin = nullptr;             // apply_host staging (lazy)
    void* d_yout = nullptr;
    cudaStream_t streams[DSPMV_MAX_STREAMS] = {};
    cudaStream_t comm_stream = nullptr;
    cudaStream_t cur_stream0 = nullptr;  // stream of schedule stream 0 in this apply
    cudaEvent_t ev_start = nullptr;
    struct Alloc {
        void* ptr;
        size_t bytes;
        bool cb;                       // from opts.alloc (else cudaMalloc)
    };
    std::vector<Alloc> allocs;
    int64_t device_bytes = 0;
    bool ready = false;                // phase 2 done (send lists, pack map)
    bool has_peers = false;            // anything to send or receive
    // DSPMV_EXCHANGE_PUT state
    bool put_mode = false;
    bool skip_exchange = false;        // DSPMV_EXCHANGE_NONE (timing baseline)
    // DSPMV_PACK_ALIAS_IF_CONTIGUOUS in effect: destination q's send list is
    // x[alias_off[q] .. + send_count[q]), sent straight from x (no Pack kernel)
    bool pack_alias = false;
    bool unpack_fused = false;         // DSPMV_UNPACK_FUSED: y_R reads the receive buffer
    std::vector<int64_t> alias_off;
    const void* cur_x = nullptr;       // x of the apply being issued / captured
    // DSPMV_ACC_EXPLICIT_IN_END: local row of each combined row (device)
    int32_t* d_ar_rows = nullptr;
    bool explicit_acc = false;
    std::vector<cudaEvent_t> g_pack_ev;  // LOCAL group graphs: Pack done, per destination
    size_t recv_stride = 0;            // elements between the two receive buffers
    unsigned epoch = 0;                // applies so far (parity selects the receive buffer)
    unsigned* d_flags = nullptr;       // [P] epoch written by each source rank
    unsigned* d_epoch = nullptr;       // this apply's epoch, device copy (PUT)
    unsigned* d_put_counter = nullptr;
    int put_nseg = 0;
    int64_t* d_seg_begin = nullptr;    // [nseg + 1]
    void** d_seg_dst = nullptr;        // [2][nseg] (parity 0 / 1)
    unsigned** d_seg_flag = nullptr;   // [nseg]
    std::vector<void*> ipc_opened;     // peer mappings to close
    bool poisoned = false;
    int live_scheds = 0;
    // streamed host input for dspmv_apply_host (built at plan time): x
    // arrives in K chunks; y_L launch group k (S blocks [grp[k], grp[k+1]))
    // reads x chunks <= k only
    struct HostPipe {
        int K = 0;
        std::vector<int64_t> x_chunk;  // [K+1] element boundaries
        std::vector<int32_t> grp;      // [K+1] S-block boundaries
        int pack_chunk = -1;           // x chunk holding max(pack_map) (-1 unknown, -2 none)
        unsigned* d_xflag = nullptr;   // [K] epoch written after chunk k lands
        cudaStream_t h2d = nullptr;
        std::vector<cudaEvent_t> ev_x;
        cudaEvent_t ev_in = nullptr;
        // y by copy engine (single rank, row-ordered S blocks, no long rows):
        // group k's blocks write y rows [yrow[k], yrow[k+1]) and count
        // themselves in d_ydone[k]; a second copy stream copies each group's
        // rows once its count reaches nblk[k]
        bool ycopy = false;
        std::vector<int64_t> yrow;     // [K+1]
        std::vector<unsigned> nblk;    // [K]
        unsigned* d_ydone = nullptr;   // [K]
        cudaStream_t d2h = nullptr;
        cudaEvent_t ev_zero = nullptr, ev_out = nullptr;
        void* y_host = nullptr;        // this apply_host's y (pinned)
        bool y_queued = false;         // enqueue_ycopy ran for this apply
    } pipe;
    bool streaming = false;            // inside dspmv_apply_host with pinned x/y
};

// One halo-exchange group of a schedule, issued once both its PostSend and
// its PostRecv have executed (R-Q16).  Coarse: every peer.  Per destination
// (R-N4): the shift by d -- send to rank r+d, receive from rank r-d -- made
// of PostSend[d] and PostRecv[-d].  COPY: the ranks data moves to / from;
// PUT: the ranks epoch flags go to / come from (both directions of every
// pair that exchanges anything, so a sender never runs two applies ahead of
// a receiver that still reads the other receive buffer).
struct ExGroup {
    int d = 0;
    std::vector<int> send_to, recv_from;
    cudaEvent_t ev = nullptr;          // recorded on the comm stream at issue
    bool ps = false, pr = false, issued = false;
    bool empty() const { return send_to.empty() && recv_from.empty(); }
};

struct Schedule {
    Plan* plan = nullptr;
    std::vector<dspmv_op> ops;
    int n_streams = 1;
    Dag dag;                           // granularity (coarse / per destination)
    // resolved against the plan (compile_exchange): exchange groups, the group
    // of every Post/Wait op, the peer rank of every per-destination Pack /
    // Unpack (-2 = all peers, -1 = nothing to do) and its PUT segment
    bool compiled = false;
    std::vector<ExGroup> groups;
    std::vector<int> op_group, op_peer, op_seg;
    cudaEvent_t ev[DSPMV_MAX_EVENTS] = {};
    bool timing = false;
    std::vector<cudaEvent_t> t0, t1;   // per op (GPU vertices only)
    cudaEvent_t step0 = nullptr, step1 = nullptr;  // START / END on the caller stream
    // GPU-resident execution (dspmv_apply_graph): the schedule captured once
    // per (x, y) into a CUDA graph with host synchronisation turned into
    // device-side joins
    cudaGraphExec_t gexec = nullptr;
    std::vector<struct Schedule*> g_group;     // LOCAL group graph: the ranks' schedules (on rank 0's)
    std::vector<const void*> g_group_ptrs;     // x_r, y_r the group graph was captured for
    struct Schedule* g_leader = nullptr;       // member of a group graph held by this schedule
    const void* gx = nullptr;
    void* gy = nullptr;
    bool g_timing = false;
    uint64_t graph_kernels = 0;        // kernel nodes per graph launch (launch counter)
    cudaEvent_t gev[DSPMV_MAX_STREAMS + 2] = {};  // fork / join helpers
    bool timed_valid = false;
    bool hash_checked = false;         // opts.debug_checks: ops agreed across ranks
    int caller_stream0 = -1;           // -1: the plan's opts.caller_stream0; 0 / 1: override
    // Timestamp aliasing.  A timing event recorded right behind another one
    // on the same stream costs ~2.3 us on B200
    // (profiles/r1_ubench_graph_events.txt), so an event that would sit at
    // the same stream position as one already recorded reuses it: an op's
    // begin event directly after START is START's event (t0_alias), and in a
    // graph whose other streams carry no nodes, END directly after an op's end
    // event is that event (end_alias).  Same timestamps, fewer records.
    std::vector<char> t0_alias, g_t0_alias;   // current apply / captured graph
    int end_alias = -1, g_end_alias = -1;
    // enqueue tracking while an apply is issued / captured
    cudaStream_t origin = nullptr;     // the caller's stream (START / END)
    bool origin_dirty = true;          // work or a wait on origin since START
    bool others_dirty = true;          // nodes on any other stream (graph)
    int origin_tail = -1;              // op whose end event is the last item on origin
    int ev_on[DSPMV_MAX_EVENTS] = {};  // schedule event -> stream it was recorded on (+1)
    cudaEvent_t begin_event(int t) const { return t0_alias[t] ? step0 : t0[t]; }
    cudaEvent_t end_event() const { return end_alias >= 0 ? t1[end_alias] : step1; }
};

}  // namespace dspmv
