/* dspmv.h -- C ABI of the B200-native distributed SpMV hot path of
 * arXiv 2203.02530 (Pearson, Javeed, Devine, "Machine Learning for CUDA+MPI
 * Design Rules").  Citations "P:n" are PAPER.md line numbers; "S:n" SPEC.md.
 *
 * What the library computes (§III-A "DAG Representation"):
 *   "A common distributed memory implementation evenly divides contiguous rows
 *    of A, x, and y evenly across MPI ranks.  A rank's y entries can then be
 *    computed as the sum of a 'local' and 'remote' matrix-vector multiplication
 *    y_L = A_L x_L and y_R = A_R x_R ... each rank must copy a subset of its x_L
 *    entries into one buffer for each other rank (the Pack vertex).
 *    Communication is done with point-to-point MPI_Isends (PostSends) and
 *    MPI_Irecvs (PostRecvs)."
 * The operations (Pack, PostSend, PostRecv, WaitSend, WaitRecv, Unpack, y_L,
 * y_R, start, end) run in the order and on the CUDA streams given by a
 * caller-supplied schedule -- one traversal P of the program DAG G_P
 * (P:239-248), with the synchronisation operations of tab:sync
 * (P:436-451).  MPI point-to-point is realised with NCCL grouped send/recv
 * over NVLink; y = y_L + y_R is combined order-free (DESIGN.md R-Q9).
 *
 * Conventions
 *  - Every call returns dspmv_status (0 = OK).  No exception crosses the ABI
 *    and nothing aborts.  dspmv_last_error() returns a thread-local message
 *    describing the last non-OK return on the calling thread.
 *  - Handles are opaque.  Lifetime: comm >= plan >= schedule; destroying a
 *    parent while children live returns DSPMV_ERR_STATE.
 *  - Calls marked COLLECTIVE must be made by every rank of the communicator
 *    with consistent arguments (same n_global, identical schedule ops).
 *  - After a CUDA or NCCL error inside a collective the plan is poisoned and
 *    every later apply returns DSPMV_ERR_STATE.
 *  - Pointers: "host" pointers are ordinary CPU memory, read (or written)
 *    only during the call; "device" pointers are CUDA global memory on the
 *    plan's device.  The library never takes ownership of caller memory.
 *  - Indices are int32 (per-rank nnz and n_global must be < 2^31,
 *    DSPMV_ERR_RANGE otherwise; DESIGN.md R-Q1).
 */
#ifndef DSPMV_H
#define DSPMV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSPMV_VERSION 1

typedef enum {
    DSPMV_OK = 0,
    DSPMV_ERR_ARG = 1,       /* bad argument (NULL, out of range, inconsistent)  */
    DSPMV_ERR_RANGE = 2,     /* sizes exceed int32 indexing                       */
    DSPMV_ERR_SCHEDULE = 3,  /* not a valid traversal / missing tab:sync sync     */
    DSPMV_ERR_DEADLOCK = 4,  /* a Wait precedes its matching Post (R-Q13)         */
    DSPMV_ERR_STATE = 5,     /* wrong lifetime / not ready / poisoned             */
    DSPMV_ERR_CUDA = 6,      /* CUDA runtime error                                */
    DSPMV_ERR_NCCL = 7,      /* NCCL error (async error seen at a Wait)           */
    DSPMV_ERR_OOM = 8        /* device or host allocation failed                  */
} dspmv_status;

typedef enum { DSPMV_F64 = 0, DSPMV_F32 = 1 } dspmv_dtype;

typedef struct dspmv_comm_s* dspmv_comm_t;
typedef struct dspmv_plan_s* dspmv_plan_t;
typedef struct dspmv_schedule_s* dspmv_schedule_t;
typedef struct dspmv_host_plan_s* dspmv_host_plan_t;
/* a cudaStream_t passed through as an opaque pointer; NULL = legacy stream */
typedef void* dspmv_stream_t;

/* Thread-local description of the last failure on this thread ("" if none). */
const char* dspmv_last_error(void);
int dspmv_version(void);

/* ------------------------------------------------------------ communicator
 * The rank <-> GPU binding: one process per GPU (NCCL), or -- for tests on a
 * single device -- an in-process group of nranks simulated ranks sharing one
 * device whose exchange is a device-to-device copy (kind LOCAL).           */
enum { DSPMV_COMM_NCCL = 0, DSPMV_COMM_LOCAL = 1, DSPMV_COMM_HOST = 2 };

/* Rank 0 obtains a 128-byte NCCL unique id; the caller broadcasts it (e.g.
 * torch.distributed.broadcast_object_list) to every rank. */
dspmv_status dspmv_comm_unique_id(unsigned char id[128]);
/* COLLECTIVE.  ncclCommInitRank on cuda_device.  *out owned by the caller,
 * release with dspmv_comm_destroy. */
dspmv_status dspmv_comm_create(const unsigned char id[128], int nranks, int rank,
                               int cuda_device, dspmv_comm_t* out);
/* nranks in-process ranks on one device; out[r] is rank r's handle. */
dspmv_status dspmv_comm_create_local(int nranks, int cuda_device, dspmv_comm_t* out);
/* Host-transport communicator (kind HOST), one per process: plan-time
 * collectives (request lists, IPC handles) go through the caller's
 * `allgather(send, recv, bytes, ctx)` (every rank contributes `bytes`, recv
 * receives nranks*bytes in rank order, returns 0 on success; e.g. backed by
 * torch.distributed gloo or MPI); every apply-time byte moves device to device
 * over peer memory, so plans on a HOST comm must use DSPMV_EXCHANGE_PUT.
 * Ranks may share a device (separate processes). */
typedef int (*dspmv_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);
dspmv_status dspmv_comm_create_host(int nranks, int rank, int cuda_device, dspmv_allgather_fn allgather,
                                    void* ctx, dspmv_comm_t* out);
/* ERR_STATE if plans created on it are still alive. */
dspmv_status dspmv_comm_destroy(dspmv_comm_t comm);
dspmv_status dspmv_comm_info(dspmv_comm_t comm, int* nranks, int* rank, int* kind);

/* ------------------------------------------------------------- partition
 * P:271-272 "evenly divides contiguous rows": row_begin[r] =
 * r*floor(n/P) + min(r, n mod P) for r = 0..P (host array of nranks+1
 * int64, written by the call).  Ranks may own 0 rows when P > n (R-Q3). */
dspmv_status dspmv_partition(int64_t n_global, int nranks, int64_t* row_begin);

/* ------------------------------------------------------------------ plan */
typedef struct {
    int32_t dtype;             /* DSPMV_F64 (default) | DSPMV_F32                        */
    int32_t vector_threshold;  /* rows with more nnz than this use the warp-per-row
                                  kernel; the rest the TMA-staged row-block kernel
                                  (2^c lanes per row, c by row length).
                                  -1 = default (256); valid 0..1024                     */
    int32_t keep_host;         /* 1: keep host copies of A_L/A_R for dspmv_plan_export  */
    int32_t comm_priority;     /* 1 (default): the internal comm stream at the highest
                                  priority.  All schedule streams share the lowest
                                  priority, so they are interchangeable (the stream
                                  bijection of the design space)             */
    int32_t block_cfg;         /* row-block kernel configuration (tile nnz / consumer
                                  warps / TMA stages), -1 = chosen per matrix from its
                                  row lengths; K1                         */
    int32_t caller_stream0;    /* 1: schedule stream 0 IS the stream passed to apply (its
                                  ops need no cross-stream wait); 0 (default): a
                                  library stream ordered after the caller's stream     */
    int32_t reserve_sms;       /* SMs left free by the persistent SpMV grid so NCCL /
                                  pack kernels can run concurrently; -1 (default) =
                                  8 when the communicator has > 1 rank, else 0         */
    int32_t exchange;          /* DSPMV_EXCHANGE_COPY (default): PostSend/PostRecv issue
                                  one NCCL group (LOCAL: device copies).
                                  DSPMV_EXCHANGE_PUT: Pack is fused with the send -- it
                                  stores each destination's segment straight into the
                                  peer's receive buffer over peer memory (NVLink; CUDA
                                  IPC handles exchanged at plan time for NCCL comms)
                                  and publishes an epoch flag; the exchange waits on the
                                  flags with stream memory operations               */
    int32_t s_kernel;          /* kernel of the rows with <= vector_threshold nnz:
                                  DSPMV_SKERNEL_AUTO (0, default): CSR-stream when the
                                  row lengths are irregular (coefficient of variation
                                  > 0.5), else the row-block kernel; a forced block_cfg
                                  implies the row-block kernel.  DSPMV_SKERNEL_BLOCK:
                                  TMA-staged row blocks.  DSPMV_SKERNEL_STREAM: a warp
                                  per row-aligned tile of <= 256 nnz gathers 8 x values
                                  per lane (coalesced col/val loads), then one lane per
                                  row sums its products in stored order (bitwise the
                                  serial CSR loop).  DSPMV_SKERNEL_SELL: the
                                  plan stores the S rows as 32-row slices (rows sorted
                                  by length within windows, entry k of the slice's rows
                                  stored contiguously); one lane per row walks its row
                                  in stored order with coalesced col/val loads and no
                                  shared memory (also bitwise the serial loop)         */
    int32_t pack_mode;         /* DSPMV_PACK_GATHER (0, default): Pack gathers
                                  sendbuf[k] = x[pack_map[k]].
                                  DSPMV_PACK_ALIAS_IF_CONTIGUOUS: when every
                                  destination's send list is a run of consecutive
                                  local rows (stencil planes), the
                                  NCCL sends read straight from x and Pack launches
                                  nothing; otherwise as GATHER.  COPY exchange only
                                  (PUT already fuses the gather with the store).
                                  dspmv_plan_info.pack_alias reports the outcome    */
    int32_t accumulate_mode;   /* DSPMV_ACC_TICKET (0, default): y = y_L + y_R combined
                                  by the second SpMV to finish each row (R-Q9).
                                  DSPMV_ACC_EXPLICIT_IN_END (debug): y_L and y_R only
                                  deposit their partials; END adds them
                                  (y_i = fl(s_L,i + s_R,i)) in one kernel on
                                  the caller's stream.  Same bits as TICKET.        */
    int32_t debug_checks;      /* 1: COLLECTIVE calls verify their arguments agree
                                  across ranks -- plan_create hashes (n_global,
                                  nranks, dtype, modes), the first apply of a
                                  schedule hashes its ops; a mismatch returns
                                  DSPMV_ERR_ARG / DSPMV_ERR_SCHEDULE on every rank.
                                  Default 0, or the env DSPMV_DEBUG_CHECKS.         */
    int32_t unpack_mode;       /* DSPMV_UNPACK_COPY (0, default): Unpack copies the
                                  receive buffer to x_halo (R-Q8).  DSPMV_UNPACK_FUSED:
                                  Unpack launches nothing and y_R gathers the halo
                                  straight from the receive buffer (PUT: the half of
                                  this apply's parity, read from the device epoch) --
                                  SURVEY 8(d): "the unpack term 2v*h_r is 0 if fused" */
    int32_t long_row_sum;      /* rows of more than vector_threshold nnz (a warp per
                                  row): DSPMV_LONG_ROW_TREE (0, default): each lane
                                  accumulates every 32nd product with a fused
                                  multiply-add, then a shuffle tree (within the R-Q11
                                  tolerance).  DSPMV_LONG_ROW_STORED: rounded products
                                  added in stored order from +0 (the serial CSR loop,
                                  P:273), so EVERY row is bitwise the oracle's; the
                                  sum is a serial chain per row (C4: +2 %, DESIGN K2) */
    /* Device memory of the plan (matrix layouts, buffers): alloc(bytes, device,
       ctx) returns device memory on `device` or NULL (-> DSPMV_ERR_OOM);
       free(ptr, bytes, device, ctx) releases it at plan_destroy (after the
       device is idle for the plan).  NULL = cudaMalloc / cudaFree.  The Python
       binding routes them to the framework's caching allocator.  Buffers peers map
       through CUDA IPC (PUT receive buffers and flags) always use cudaMalloc. */
    void* (*alloc)(size_t bytes, int device, void* ctx);
    void (*free)(void* ptr, size_t bytes, int device, void* ctx);
    void* alloc_ctx;
} dspmv_plan_opts;

enum { DSPMV_PACK_GATHER = 0, DSPMV_PACK_ALIAS_IF_CONTIGUOUS = 1 };
enum { DSPMV_ACC_TICKET = 0, DSPMV_ACC_EXPLICIT_IN_END = 1 };
enum { DSPMV_UNPACK_COPY = 0, DSPMV_UNPACK_FUSED = 1 };
enum { DSPMV_LONG_ROW_TREE = 0, DSPMV_LONG_ROW_STORED = 1 };

enum { DSPMV_EXCHANGE_COPY = 0, DSPMV_EXCHANGE_PUT = 1,
       /* timing baseline only (SURVEY 8(d) overlap efficiency, T_noexch): Post/Wait
          run their synchronisation but move no data, so y is WRONG on rows with
          remote entries.  Never a product mode. */
       DSPMV_EXCHANGE_NONE = 2 };
enum { DSPMV_SKERNEL_AUTO = 0, DSPMV_SKERNEL_BLOCK = 1, DSPMV_SKERNEL_STREAM = 2, DSPMV_SKERNEL_STREAM_TMA = 3,
       DSPMV_SKERNEL_SELL = 4 };

void dspmv_plan_opts_default(dspmv_plan_opts* opts);

/* COLLECTIVE (a1).  The caller passes ITS row block [row_begin,
 * row_end) of A = dspmv_partition(n_global, nranks)[rank..rank+1] as host CSR:
 *   rowptr     host int64[n_local+1] (offsets; rowptr[0] need not be 0),
 *   col_global host int32[nnz], global column ids in [0, n_global), any order
 *              (order is preserved inside A_L and A_R rows, R-Q5),
 *   val        host dtype[nnz].
 * Arrays are read during the call only.  The plan splits A_L / A_R, builds
 * the halo list (ascending global id, R-Q4), exchanges request lists with the
 * owners (NCCL; for LOCAL comms the exchange completes when the last rank of
 * the group has called plan_create), builds pack maps, row blocks, uploads to
 * the device and allocates the exchange buffers.  opts may be NULL. */
dspmv_status dspmv_plan_create(dspmv_comm_t comm, int64_t n_global, int64_t n_local,
                               const int64_t* rowptr, const int32_t* col_global,
                               const void* val, const dspmv_plan_opts* opts,
                               dspmv_plan_t* out);
dspmv_status dspmv_plan_destroy(dspmv_plan_t plan);

typedef struct {
    int64_t n_global, row_begin, row_end;
    int64_t nnz_local, nnz_remote;   /* nnz of A_L, A_R                                */
    int64_t n_remote_rows;           /* |R_r|: rows with >= 1 remote entry             */
    int64_t n_halo, n_send;          /* h_r (entries received), s_r (entries sent)     */
    int32_t n_recv_peers, n_send_peers;
    int32_t n_blocks_local, n_vrows_local;    /* row blocks / warp-per-row rows, A_L   */
    int32_t n_blocks_remote, n_vrows_remote;  /* same for A_R                          */
    int32_t grid_local, grid_remote;          /* persistent grid of the block kernel   */
    int32_t rank, nranks, dtype, ready;
    int64_t device_bytes;
    int32_t s_kernel_local, s_kernel_remote;  /* DSPMV_SKERNEL_BLOCK / _STREAM(_TMA)     */
    int32_t pack_alias;              /* 1: sends read x directly, Pack is empty
                                        (host plans: 1 if ALIAS_IF_CONTIGUOUS would
                                        alias this rank's send lists)             */
    int32_t accumulate_mode;         /* DSPMV_ACC_* in use                         */
    int32_t unpack_fused;            /* 1: y_R reads the receive buffer            */
} dspmv_plan_info;
dspmv_status dspmv_plan_info_get(dspmv_plan_t plan, dspmv_plan_info* out);

/* Bit-exact test hook: copy one plan array to host_dst (capacity `bytes`).
 * *needed (may be NULL) receives the array's byte size.  Index arrays are
 * int32; value arrays the plan dtype.  AL_* / AR_* need opts.keep_host = 1. */
enum {
    DSPMV_HALO_GID = 0,   /* int32[h]   global ids of x_R, ascending                  */
    DSPMV_RECV_COUNTS,    /* int32[P]   halo entries owned by each rank                */
    DSPMV_RECV_DISPL,     /* int32[P]   exclusive prefix of RECV_COUNTS               */
    DSPMV_SEND_COUNTS,    /* int32[P]   entries each rank requests from this rank      */
    DSPMV_SEND_DISPL,     /* int32[P]                                                  */
    DSPMV_PACK_MAP,       /* int32[s]   local x index of each send-buffer entry (R-Q7) */
    DSPMV_AL_ROWPTR,      /* int32[n_local+1]                                          */
    DSPMV_AL_COL,         /* int32[nnz_L] local column (global - row_begin)            */
    DSPMV_AR_ROWS,        /* int32[|R|] local row of each compressed A_R row           */
    DSPMV_AR_ROWPTR,      /* int32[|R|+1]                                              */
    DSPMV_AR_COL,         /* int32[nnz_R] position in HALO_GID                         */
    DSPMV_AL_VAL,         /* dtype[nnz_L]                                              */
    DSPMV_AR_VAL          /* dtype[nnz_R]                                              */
};
dspmv_status dspmv_plan_export(dspmv_plan_t plan, int what, void* host_dst, size_t bytes,
                               size_t* needed);

/* Host-only twin of plan_create for CPU tests and the oracle comparison:
 * all ranks' plans from the global host CSR in one process (no device).
 * val_global may be NULL (values then not exportable). */
dspmv_status dspmv_plan_build_host(int nranks, int64_t n_global, const int64_t* rowptr_global,
                                   const int32_t* col_global, const void* val_global,
                                   int dtype, dspmv_host_plan_t* out);
dspmv_status dspmv_host_plan_info(dspmv_host_plan_t hp, int rank, dspmv_plan_info* out);
dspmv_status dspmv_host_plan_export(dspmv_host_plan_t hp, int rank, int what, void* host_dst,
                                    size_t bytes, size_t* needed);
dspmv_status dspmv_host_plan_destroy(dspmv_host_plan_t hp);

/* Host-only, ONE rank: the distributed planning protocol that
 * dspmv_plan_create runs over NCCL, with the transport left to the caller
 * (used by the multi-process gloo tests).
 *   1. dspmv_rank_plan_build_host: split + halo of this rank's rows (same
 *      arguments as dspmv_plan_create); the handle holds one rank (index 0 in
 *      dspmv_host_plan_info/export).
 *   2. dspmv_host_plan_requests: the ascending global ids this rank needs from
 *      `owner` (its halo segment); send them to `owner`.
 *   3. dspmv_host_plan_set_requests: lists[r] (counts[r] entries) = what rank
 *      r requested from this rank; builds send counts/displacements and the
 *      pack map (R-Q7).  ERR_ARG if an id is not owned by this rank. */
dspmv_status dspmv_rank_plan_build_host(int nranks, int rank, int64_t n_global, int64_t n_local,
                                        const int64_t* rowptr, const int32_t* col_global,
                                        const void* val, int dtype, dspmv_host_plan_t* out);
dspmv_status dspmv_host_plan_requests(dspmv_host_plan_t hp, int owner, int32_t* dst, size_t cap,
                                      size_t* count);
dspmv_status dspmv_host_plan_set_requests(dspmv_host_plan_t hp, const int32_t* const* lists,
                                          const int32_t* counts);

/* Host-only, test hook: the device row layout the planner builds for one
 * matrix (rowptr int64[nrows+1], relative) -- S-group row order (int32[nS]),
 * block descriptors (int32[nb*16]: r0 r1 p0 p1 flag|class<<8 warp bounds),
 * V-group rows (int32[nV]) -- with block configuration `cfg` (-1 = auto) and
 * vector threshold `vthr` (-1 = default).  Pass NULL outputs to get sizes. */
dspmv_status dspmv_layout_host(const int64_t* rowptr, int32_t nrows, int dtype, int cfg, int vthr,
                               int32_t* s_rows, int32_t* n_s, int32_t* desc, int32_t* n_blocks,
                               int32_t* v_rows, int32_t* n_v, int32_t* cfg_used);
/* Host-only, test hook: the CSR-stream form of the same matrix -- whether
 * s_kernel (DSPMV_SKERNEL_*; AUTO = by row-length variation, as
 * dspmv_plan_create decides) selects it (*stream_used), the tiles
 * (int32[2*n_tiles]: [r0, r1) in S-row indices, <= 256 nnz and <= 64 rows
 * each; S rows in matrix order) and the V-group rows (int32[nV], rows of
 * more than min(vthr, 256) nnz).  Tiles and V rows are returned whatever
 * *stream_used says.  Pass NULL outputs to get sizes. */
/* Host-only, test hook: the sliced form (DSPMV_SKERNEL_SELL) of the same
 * matrix's S rows (rows of <= min(vthr, 256) nnz, -1 = default), with sort
 * window `window` rows (-1 = default, K1d):
 *   slice_base int32[n_slices+1]  first stored entry of each slice
 *   lane_row   int32[32*n_slices] S-row index of each lane (-1: empty lane)
 *   lane_len   int32[32*n_slices] nnz of the lane's row
 *   entry_src  int32[nnz_S]       position, in the S group's CSR order (the
 *                                 rows' entries back to back in S-row order),
 *                                 of each stored entry
 *   chunks     int32[n_chunks+1]  first slice of each work chunk
 * Pass NULL outputs to get the sizes (*n_slices, *n_entries, *n_chunks). */
dspmv_status dspmv_sell_layout_host(const int64_t* rowptr, int32_t nrows, int vthr, int window,
                                    int32_t* slice_base, int32_t* lane_row, int32_t* lane_len,
                                    int32_t* entry_src, int32_t* chunks, int32_t* n_slices,
                                    int64_t* n_entries, int32_t* n_chunks);
dspmv_status dspmv_stream_layout_host(const int64_t* rowptr, int32_t nrows, int vthr, int s_kernel,
                                      int32_t* tiles, int32_t* n_tiles, int32_t* v_rows, int32_t* n_v,
                                      int32_t* stream_used);

/* ------------------------------------------------------------ schedules
 * A schedule is a traversal of the program DAG with every GPU
 * vertex bound to a stream (BoundGPU_s, tab:vertices P:250-264) and the
 * synchronisation operations of tab:sync as explicit ops.
 *
 * DAG (SPEC S:125 + DESIGN.md R-Q13):  start->Pack, start->y_L,
 * start->PostRecv, Pack->PostSend, PostSend->WaitSend, PostRecv->WaitRecv,
 * WaitRecv->Unpack, Unpack->y_R, y_L->end, y_R->end, WaitSend->end,
 * PostSend->WaitRecv, PostRecv->WaitSend.
 * GPU vertices: PACK, SPMV_LOCAL (y_L), UNPACK, SPMV_REMOTE (y_R); all others
 * are synchronous CPU operations.
 *
 * Per-destination granularity ("a set of parallel independent
 * vertices for each separate pack and MPI_Isend"; DESIGN.md R-N4): the six
 * exchange vertices may instead carry a peer offset d != 0 (dspmv_op.peer),
 * meaning "the exchange with rank r+d" on every rank r (SPMD).  With the
 * send-offset set S, the DAG has Pack[d], PostSend[d], WaitSend[d] and
 * PostRecv[-d], WaitRecv[-d], Unpack[-d] for each d in S, the coarse edges
 * per offset (Unpack[e]->y_R for every e, WaitSend[d]->end for every d) and
 * the deadlock edges PostSend[d]->WaitRecv[-d], PostRecv[-d]->WaitSend[d].
 * A schedule is all coarse (peer 0) or all per destination.  A vertex whose
 * rank r+d does not exist or exchanges nothing with r does nothing; at
 * schedule_create every peer the plan exchanges with must be named. */
typedef enum {
    DSPMV_OP_START = 0,
    DSPMV_OP_PACK = 1,         /* GPU: sendbuf[k] = x[pack_map[k]]                   */
    DSPMV_OP_SPMV_LOCAL = 2,   /* GPU: y_L = A_L x_L (+ order-free combine)          */
    DSPMV_OP_POST_SEND = 3,    /* CPU: MPI_Isend x peers -> NCCL (R-Q16)             */
    DSPMV_OP_POST_RECV = 4,    /* CPU: MPI_Irecv x peers                             */
    DSPMV_OP_WAIT_SEND = 5,    /* CPU: MPI_Wait on the sends                         */
    DSPMV_OP_WAIT_RECV = 6,    /* CPU: MPI_Wait on the receives                      */
    DSPMV_OP_UNPACK = 7,       /* GPU: x_halo = recvbuf (R-Q8)                       */
    DSPMV_OP_SPMV_REMOTE = 8,  /* GPU: y_R = A_R x_R (+ order-free combine)          */
    DSPMV_OP_END = 9,
    DSPMV_OP_EVENT_RECORD = 10,      /* cudaEventRecord(event, stream)  "CER"       */
    DSPMV_OP_EVENT_SYNC = 11,        /* cudaEventSynchronize(event)     "CES"       */
    DSPMV_OP_STREAM_WAIT_EVENT = 12  /* cudaStreamWaitEvent(stream, event) "CSWE"   */
} dspmv_op_kind;

typedef struct {
    int32_t kind;      /* dspmv_op_kind                                        */
    int32_t stream;    /* GPU vertices, CER, CSWE: 0..n_streams-1; else ignored */
    int32_t event;     /* CER, CES, CSWE: 0..DSPMV_MAX_EVENTS-1; else ignored   */
    int32_t peer;      /* exchange vertices: 0 = every peer (coarse), d != 0 =
                          the peer at rank offset d (per destination); must be
                          0 for start, y_L, y_R, end; ignored for sync ops     */
} dspmv_op;

#define DSPMV_MAX_STREAMS 4
#define DSPMV_MAX_EVENTS 64
#define DSPMV_MAX_OPS 256

/* Host-only.  DSPMV_OK if ops is a valid schedule: every DAG vertex exactly
 * once, START first, END last, topological, every DAG edge u->v enforced by
 * host order, stream order or the sync ops as tab:sync requires, each event
 * recorded once before any CES/CSWE uses it.  ERR_DEADLOCK if a Wait precedes
 * its matching Post; ERR_SCHEDULE otherwise. */
dspmv_status dspmv_schedule_validate(const dspmv_op* ops, int n_ops, int n_streams);

/* Host-only.  Build a schedule from the order of the 10 DAG vertices
 * (order[i] = vertex kind) and a stream per GPU vertex (streams[i] for
 * order[i]; ignored for CPU vertices), inserting syncs per tab:sync right
 * before the vertex that needs them, predecessors in DAG edge order, already
 * enforced edges inserting nothing, events numbered 0,1,2,....
 * Writes up to cap ops to out; *n_out = count. */
dspmv_status dspmv_schedule_derive(const int32_t* order, const int32_t* streams, int n_streams,
                                   dspmv_op* out, int cap, int* n_out);
/* Same for any granularity: order[i] / peers[i] (NULL = all 0) name the
 * n_vertices DAG vertices in traversal order (per destination: 4 + 6|S|). */
dspmv_status dspmv_schedule_derive_peers(const int32_t* order, const int32_t* streams, const int32_t* peers,
                                         int n_vertices, int n_streams, dspmv_op* out, int cap, int* n_out);

/* Host-only.  The program DAG of a granularity: n_offsets = 0 -> coarse,
 * else the per-destination DAG of the send-offset set `offsets`.  Writes
 * the vertices (kinds[i], peers[i], i < *n_v; in the order start, send side
 * per offset, y_L, receive side per offset, y_R, end) and the edges
 * (edges[3*j..3*j+2] = u, v, 1 if a deadlock edge (R-Q13 / R-N4), j < *n_e).
 * Pass NULL arrays to get the counts. */
dspmv_status dspmv_schedule_dag(const int32_t* offsets, int n_offsets, int32_t* kinds, int32_t* peers, int cap_v,
                                int* n_v, int32_t* edges, int cap_e, int* n_e);

/* Host-only.  Orderable synchronisation (DESIGN.md R-N5): the
 * legal next ops after `prefix` (a schedule prefix of the DAG of `offsets`,
 * n_offsets = 0 -> coarse).  For every frontier vertex v and stream choice
 * (first-use bijection pruning) the move is v itself if every
 * edge u->v is enforced, else the next sync step of the first unmet
 * predecessor u: CER on u's stream (event id = number of CERs so far) if none
 * was recorded there after u, else CES (CPU v) / CSWE on v's stream (GPU v)
 * on the latest such event.  Empty prefix -> START.  Duplicates removed. */
dspmv_status dspmv_schedule_moves(const int32_t* offsets, int n_offsets, const dspmv_op* prefix, int n_prefix,
                                  int n_streams, dspmv_op* out, int cap, int* n_out);

/* Host-only.  External schedule text format: one op per line
 * "<name> <kind> [stream=<i>] [event=<id>] [peer=<d>]", kind in {Cpu, BoundGpu,
 * EventRecord, EventSync, StreamWaitEvent}; names start, Pack, y_L,
 * PostSend, PostRecv, WaitSend, WaitRecv, Unpack, y_R, end, per-destination
 * vertices as e.g. Pack[+1] (sync op names are free text, e.g.
 * CER-after-Pack).  Blank lines and '#' comments ignored.
 * *n_streams = 1 + highest stream used. */
dspmv_status dspmv_schedule_parse(const char* text, dspmv_op* out, int cap, int* n_out,
                                  int* n_streams);
/* Host-only.  Inverse of parse (auto-named syncs CER-after-X / CES-b4-Y). */
dspmv_status dspmv_schedule_format(const dspmv_op* ops, int n_ops, char* buf, size_t cap);

/* Validate and compile a schedule for a plan (pre-creates its events).
 * Not collective, but every rank must use identical ops in apply.
 * ERR_SCHEDULE if a per-destination schedule names no vertices for a peer
 * offset this rank exchanges data with. */
dspmv_status dspmv_schedule_create(dspmv_plan_t plan, const dspmv_op* ops, int n_ops,
                                   int n_streams, dspmv_schedule_t* out);
dspmv_status dspmv_schedule_destroy(dspmv_schedule_t sched);
/* Per-op CUDA-event timing on the op's stream (2 event records per timed
 * op).  enable: 0 off, 1 every GPU vertex, else a bit mask (1 << op kind) of
 * the GPU vertex kinds to time (bits of POST_SEND / POST_RECV time the
 * halo exchange on the comm stream, reported at the Post that issues it);
 * bit (1 << DSPMV_OP_START) additionally
 * records an event on the caller stream at START and at END.  After an
 * apply, ms[i] = device time of ops[i] (0 for untimed ops) and, with the
 * START bit, ms[0] = END - START on the caller stream (the whole apply). */
/* Bind schedule stream 0 to the caller's stream for this schedule (mode 1),
 * to a library stream (0), or follow the plan's opts.caller_stream0 (-1,
 * default).  With 1, an op at the head of stream 0 needs no fork from the
 * caller's stream (and START's timing event doubles as its begin event); the
 * two schedule streams are then no longer interchangeable, so design-space
 * sweeps keep 0 and apply 1 only when timing a chosen schedule. */
dspmv_status dspmv_schedule_set_caller_stream0(dspmv_schedule_t sched, int mode);
dspmv_status dspmv_schedule_set_timing(dspmv_schedule_t sched, int enable);
dspmv_status dspmv_schedule_op_times(dspmv_schedule_t sched, float* ms, int n);
/* Per-op timeline of the last apply (needs timing with the START bit):
 * begin_ms[i] / end_ms[i] = start / end of timed op i relative to START on
 * the caller stream (-1 for untimed ops); index 0 holds [0, END]. */
dspmv_status dspmv_schedule_op_timeline(dspmv_schedule_t sched, float* begin_ms, float* end_ms, int n);

/* ----------------------------------------------------------------- apply
 * COLLECTIVE for NCCL comms (every rank executes the same P).
 * x_local, y_local: device arrays of n_local elements of the plan dtype, on
 * the plan's device, 16-byte aligned, not aliasing.  Work is ordered after
 * prior work on `stream`.  Returns after END, i.e. y is complete (END is a
 * host synchronisation point).  Not re-entrant per plan. */
dspmv_status dspmv_apply(dspmv_schedule_t sched, const void* x_local, void* y_local,
                         dspmv_stream_t stream);
/* Same with HOST x/y, all transfers inside the call (the end-to-end path).
 * Pageable memory: H2D copy of x, apply, D2H copy of y.  Pinned (page-locked,
 * device-mapped) x and y: x is copied in up to 8 chunks and y_L runs, row-block
 * group by group, behind the chunk each group reads; the SpMV kernels store y
 * directly into the mapped host buffer.  Same bits either way. */
dspmv_status dspmv_apply_host(dspmv_schedule_t sched, const void* x_host, void* y_host,
                              dspmv_stream_t stream);
/* GPU-resident execution of the same schedule (NEXT-3 (iii)): on first use
 * (and whenever x / y change) the schedule is captured into a CUDA graph in
 * which every host synchronisation point (CES, WaitSend, WaitRecv) becomes a
 * device-side join of all streams on that event, the NCCL exchange is captured
 * on the comm stream, and START/END fork from / join into `stream`; each call
 * then launches the graph.  Stream-ordered: returns immediately, y is complete
 * when `stream` reaches this point.  Same results as dspmv_apply.  PUT
 * exchange: the apply's epoch lives in device memory (bumped by the graph's
 * first node), the fused Pack+put kernels pick the receive-buffer parity from
 * it and the wait on the sources' flags is a kernel (traps after ~30 s
 * instead of hanging on a dead peer), so the fused exchange runs without any
 * host round trip.  LOCAL groups with > 1 rank use
 * dspmv_apply_graph_group; `stream` must not be NULL. */
dspmv_status dspmv_apply_graph(dspmv_schedule_t sched, const void* x_local, void* y_local,
                               dspmv_stream_t stream);
/* Capture (or re-capture) the graph dspmv_apply_graph would launch for these
 * x/y, without launching it.  Not collective: lets SPMD callers agree that
 * every rank can run the graph before any rank launches one (an apply some
 * ranks run and others do not would desynchronise the PUT epochs). */
dspmv_status dspmv_apply_graph_prepare(dspmv_schedule_t sched, const void* x_local, void* y_local,
                                       dspmv_stream_t stream);
/* LOCAL comms: all nranks ranks of one in-process group in lock-step (op k on
 * every rank before op k+1).  scheds[r], x[r], y[r] belong to rank r. */
dspmv_status dspmv_apply_group(const dspmv_schedule_t* scheds, int nranks,
                               const void* const* x_local, void* const* y_local,
                               dspmv_stream_t stream);

/* COLLECTIVE over a LOCAL group, from one host thread: the schedules of ranks
 * 0..nranks-1 captured in lock-step into ONE CUDA graph -- every rank's ops
 * on that rank's own streams, host syncs turned into device-side joins as in
 * dspmv_apply_graph, the exchange as device copies ordered after the
 * senders' Pack kernels (COPY) or flag-wait kernels on the device epoch
 * (PUT) -- and launched on `stream` (non-default).  Stream-ordered: returns
 * without waiting.  Re-captured when a schedule, x/y pointer or the timing
 * setting changes.  The graph is held by scheds[0]; destroy the group's
 * schedules together. */
dspmv_status dspmv_apply_graph_group(const dspmv_schedule_t* scheds, int nranks, const void* const* x,
                                     void* const* y, dspmv_stream_t stream);

/* ------------------------------------------------------------- utilities */
/* Read a device scratch buffer of 2x the L2 size (allocated on first use)
 * on `stream`, evicting the working set from L2 between timed iterations. */
dspmv_status dspmv_l2_flush(int cuda_device, dspmv_stream_t stream);
/* Number of kernels this library has launched since it was loaded (kernel
 * nodes of a captured graph count at every dspmv_apply_graph). */
dspmv_status dspmv_launch_count(uint64_t* count);
/* Instrumented builds only (make PROFILE=1 -> libdspmv_prof.so): per-phase
 * clock64 totals of the row-block kernel ([0] producer waiting for an empty
 * slot, [1] producer issuing, [2] consumers waiting for a full slot,
 * [3] consumer row passes, [4] blocks, [5] consumer passes).  *n_out = 0 in
 * normal builds. */
dspmv_status dspmv_profile_counters(unsigned long long* out, int n, int reset, int* n_out);

#ifdef __cplusplus
}
#endif
#endif /* DSPMV_H */
