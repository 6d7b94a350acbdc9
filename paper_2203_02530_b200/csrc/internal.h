// internal.h -- shared internals of libdspmv (not part of the ABI).
#pragma once

#include <cstdint>
#include <cstring>
#include <array>
#include <string>
#include <vector>

#include "../../include/dspmv.h"

namespace dspmv {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
dspmv_status fail(dspmv_status st, const std::string& msg);

// ------------------------------------------------------- row-block kernel
// Geometry of the TMA-staged row-block kernel (kernels.cu): a block is a run
// of consecutive rows with <= tile nonzeros and <= rowmax rows, split at plan
// time into `warps` consumer-warp sub-ranges; one producer warp stages whole
// blocks into a ring of `stages` shared-memory slots with 1-D TMA copies.
struct BlockCfg {
    int tile, rowmax, warps, stages, min_ctas;  // min_ctas: __launch_bounds__ occupancy
    int chunk;                                  // x gathers in flight per lane (one lane per row)
    int lane_max;                               // rows with <= lane_max nnz: one lane per row
};
constexpr BlockCfg kBlockCfgs[] = {
    // tile  rowmax warps stages min_ctas chunk lane_max  (rowmax = 32 x warps: one row per lane)
    {2048, 256, 8, 2, 4, 8, 8},     // 0  fp32 short rows
    {1024, 128, 4, 2, 6, 8, 8},     // 1
    {2048, 256, 8, 3, 2, 8, 8},     // 2
    {1024, 128, 4, 3, 5, 8, 8},     // 3  fp64 short / irregular rows (default)
    {768, 96, 3, 3, 7, 8, 8},       // 4
    {4096, 256, 8, 2, 2, 16, 32},   // 5  long uniform rows: 8 warps, one lane per row up to 32 nnz
    {4096, 128, 4, 2, 2, 32, 32},   // 6  long rows, 4 warps, 32 gathers in flight
    {3072, 96, 3, 2, 3, 32, 32},    // 7  long rows: 3 warps, 3 CTAs/SM
};
constexpr int kNumBlockCfgs = sizeof(kBlockCfgs) / sizeof(kBlockCfgs[0]);
constexpr int kDefaultBlockCfg = 3;   // short rows (one lane per row)
constexpr int kShortRowBlockCfgF32 = 0;  // fp32 short rows: bigger blocks (measured 85 % vs 77 %)
constexpr int kLongRowBlockCfgF64 = 5;  // long, uniform rows, fp64: 8 warps, one lane per row (C3 91.6 % vs 86 %)
constexpr int kLongRowBlockCfg = 6;     // long, uniform rows, fp32: 4 warps, 32 gathers in flight (89 % vs 79 %)
constexpr int kAutoReserveSms = 8;    // SMs left to NCCL/pack when nranks > 1 (free on B200: y_L
                                      // time unchanged with 148-16 SMs)
constexpr int kTileMin = 1024;        // smallest tile among the auto-chosen configs
constexpr int kTileMax = 2048;     // vector_threshold upper bound (a row fits a block)
constexpr int kPad = 8;            // device arrays padded (aligned over-read)
constexpr int kDescInts = 16;      // per-block descriptor: r0 r1 p0 p1 flag wb[0..warps]
constexpr int kStreamTile = 256;   // CSR-stream tile: nnz per warp pass (8 per lane)
constexpr int kStreamRows = 64;    // CSR-stream tile: rows
constexpr int kStreamWarps = 8;    // CSR-stream tiles per TMA-fed block (K1c)
#ifndef DSPMV_STREAM_CTA_WARPS
#define DSPMV_STREAM_CTA_WARPS 20
#endif
constexpr int kStreamCtaWarps = DSPMV_STREAM_CTA_WARPS;   // K1b CTA: warps (one tile each); 20 x 2 CTAs/SM measured 1 % faster than 8 x 5 on C4
constexpr int kStreamGrab = 8;          // K1b: consecutive tiles per work batch (4-8 measured best; 1: 0.77-0.81 ms)
constexpr bool kStreamDynamic = true;   // K1b: batches from an atomic counter (C4 0.700-0.703 ms vs 0.709-0.716 static)
// CSR-stream with a TMA producer (spmv_stream_tma_kernel): a block is kStreamWarps
// consecutive tiles, staged whole (col, val, rowptr slice) by one producer warp
constexpr int kSTBlockNnz = kStreamWarps * kStreamTile;    // 2048
constexpr int kSTBlockRows = kStreamWarps * kStreamRows;   // 512
// Sliced CSR (spmv_sell_kernel, DSPMV_SKERNEL_SELL): 32-row slices, lane l
// owns row l; within windows of kSellWindow S rows the rows are sorted by
// length (descending, stable), so the lanes still active at entry k are a
// prefix 0..m_k-1 and entry k of the slice is stored as m_k consecutive values
// Producer-side L2 prefetch (cp.async.bulk.prefetch.L2) of a later block's
// matrix slices: the row-block kernel prefetches block b + d*grid while it
// stages block b (C3 y_L 0.953 -> 0.875 ms at d = 1 or 2, C2 unchanged at 1)
constexpr int kBlockL2Prefetch = 1;
constexpr int kSellWindow = 256;
constexpr int kSellChunkCost = 2048;   // work chunk: ~entries (+ overheads) per warp grab (dynamic: 2048 best)
#ifndef DSPMV_SELL_CTA_WARPS
#define DSPMV_SELL_CTA_WARPS 8
#endif
constexpr int kSellCtaWarps = DSPMV_SELL_CTA_WARPS;
constexpr int kSellUnroll = 4;     // x gathers in flight per lane (DSPMV_SELL_UNROLL: 4 / 8 / 16)
constexpr int kDefaultStVariant = 2;   // kernels.cu kStVariants: 3 slots, 2 CTAs/SM, pipelined
constexpr int kDefaultVectorThreshold = 256;  // rows above: warp-per-row kernel
constexpr int kMaxClass = 5;       // row classes: 2^c lanes per row, c = 0..5
constexpr int kBinWindow = 4096;   // rows are binned by class within such windows

// ----------------------------------------------------------- host planner
// One rank's split of its rows (a1): A_L, A_R, halo, pack map.
struct RankPlan {
    int rank = 0, nranks = 1;
    int64_t n_global = 0, row_begin = 0, row_end = 0;
    int esize = 8;                    // bytes per value
    std::vector<int32_t> al_rowptr, al_col;
    std::vector<uint8_t> al_val;
    std::vector<int32_t> ar_rows, ar_rowptr, ar_col;
    std::vector<uint8_t> ar_val;
    std::vector<int32_t> halo_gid;
    std::vector<int32_t> recv_count, recv_displ;   // [P]
    std::vector<int32_t> send_count, send_displ;   // [P] (phase 2)
    std::vector<int32_t> pack_map;                 // [s]  (phase 2)
    int64_t n_local() const { return row_end - row_begin; }
};

std::vector<int64_t> partition(int64_t n, int P);
// Phase 1: split + halo of rank r (needs only its own rows).  val may be null.
dspmv_status plan_phase1(int64_t n_global, int nranks, int rank, int64_t n_local,
                         const int64_t* rowptr, const int32_t* col, const void* val,
                         int esize, RankPlan& out);
// Phase 2 given every rank's halo: send counts/displ + pack map of rank p.
void plan_phase2_from_requests(RankPlan& p, const std::vector<std::vector<int32_t>>& requests);
// DSPMV_PACK_ALIAS_IF_CONTIGUOUS: every destination's send list consecutive?
bool pack_alias_offsets(const RankPlan& h, std::vector<int64_t>& off);
// requests[r] = global ids rank p must send to rank r (ascending)
std::vector<int32_t> halo_segment_for(const RankPlan& r, int owner);

// Row layout for one matrix (A_L or A_R) in device order.
struct Layout {
    int32_t nrows = 0;                 // matrix rows
    // S group: rows with len <= vthr, in ascending matrix-row order
    int32_t nS = 0, nb = 0;
    std::vector<int32_t> s_rowptr, s_col, s_desc, s_out, s_slot;
    std::vector<uint8_t> s_val;
    bool s_identity = true;            // s_out[i] == i
    bool s_has_slot = false;
    // V group: rows with len > vthr (warp-per-row)
    int32_t nV = 0;
    std::vector<int32_t> v_rowptr, v_col, v_out, v_slot;
    std::vector<uint8_t> v_val;
    bool v_has_slot = false;
    // CSR-stream form of the S group (irregular row lengths): row-aligned
    // tiles [r0, r1) of <= kStreamTile nnz and <= kStreamRows rows, S rows in
    // matrix-row order (no class binning)
    bool stream = false;
    std::vector<int32_t> s_tiles;      // 2 per tile
    // the same tiles grouped kStreamWarps at a time for the TMA-producer
    // variant: r0 r1 p0 p1 flag tb[0..kStreamWarps] per block (kDescInts)
    std::vector<int32_t> s_tdesc;
    // sliced form (DSPMV_SKERNEL_SELL): slice s covers lanes 32s..32s+31;
    // sl_srow = S-row index of the lane (-1: empty lane), sl_len its nnz;
    // the slice's entries start at sl_base[s] in sl_col / sl_val
    bool sell = false;
    std::vector<int32_t> sl_base, sl_srow, sl_col;
    std::vector<int32_t> sl_chunk;     // first slice of each work chunk (+ end)
    std::vector<uint16_t> sl_len;
    std::vector<uint8_t> sl_val;
};
// out_row / slot nullable: identity / no combine.
// Plan-time choice of the row-block configuration for one matrix: measured
// on B200 (K1 table), one-lane-per-row matrices (7-pt stencils,
// power-law) run best with cfg 3, long uniform rows (27-pt) with cfg 0.
int auto_block_cfg(const int32_t* rowptr, int32_t nrows, int vthr, int esize);
// Plan-time choice of the S-group kernel: CSR-stream for irregular row
// lengths (coefficient of variation > 0.5, e.g. the power-law G2), the
// TMA-staged row-block kernel otherwise (stencils, banded)
bool auto_stream(const int32_t* rowptr, int32_t nrows, int vthr);
void build_layout(const int32_t* rowptr, int32_t nrows, const int32_t* col, const uint8_t* val,
                  int esize, const int32_t* out_row, const int32_t* slot, int vthr,
                  const BlockCfg& cfg, Layout& L, bool stream = false, bool sell = false, int sell_win = 0);
int sell_window();   // kSellWindow, or DSPMV_SELL_WINDOW (sweeps); sell_win > 0 overrides
int sell_chunk_cost();   // kSellChunkCost, or DSPMV_SELL_CHUNK (sweeps)

// -------------------------------------------------------------- schedules
// A DAG vertex instance: kind + peer offset (0 = coarse / not an exchange vertex)
struct DagVertex {
    int kind;
    int peer;
};
// The program DAG of one granularity (schedule.cpp build_dag).
struct Dag {
    std::vector<DagVertex> v;
    std::vector<std::array<int, 3>> edges;  // u, v, deadlock edge
    bool fine = false;
    std::vector<int> offsets;                // S (sorted); {0} when coarse
    int find(int kind, int peer) const;
};
bool build_dag(const std::vector<DagVertex>& present, Dag& g, std::string& why);
struct SchedCheck {
    dspmv_status st = DSPMV_OK;
    std::string why;
    Dag dag;
    std::vector<int> inst;                   // op -> DAG vertex id (-1 for syncs)
};
bool is_gpu_vertex(int kind);
bool is_dag_vertex(int kind);
bool is_exchange_vertex(int kind);
SchedCheck validate_schedule(const dspmv_op* ops, int n_ops, int n_streams);
const char* vertex_name(int kind);
std::string vertex_label(int kind, int peer);

}  // namespace dspmv
