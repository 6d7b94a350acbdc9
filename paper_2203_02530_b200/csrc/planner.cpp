// planner.cpp -- host planner: row partition (a0), local/remote split, halo
// list and pack maps (a1), and the device row layout of A_L / A_R.
//
// PAPER.md §III-A: "evenly divides contiguous rows of A, x, and y
// ... A_L has the column entries of A that correspond to x_L ... A_R has the
// rest ... A is considered to be static, so the entries that make up x_R are
// fixed ... each rank must copy a subset of its x_L entries into one buffer
// for each other rank (the Pack vertex)".  Readings: DESIGN.md R-Q3 (uneven
// partition), R-Q4 (halo ascending by global id => grouped by owner), R-Q5
// (stored order kept), R-Q6 (compressed A_R rows), R-Q7 (pack-map order).
#include <algorithm>
#include <cstdlib>
#include <numeric>

#include "internal.h"

namespace dspmv {

std::vector<int64_t> partition(int64_t n, int P) {
    std::vector<int64_t> rb(P + 1);
    const int64_t q = n / P, rem = n % P;
    for (int r = 0; r <= P; ++r) rb[r] = r * q + std::min<int64_t>(r, rem);
    return rb;
}

dspmv_status plan_phase1(int64_t n_global, int nranks, int rank, int64_t n_local,
                         const int64_t* rowptr, const int32_t* col, const void* val,
                         int esize, RankPlan& out) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(DSPMV_ERR_ARG, "bad rank/nranks");
    if (n_global < 0) return fail(DSPMV_ERR_ARG, "n_global < 0");
    if (n_global >= (int64_t(1) << 31)) return fail(DSPMV_ERR_RANGE, "n_global >= 2^31");
    const std::vector<int64_t> rb = partition(n_global, nranks);
    const int64_t b = rb[rank], e = rb[rank + 1];
    if (n_local != e - b)
        return fail(DSPMV_ERR_ARG, "n_local " + std::to_string(n_local) + " != partition size " +
                                       std::to_string(e - b));
    if (n_local > 0 && (!rowptr || (!col && rowptr[n_local] != rowptr[0])))
        return fail(DSPMV_ERR_ARG, "null CSR array");
    const int64_t base = n_local > 0 ? rowptr[0] : 0;
    const int64_t nnz = n_local > 0 ? rowptr[n_local] - base : 0;
    for (int64_t i = 0; i < n_local; ++i)
        if (rowptr[i + 1] < rowptr[i]) return fail(DSPMV_ERR_ARG, "rowptr not monotone");
    if (nnz >= (int64_t(1) << 31)) return fail(DSPMV_ERR_RANGE, "per-rank nnz >= 2^31");
    for (int64_t p = 0; p < nnz; ++p)
        if (col[p] < 0 || col[p] >= n_global)
            return fail(DSPMV_ERR_ARG, "column id out of range at nz " + std::to_string(p));

    out = RankPlan();
    out.rank = rank;
    out.nranks = nranks;
    out.n_global = n_global;
    out.row_begin = b;
    out.row_end = e;
    out.esize = esize;
    const uint8_t* v = static_cast<const uint8_t*>(val);

    // count local / remote per row
    int64_t nL = 0, nR = 0, nRrows = 0;
    for (int64_t i = 0; i < n_local; ++i) {
        int64_t r_here = 0;
        for (int64_t p = rowptr[i] - base; p < rowptr[i + 1] - base; ++p) {
            const int32_t j = col[p];
            if (j >= b && j < e) ++nL; else ++r_here;
        }
        nR += r_here;
        nRrows += r_here > 0;
    }
    out.al_rowptr.resize(n_local + 1);
    out.al_col.resize(nL);
    if (v) out.al_val.resize(size_t(nL) * esize);
    out.ar_rows.reserve(nRrows);
    out.ar_rowptr.reserve(nRrows + 1);
    out.ar_rowptr.push_back(0);
    std::vector<int32_t> ar_gcol;
    ar_gcol.reserve(nR);
    if (v) out.ar_val.resize(size_t(nR) * esize);

    int64_t qL = 0, qR = 0;
    out.al_rowptr[0] = 0;
    for (int64_t i = 0; i < n_local; ++i) {
        bool had = false;
        for (int64_t p = rowptr[i] - base; p < rowptr[i + 1] - base; ++p) {
            const int32_t j = col[p];
            if (j >= b && j < e) {
                out.al_col[qL] = int32_t(j - b);
                if (v) std::memcpy(&out.al_val[size_t(qL) * esize], v + size_t(p) * esize, esize);
                ++qL;
            } else {
                ar_gcol.push_back(j);
                if (v) std::memcpy(&out.ar_val[size_t(qR) * esize], v + size_t(p) * esize, esize);
                ++qR;
                had = true;
            }
        }
        out.al_rowptr[i + 1] = int32_t(qL);
        if (had) {
            out.ar_rows.push_back(int32_t(i));
            out.ar_rowptr.push_back(int32_t(qR));
        }
    }
    // halo: sorted unique remote columns
    out.halo_gid = ar_gcol;
    std::sort(out.halo_gid.begin(), out.halo_gid.end());
    out.halo_gid.erase(std::unique(out.halo_gid.begin(), out.halo_gid.end()), out.halo_gid.end());
    out.ar_col.resize(ar_gcol.size());
    for (size_t p = 0; p < ar_gcol.size(); ++p)
        out.ar_col[p] = int32_t(std::lower_bound(out.halo_gid.begin(), out.halo_gid.end(),
                                                 ar_gcol[p]) - out.halo_gid.begin());
    // owner segments
    out.recv_count.assign(nranks, 0);
    out.recv_displ.assign(nranks, 0);
    for (int32_t j : out.halo_gid) {
        const int owner = int(std::upper_bound(rb.begin(), rb.end(), int64_t(j)) - rb.begin()) - 1;
        out.recv_count[owner]++;
    }
    for (int p = 1; p < nranks; ++p) out.recv_displ[p] = out.recv_displ[p - 1] + out.recv_count[p - 1];
    out.send_count.assign(nranks, 0);
    out.send_displ.assign(nranks, 0);
    return DSPMV_OK;
}

std::vector<int32_t> halo_segment_for(const RankPlan& r, int owner) {
    const int32_t o = r.recv_displ[owner], c = r.recv_count[owner];
    return std::vector<int32_t>(r.halo_gid.begin() + o, r.halo_gid.begin() + o + c);
}

void plan_phase2_from_requests(RankPlan& p, const std::vector<std::vector<int32_t>>& requests) {
    const int P = p.nranks;
    p.send_count.assign(P, 0);
    p.send_displ.assign(P, 0);
    p.pack_map.clear();
    for (int r = 0; r < P; ++r) {
        p.send_count[r] = int32_t(requests[r].size());
        if (r > 0) p.send_displ[r] = p.send_displ[r - 1] + p.send_count[r - 1];
        for (int32_t g : requests[r]) p.pack_map.push_back(int32_t(g - p.row_begin));
    }
}

// DSPMV_PACK_ALIAS_IF_CONTIGUOUS: true when the send list
// to every destination is a run of consecutive local rows; off[q] is then
// its first row (host-only, phase 2 done).
bool pack_alias_offsets(const RankPlan& h, std::vector<int64_t>& off) {
    off.assign(size_t(h.nranks), 0);
    if (h.pack_map.empty() || h.send_count.empty()) return false;
    for (int q = 0; q < h.nranks; ++q) {
        const int32_t c = h.send_count[q], d = h.send_displ[q];
        if (c <= 0) continue;
        const int32_t b = h.pack_map[d];
        for (int32_t k = 1; k < c; ++k)
            if (h.pack_map[d + k] != b + k) return false;
        off[q] = b;
    }
    return true;
}

// ---------------------------------------------------------------- layout
int auto_block_cfg(const int32_t* rowptr, int32_t nrows, int vthr, int esize) {
    int64_t nnz = 0, nnz_short = 0, rows = 0;
    for (int32_t i = 0; i < nrows; ++i) {
        const int32_t len = rowptr[i + 1] - rowptr[i];
        if (len > vthr) continue;
        nnz += len;
        ++rows;
        if (len <= 8) nnz_short += len;
    }
    if (rows == 0) return kDefaultBlockCfg;
    const double avg = double(nnz) / double(rows);
    if (2 * nnz_short < nnz && avg >= 20.0) return esize == 8 ? kLongRowBlockCfgF64 : kLongRowBlockCfg;
    return esize == 4 ? kShortRowBlockCfgF32 : kDefaultBlockCfg;
}

int sell_window() {   // read at every plan creation (sweeps change it between plans)
    const char* ev = std::getenv("DSPMV_SELL_WINDOW");
    const int v = ev ? std::atoi(ev) : kSellWindow;
    return std::max(32, v - v % 32);
}

int sell_chunk_cost() {   // read at every plan creation (sweeps)
    const char* ev = std::getenv("DSPMV_SELL_CHUNK");
    return ev ? std::max(1, std::atoi(ev)) : kSellChunkCost;
}

// Sliced form of the S group (DSPMV_SKERNEL_SELL).  Within each window of
// sell_window() S rows the rows are ordered by length, longest first (ties
// in row order), and cut into slices of 32 lanes.  Entry k of every row of a
// slice still longer than k is stored at sl_base[s] + (entries of the slice
// before k) + lane, so the m_k lanes active at k read m_k consecutive values.
// Each row's own entries keep their CSR order (the serial loop's).
static void build_sell(Layout& L, int esize, int window) {
    const int32_t nS = L.nS, W = window > 0 ? std::max(32, window - window % 32) : sell_window();
    const int64_t ns = (int64_t(nS) + 31) / 32 + (nS ? (nS / W + 1) : 0);  // upper bound (partial slices per window)
    L.sl_base.clear();
    L.sl_srow.clear();
    L.sl_len.clear();
    L.sl_base.reserve(size_t(ns) + 1);
    const int64_t nnz = L.s_rowptr[nS];
    L.sl_col.assign(size_t(nnz) + kPad, 0);
    L.sl_val.assign((size_t(nnz) + kPad) * esize, 0);
    std::vector<int32_t> order;
    int64_t q = 0;
    for (int32_t w0 = 0; w0 < nS; w0 += W) {
        const int32_t w1 = std::min(nS, w0 + W);
        order.resize(size_t(w1 - w0));
        for (int32_t r = w0; r < w1; ++r) order[size_t(r - w0)] = r;
        auto len = [&](int32_t r) { return L.s_rowptr[r + 1] - L.s_rowptr[r]; };
        std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return len(a) > len(b); });
        for (size_t s0 = 0; s0 < order.size(); s0 += 32) {
            const size_t s1 = std::min(order.size(), s0 + 32);
            L.sl_base.push_back(int32_t(q));
            for (size_t t = s0; t < s0 + 32; ++t) {
                L.sl_srow.push_back(t < s1 ? order[t] : -1);
                L.sl_len.push_back(t < s1 ? uint16_t(len(order[t])) : uint16_t(0));
            }
            const int32_t width = len(order[s0]);
            for (int32_t k = 0; k < width; ++k) {
                for (size_t t = s0; t < s1 && len(order[t]) > k; ++t) {
                    const int32_t src = L.s_rowptr[order[t]] + k;
                    L.sl_col[size_t(q)] = L.s_col[size_t(src)];
                    std::memcpy(&L.sl_val[size_t(q) * esize], &L.s_val[size_t(src) * esize], size_t(esize));
                    ++q;
                }
            }
        }
    }
    L.sl_base.push_back(int32_t(q));
    // Work chunks: runs of consecutive slices of about equal cost (entries +
    // per-iteration and per-slice overhead).  Warps stride over chunks, so the
    // rows in flight stay a moving front (x locality) and a window's wide
    // first slice does not always land on the same warps.
    const int64_t target = sell_chunk_cost();
    L.sl_chunk.clear();
    int64_t acc = 0;
    const int32_t nsl = int32_t(L.sl_base.size()) - 1;
    for (int32_t s = 0; s < nsl; ++s) {
        if (acc == 0) L.sl_chunk.push_back(s);
        acc += int64_t(L.sl_base[s + 1] - L.sl_base[s]) + 8 * int64_t(L.sl_len[size_t(32) * s]) + 64;
        if (acc >= target) acc = 0;
    }
    L.sl_chunk.push_back(nsl);
}

bool auto_stream(const int32_t* rowptr, int32_t nrows, int vthr) {
    double s1 = 0, s2 = 0;
    int64_t rows = 0;
    for (int32_t i = 0; i < nrows; ++i) {
        const double len = rowptr[i + 1] - rowptr[i];
        if (len > vthr) continue;
        s1 += len;
        s2 += len * len;
        ++rows;
    }
    if (rows < 2 || s1 <= 0) return false;
    const double mean = s1 / double(rows), var = s2 / double(rows) - mean * mean;
    return var > 0.25 * mean * mean;   // CV > 0.5
}

void build_layout(const int32_t* rowptr, int32_t nrows, const int32_t* col, const uint8_t* val,
                  int esize, const int32_t* out_row, const int32_t* slot, int vthr,
                  const BlockCfg& cfg, Layout& L, bool stream, bool sell, int sell_win) {
    L = Layout();
    L.nrows = nrows;
    L.stream = stream || sell;
    L.sell = sell;
    stream = L.stream;
    if (stream) vthr = std::min(vthr, kStreamTile);   // a CSR-stream tile holds any S row
    std::vector<int32_t> srows, vrows;
    srows.reserve(nrows);
    for (int32_t i = 0; i < nrows; ++i) {
        if (rowptr[i + 1] - rowptr[i] > vthr) vrows.push_back(i); else srows.push_back(i);
    }
    // Row-length binning (north_star: sub-warp-per-row chosen by row length):
    // class c = log2(lanes per row), the smallest c with len <= 8 * 2^c.  Within
    // windows of kBinWindow S rows the rows are stable-partitioned by class, so
    // a block never mixes classes and y writes stay local to the window.
    // rows up to the configuration's lane_max nnz stay in class 0 (one lane per row)
    static const int max_class_env = [] {
        const char* v = std::getenv("DSPMV_MAX_CLASS");
        return v ? std::atoi(v) : kMaxClass;
    }();
    const int one_lane_len = cfg.lane_max;
    auto row_class = [&](int32_t i) {
        const int32_t len = rowptr[i + 1] - rowptr[i];
        if (stream || len <= one_lane_len) return 0;   // CSR-stream: matrix-row order
        int c = 0;
        while (c < kMaxClass && len > (8 << c)) ++c;
        return std::min(c, max_class_env);
    };
    {
        std::vector<int32_t> sorted;
        sorted.reserve(srows.size());
        for (size_t w0 = 0; w0 < srows.size(); w0 += kBinWindow) {
            const size_t w1 = std::min(srows.size(), w0 + kBinWindow);
            for (int c = 0; c <= kMaxClass; ++c)
                for (size_t k = w0; k < w1; ++k)
                    if (row_class(srows[k]) == c) sorted.push_back(srows[k]);
        }
        srows.swap(sorted);
    }
    std::vector<uint8_t> scls(srows.size());
    for (size_t k = 0; k < srows.size(); ++k) scls[k] = uint8_t(row_class(srows[k]));
    L.nS = int32_t(srows.size());
    L.nV = int32_t(vrows.size());
    auto gather = [&](const std::vector<int32_t>& rows, std::vector<int32_t>& rp,
                      std::vector<int32_t>& c, std::vector<uint8_t>& v, std::vector<int32_t>& out,
                      std::vector<int32_t>& sl, bool& has_slot, bool& ident) {
        const size_t n = rows.size();
        int64_t tot = 0;
        for (int32_t i : rows) tot += rowptr[i + 1] - rowptr[i];
        rp.assign(n + 1 + kPad, 0);
        c.assign(size_t(tot) + kPad, 0);
        v.assign((size_t(tot) + kPad) * esize, 0);
        out.resize(n);
        sl.resize(n);
        has_slot = false;
        ident = true;
        int64_t q = 0;
        for (size_t k = 0; k < n; ++k) {
            const int32_t i = rows[k];
            const int32_t len = rowptr[i + 1] - rowptr[i];
            std::memcpy(&c[q], col + rowptr[i], size_t(len) * 4);
            if (val) std::memcpy(&v[size_t(q) * esize], val + size_t(rowptr[i]) * esize, size_t(len) * esize);
            q += len;
            rp[k + 1] = int32_t(q);
            out[k] = out_row ? out_row[i] : i;
            sl[k] = slot ? slot[i] : -1;
            if (sl[k] >= 0) has_slot = true;
            if (out[k] != int32_t(k)) ident = false;
        }
        for (size_t k = n + 1; k < rp.size(); ++k) rp[k] = int32_t(q);  // padded tail
    };
    bool dummy = true;
    gather(srows, L.s_rowptr, L.s_col, L.s_val, L.s_out, L.s_slot, L.s_has_slot, L.s_identity);
    gather(vrows, L.v_rowptr, L.v_col, L.v_val, L.v_out, L.v_slot, L.v_has_slot, dummy);
    // Row blocks of the S group: greedy runs of one class c with <= tile nnz
    // and <= rowmax >> c rows (each consumer warp then handles 32 >> c rows,
    // 2^c lanes per row, in one pass).  Descriptor: r0 r1 p0 p1
    // (flag | c << 8) wb[0..warps]; wb split the rows evenly over the warps.
    L.s_desc.clear();
    int32_t r = 0;
    const int W = cfg.warps;
    while (r < L.nS) {
        const int32_t r0 = r;
        const int32_t p0 = L.s_rowptr[r0];
        const int c = scls[r0];
        const int32_t rowmax = std::max(1, cfg.rowmax >> c);
        bool flag = false;
        while (r < L.nS && scls[r] == c && r - r0 < rowmax && L.s_rowptr[r + 1] - p0 <= cfg.tile) {
            flag |= L.s_slot[r] >= 0;
            ++r;
        }
        const int32_t r1 = r, p1 = L.s_rowptr[r1];
        int32_t d[kDescInts] = {};
        d[0] = r0;
        d[1] = r1;
        d[2] = p0;
        d[3] = p1;
        d[4] = (flag ? 1 : 0) | (c << 8);
        // consumer warps process one row per lane: split the rows evenly
        const int32_t rpw = (r1 - r0 + W - 1) / W;
        for (int w = 0; w <= W; ++w) d[5 + w] = std::min(r1, r0 + w * rpw);
        L.s_desc.insert(L.s_desc.end(), d, d + kDescInts);
    }
    L.nb = int32_t(L.s_desc.size() / kDescInts);
    if (sell) build_sell(L, esize, sell_win);
    if (stream) {
        // CSR-stream tiles: greedy runs of rows with <= kStreamTile nnz and
        // <= kStreamRows rows (every S row has <= vthr <= kStreamTile nnz)
        L.s_tiles.clear();
        for (int32_t t0 = 0; t0 < L.nS;) {
            int32_t t1 = t0;
            while (t1 < L.nS && t1 - t0 < kStreamRows && L.s_rowptr[t1 + 1] - L.s_rowptr[t0] <= kStreamTile) ++t1;
            L.s_tiles.push_back(t0);
            L.s_tiles.push_back(t1);
            t0 = t1;
        }
        // TMA-producer blocks: kStreamWarps consecutive tiles (tile w of a
        // block is consumer warp w's), flag = any row needs the combine
        L.s_tdesc.clear();
        const int32_t nt = int32_t(L.s_tiles.size() / 2);
        for (int32_t b = 0; b < nt; b += kStreamWarps) {
            const int32_t e = std::min(nt, b + kStreamWarps);
            int32_t d[kDescInts] = {};
            d[0] = L.s_tiles[2 * b];
            d[1] = L.s_tiles[2 * (e - 1) + 1];
            d[2] = L.s_rowptr[d[0]];
            d[3] = L.s_rowptr[d[1]];
            bool flag = false;
            for (int32_t r = d[0]; r < d[1]; ++r) flag |= L.s_slot[r] >= 0;
            d[4] = flag ? 1 : 0;
            for (int w = 0; w <= kStreamWarps; ++w) d[5 + w] = b + w < e ? L.s_tiles[2 * (b + w)] : d[1];
            L.s_tdesc.insert(L.s_tdesc.end(), d, d + kDescInts);
        }
    }
}

}  // namespace dspmv
