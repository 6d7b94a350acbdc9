// kernels.cu -- the sm_100a kernels of the distributed SpMV hot path.
//
//   spmv_block_kernel  y_L / y_R rows with <= vector_threshold nnz.  A
//                      persistent grid walks plan-time row blocks (<= tile
//                      nonzeros, <= rowmax rows).  Warp-specialised: one
//                      producer warp stages each whole block (val, col, rowptr
//                      slices) into a ring of shared-memory slots with 1-D TMA
//                      bulk copies (cp.async.bulk, L2 evict_first) signalled on
//                      per-slot "full" mbarriers, running up to `stages` blocks
//                      ahead; `warps` consumer warps each own a plan-time
//                      sub-range of the block's rows: they gather x (read-only
//                      path) one lane per row -- coalesced for banded rows --
//                      and sum each row sequentially in stored order with
//                      products and sums rounded separately (the rounding of
//                      the oracle's O1 loop), then release the slot on its
//                      "empty" mbarrier.  No CTA-wide barrier in the loop.
//   spmv_stream_kernel the same rows for irregular matrices (CSR-stream): a
//                      warp per row-aligned tile of <= 256 nnz loads col/val
//                      coalesced, keeps 8 x gathers per lane in flight, writes
//                      the products to shared memory, then one lane per row
//                      sums them in stored order (bitwise the O1 loop)
//   spmv_vector_kernel rows with > vector_threshold nnz: one warp per row,
//                      unrolled coalesced loads, warp-shuffle reduction.
//   pack_kernel        sendbuf[k] = x[pack_map[k]]
//   copy_kernel        x_halo = recvbuf (Unpack, DESIGN.md R-Q8); element-wise
//                      for unaligned per-destination segments
//   flush_kernel       L2 eviction between timed iterations (reads 2x L2)
//
// y = y_L + y_R on rows with remote entries is combined without an extra DAG
// vertex (DESIGN.md R-Q9): each op stores its partial in its own slot, then
// bumps a per-row ticket with acq_rel; the second arriver adds the two slots.
// fl(a+b) = fl(b+a), so y is bitwise identical for every schedule.
// SpMV is not a dense contraction: no tensor cores (north_star).
#include <cuda/atomic>
#include <atomic>
#include <cuda_runtime.h>
#include <cstdlib>

#include "runtime.h"

namespace dspmv {

std::atomic<uint64_t> g_launches{0};

#ifdef DSPMV_PROFILE
// Instrumented build (make PROFILE=1): per-phase clock64 totals of the
// row-block kernel, summed over warps -- [0] producer waiting for an empty
// slot, [1] producer issuing, [2] consumer waiting for a full slot,
// [3] consumer row passes, [4] blocks, [5] consumer passes.
__device__ unsigned long long g_prof[8];
#define PROF_T0() const long long _t0 = clock64()
#define PROF_ADD(i, t0) atomicAdd(&g_prof[i], (unsigned long long)(clock64() - (t0)))
#define PROF_INC(i, n) atomicAdd(&g_prof[i], (unsigned long long)(n))
#else
#define PROF_T0()
#define PROF_ADD(i, t0)
#define PROF_INC(i, n)
#endif

namespace {

constexpr int kThreads = 256;   // vector / pack kernels

template <typename T, int TILE, int RMAX>
struct __align__(16) Stage {
    T val[TILE + kPad];
    int32_t col[TILE + kPad];
    int32_t rp[RMAX + kPad];
    int32_t hdr[kDescInts];  // r0 r1 a0 ra0 flag wb[0..warps]
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// 1-D TMA bulk copy global -> shared, completion counted on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

// 1-D bulk prefetch global -> L2 (no shared memory, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(bytes), "l"(pol)
                 : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename T>
__device__ __forceinline__ T ld_stream_ef(const T* p, uint64_t pol);
template <>
__device__ __forceinline__ int32_t ld_stream_ef(const int32_t* p, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ double ld_stream_ef(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
template <>
__device__ __forceinline__ float ld_stream_ef(const float* p, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// Streamed x (dspmv_apply_host): wait until the copy stream has published this
// apply's epoch for the chunk; trap after ~30 s rather than hang the device.
__device__ __forceinline__ void wait_xflag(const unsigned* flag, unsigned epoch) {
    unsigned long long t0 = 0;
    while (ld_acquire_gpu(flag) < epoch) {
        __nanosleep(256);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (!t0) t0 = t;
        else if (t - t0 > 30ull * 1000000000ull) __trap();
    }
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// x gathers: read-only path with an L2 evict_last hint (x stays resident
// while the evict_first matrix streams pass through L2).  Irregular matrices
// also skip L1 allocation (no reuse there; measured +10 % on C4), banded ones
// keep it (neighbouring rows share x lines; C3).
template <bool kNoL1>
__device__ __forceinline__ double ldg_x(const double* p, uint64_t pol) {
    double v;
    if constexpr (kNoL1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
template <bool kNoL1>
__device__ __forceinline__ float ldg_x(const float* p, uint64_t pol) {
    float v;
    if constexpr (kNoL1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    return v;
}

// x still arriving (dspmv_apply_host pipeline, SpmvOperands::xflag): the
// producer lane acquires the chunk flag and the mbarrier hands that on to the
// consumers, but the read-only (.nc) path requires x to be immutable for the
// whole kernel -- so the streamed-x instantiation (kCoh) gathers with plain
// weak global loads (L1 not allocated), which the acquire chain orders.
template <bool kNoL1, bool kCoh>
__device__ __forceinline__ double load_x(const double* p, uint64_t pol) {
    if constexpr (kCoh) {
        double v;
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
        return v;
    } else {
        return ldg_x<kNoL1>(p, pol);
    }
}
template <bool kNoL1, bool kCoh>
__device__ __forceinline__ float load_x(const float* p, uint64_t pol) {
    if constexpr (kCoh) {
        float v;
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
        return v;
    } else {
        return ldg_x<kNoL1>(p, pol);
    }
}

// The x operand of an SpMV op: fixed, or (fused Unpack of a PUT plan inside a
// graph) the receive-buffer half of this apply's epoch parity.
template <typename T>
__device__ __forceinline__ const T* resolve_x(const SpmvOperands& o) {
    const T* x = static_cast<const T*>(o.x);
    if (o.x_epoch) x += ((*o.x_epoch) & 1u) * o.x_parity_elems;
    return x;
}

template <typename T> __device__ __forceinline__ T mul_rn(T a, T b);
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <typename T> __device__ __forceinline__ T add_rn(T a, T b);
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
template <typename T> __device__ __forceinline__ T fma_rn(T a, T b, T c);
template <> __device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
template <> __device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

struct BlockArgs {
    const int32_t* rowptr;
    const int32_t* col;
    const void* val;
    const int32_t* desc;
    const int32_t* out;
    const int32_t* slot;
    int32_t b0, nb;     // row blocks [b0, nb)
    int32_t l2pf;       // > 0: the producer also prefetches block b + l2pf*grid into L2
};

struct VecArgs {
    const int32_t* rowptr;
    const int32_t* col;
    const void* val;
    const int32_t* out;
    const int32_t* slot;
    int32_t nV;
    int32_t ordered;     // 1: products summed in stored order (bitwise O1), 0: FMA lanes + shuffle tree
};

// Deposit a partial of a combined row; the second arriver writes y (R-Q9).
template <typename T>
__device__ __forceinline__ void combine(T acc, int32_t k, int32_t orow, const SpmvOperands& o) {
    static_cast<T*>(o.my_part)[k] = acc;
    if (o.explicit_acc) return;   // END adds the two partials (debug mode)
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> tk(o.ticket[k]);
    const unsigned old = tk.fetch_add(1u, cuda::memory_order_acq_rel);
    if (old & 1u) {
        const T other = *reinterpret_cast<const volatile T*>(static_cast<const T*>(o.other_part) + k);
        static_cast<T*>(o.y)[orow] = add_rn(acc, other);
    }
}

// apply_host with y leaving by copy engine: block b's rows are stored (its
// slot was released by every consumer warp, mbarrier acquire); make them
// visible device-wide, then count the block in its x-chunk group
__device__ __forceinline__ void block_done(const BlockArgs& a, const SpmvOperands& o, int b) {
    const int g = __ldg(a.desc + size_t(b) * kDescInts + 15);
    __threadfence();
    atomicAdd(o.ydone + g, 1u);
}

template <int CFG>
struct Cfg {
    static constexpr int kTile = kBlockCfgs[CFG].tile;
    static constexpr int kRowMax = kBlockCfgs[CFG].rowmax;
    static constexpr int kWarps = kBlockCfgs[CFG].warps;
    static constexpr int kStages = kBlockCfgs[CFG].stages;
    static constexpr int kThreadsPerCta = (kWarps + 1) * 32;
    // irregular / short-row configs skip L1 for x (no reuse); long uniform
    // rows keep it (neighbouring rows share x lines)
    static constexpr bool kNoL1 = kBlockCfgs[CFG].chunk < 16;
    template <typename T>
    static constexpr int smem_bytes() {
        return kStages * int(sizeof(Stage<T, kTile, kRowMax>)) + 2 * kStages * 8;
    }
};

// One consumer warp's rows [w0, w1) of a staged block, L lanes per row
// (L = 1: one lane per row, products and sums rounded separately in stored
// order = the oracle's O1 loop, bitwise; L > 1: each lane sums every L-th
// entry, then a shuffle tree over the L lanes -- tolerance, R-Q10).  Lanes
// of consecutive rows read consecutive columns for banded rows, so the x
// gathers coalesce; up to 8 gathers per lane are in flight per chunk.
template <typename T, bool kIdentity, bool kOneLane, int CH, bool kNoL1, bool kCoh, typename St>
__device__ __forceinline__ void block_rows(const St& S, int lgL_rt, int w0, int w1, int a0, int ra0,
                                           bool blk_combine, int lane, const T* __restrict__ x,
                                           T* __restrict__ y, const int32_t* __restrict__ out,
                                           const int32_t* __restrict__ slot, SpmvOperands o, uint64_t xpol) {
    const int lgL = kOneLane ? 0 : lgL_rt;
    const int L = 1 << lgL;           // lanes per row (warp-uniform)
    const int G = 32 >> lgL;          // rows per warp pass
    const int sub = lane & (L - 1), grp = lane >> lgL;
    for (int rb = w0; rb < w1; rb += G) {
        const int r = rb + grp;
        const bool valid = r < w1;
        T acc = T(0);
        if (valid) {
            const int32_t e0 = S.rp[r - ra0] - a0, e1 = S.rp[r + 1 - ra0] - a0;
            for (int q = e0 + sub; q < e1; q += CH * L) {
                T xv[CH];
#pragma unroll
                for (int k = 0; k < CH; ++k)
                    if (q + k * L < e1) {
#ifdef DSPMV_DIAG_GATHER
                        // diagnostic builds: 1 = no gather (x value = column id), 2 = local gather x[row]
                        if (DSPMV_DIAG_GATHER == 1) xv[k] = T(S.col[q + k * L]);
                        else xv[k] = ldg_x<kNoL1>(x + (r & 0xfffff), xpol);
#else
                        xv[k] = load_x<kNoL1, kCoh>(x + S.col[q + k * L], xpol);
#endif
                    }
#pragma unroll
                for (int k = 0; k < CH; ++k)
                    if (q + k * L < e1) acc = add_rn(acc, mul_rn(S.val[q + k * L], xv[k]));
            }
        }
        for (int off = L >> 1; off > 0; off >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        if (valid && sub == 0) {
            const int32_t orow = kIdentity ? r : out[r];
            if (blk_combine) {
                const int32_t k = slot[r];
                if (k >= 0) {
                    combine<T>(acc, k, orow, o);
                    continue;
                }
            }
            __stcs(y + orow, acc);
        }
    }
}

template <typename T, int CFG, bool kCombine, bool kIdentity, bool kCoh>
__global__ void __launch_bounds__(Cfg<CFG>::kThreadsPerCta, kBlockCfgs[CFG].min_ctas)
    spmv_block_kernel(BlockArgs a, SpmvOperands o) {
    using C = Cfg<CFG>;
    using St = Stage<T, C::kTile, C::kRowMax>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    St* st = reinterpret_cast<St*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + C::kStages * sizeof(St));
    uint64_t* empty = full + C::kStages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], C::kWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == C::kWarps) {
        // ------------------------------------------------ producer warp
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int it = 0;
            for (int b = a.b0 + blockIdx.x; b < a.nb; b += gridDim.x, ++it) {
                const int s = it % C::kStages;
                const int u = it / C::kStages;
#ifdef DSPMV_PROFILE
                const long long tw = clock64();
#endif
                if (u > 0) {
                    mbar_wait(&empty[s], (u - 1) & 1);
                    if (kCoh && o.ydone) block_done(a, o, b - C::kStages * int(gridDim.x));
                }
#ifdef DSPMV_PROFILE
                PROF_ADD(0, tw);
                const long long ti = clock64();
#endif
                const int4* d = reinterpret_cast<const int4*>(a.desc + size_t(b) * kDescInts);
                const int4 d0 = __ldg(d), d1 = __ldg(d + 1), d2 = __ldg(d + 2), d3 = __ldg(d + 3);
                if (o.xflag) wait_xflag(o.xflag + d3.w, o.epoch);  // streamed x: chunks <= desc[15] landed
                const int32_t r0 = d0.x, r1 = d0.y, p0 = d0.z, p1 = d0.w;
                const int32_t a0 = p0 & ~3, a1 = (p1 + 3) & ~3;
                const int32_t ra0 = r0 & ~3, ra1 = (r1 + 1 + 3) & ~3;
                St& S = st[s];
                // hdr: r0 r1 a0 ra0 flag wb[0..warps] (wb = desc[5..])
                reinterpret_cast<int4*>(S.hdr)[0] = make_int4(r0, r1, a0, ra0);
                reinterpret_cast<int4*>(S.hdr)[1] = d1;
                reinterpret_cast<int4*>(S.hdr)[2] = d2;
                reinterpret_cast<int4*>(S.hdr)[3] = d3;
                const uint32_t nz = uint32_t(a1 - a0);
                const uint32_t bv = nz * sizeof(T), bc = nz * 4u, br = uint32_t(ra1 - ra0) * 4u;
                fence_proxy_async();
                mbar_arrive_expect_tx(&full[s], bv + bc + br);
                if (nz) {
                    bulk_g2s(S.val, static_cast<const T*>(a.val) + a0, bv, &full[s], pol);
                    bulk_g2s(S.col, a.col + a0, bc, &full[s], pol);
                }
                bulk_g2s(S.rp, a.rowptr + ra0, br, &full[s], pol);
                if (a.l2pf != 0) {   // a later block of this CTA: HBM -> L2 now, so its TMA load hits L2
                    const int bn = b + (a.l2pf > 0 ? a.l2pf : -a.l2pf) * int(gridDim.x);
                    if (bn < a.nb) {
                        const int4 e0 = __ldg(reinterpret_cast<const int4*>(a.desc + size_t(bn) * kDescInts));
                        const int32_t c0 = e0.z & ~3, c1 = (e0.w + 3) & ~3;
                        if (c1 > c0 && a.l2pf > 0) {
                            bulk_prefetch_l2(static_cast<const T*>(a.val) + c0, uint32_t(c1 - c0) * sizeof(T));
                            bulk_prefetch_l2(a.col + c0, uint32_t(c1 - c0) * 4u);
                        } else if (c1 > c0) {   // l2pf < 0 (sweeps): with the evict_first policy
                            bulk_prefetch_l2(static_cast<const T*>(a.val) + c0, uint32_t(c1 - c0) * sizeof(T), pol);
                            bulk_prefetch_l2(a.col + c0, uint32_t(c1 - c0) * 4u, pol);
                        }
                    }
                }
#ifdef DSPMV_PROFILE
                PROF_ADD(1, ti);
                PROF_INC(4, 1);
#endif
            }
            if (kCoh && o.ydone) {   // the last blocks of this CTA: wait until consumed, then count
                for (int j = it > C::kStages ? it - C::kStages : 0; j < it; ++j) {
                    mbar_wait(&empty[j % C::kStages], (j / C::kStages) & 1);
                    block_done(a, o, a.b0 + int(blockIdx.x) + j * int(gridDim.x));
                }
            }
        }
        return;
    }

    // ------------------------------------------------------ consumer warps
    const T* __restrict__ x = resolve_x<T>(o);
    T* __restrict__ y = static_cast<T*>(o.y);
    const int32_t* __restrict__ out = a.out;
    const int32_t* __restrict__ slot = a.slot;
    const uint64_t xpol = policy_evict_last();
    int it = 0;
    for (int b = a.b0 + blockIdx.x; b < a.nb; b += gridDim.x, ++it) {
        const int s = it % C::kStages;
        const int u = it / C::kStages;
#ifdef DSPMV_PROFILE
        const long long tf = clock64();
#endif
        mbar_wait(&full[s], u & 1);
#ifdef DSPMV_PROFILE
        if (lane == 0) PROF_ADD(2, tf);
        const long long tc = clock64();
#endif
        St& S = st[s];
        const int32_t a0 = S.hdr[2], ra0 = S.hdr[3];
        const bool blk_combine = kCombine && (S.hdr[4] & 1) != 0;
        const int32_t w0 = S.hdr[5 + warp], w1 = S.hdr[6 + warp];

        const int lgL = S.hdr[4] >> 8;
        if (lgL == 0)
            block_rows<T, kIdentity, true, kBlockCfgs[CFG].chunk, C::kNoL1, kCoh>(S, 0, w0, w1, a0, ra0, blk_combine,
                                                                                  lane, x, y, out, slot, o, xpol);
        else
            block_rows<T, kIdentity, false, 8, C::kNoL1, kCoh>(S, lgL, w0, w1, a0, ra0, blk_combine, lane, x, y, out,
                                                               slot, o, xpol);
        __syncwarp();
#ifdef DSPMV_PROFILE
        if (lane == 0) {
            PROF_ADD(3, tc);
            PROF_INC(5, 1);
        }
#endif
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

// Rows > vector_threshold: warp w of nw takes rows w, w + nw, ...
// Ordered (a.ordered): lane l forms the rounded products of entries l, l+32,
// .. (4 chunks of 32 in flight), then the warp adds them to acc in stored
// order through shuffles -- acc = acc + p from +0, the oracle's loop,
// so these rows are bitwise O1 too (the chain is serial: a 4,096-nnz row takes
// tens of microseconds, which the dynamic tile hand-out of K1b absorbs).
// Otherwise each lane accumulates every 32nd product with a fused
// multiply-add (__fma_rn), then a shuffle tree adds the 32 lane sums: a
// different order and rounding, checked by the R-Q11 tolerance (R-Q10).
template <typename T, bool kCombine>
__device__ __forceinline__ void vector_rows_ordered(const VecArgs& a, const SpmvOperands& o, int w, int nw) {
    const int lane = threadIdx.x & 31;
    const T* __restrict__ val = static_cast<const T*>(a.val);
    const T* __restrict__ x = resolve_x<T>(o);
    const uint64_t xpol = policy_evict_last();
    for (int i = w; i < a.nV; i += nw) {
        const int32_t p0 = __ldg(a.rowptr + i), p1 = __ldg(a.rowptr + i + 1);
        T acc = T(0);
        for (int32_t b = p0; b < p1; b += 128) {
            int32_t c[4];
            T v[4], pr[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int32_t q = b + 32 * u + lane;
                c[u] = q < p1 ? __ldcs(a.col + q) : 0;
                v[u] = q < p1 ? __ldcs(val + q) : T(0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                pr[u] = b + 32 * u + lane < p1 ? mul_rn(v[u], ldg_x<true>(x + c[u], xpol)) : T(0);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int m = min(32, p1 - (b + 32 * u));   // warp-uniform
#pragma unroll 8
                for (int k = 0; k < m; ++k) acc = add_rn(acc, __shfl_sync(0xffffffffu, pr[u], k));
            }
        }
        if (lane == 0) {
            const int32_t orow = a.out[i];
            if (kCombine) {
                const int32_t k = a.slot[i];
                if (k >= 0) {
                    combine<T>(acc, k, orow, o);
                    continue;
                }
            }
            static_cast<T*>(o.y)[orow] = acc;
        }
    }
}

template <typename T, bool kCombine>
__device__ __forceinline__ void vector_rows(const VecArgs& a, const SpmvOperands& o, int w, int nw) {
    if (a.ordered) {
        vector_rows_ordered<T, kCombine>(a, o, w, nw);
        return;
    }
    const int lane = threadIdx.x & 31;
    const T* __restrict__ val = static_cast<const T*>(a.val);
    const T* __restrict__ x = resolve_x<T>(o);
    const uint64_t xpol = policy_evict_last();
    for (int i = w; i < a.nV; i += nw) {
        const int32_t p0 = __ldg(a.rowptr + i), p1 = __ldg(a.rowptr + i + 1);
        T acc = T(0);
        int p = p0 + lane;
        for (; p + 96 < p1; p += 128) {
            int32_t c[4];
            T v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                c[u] = __ldcs(a.col + p + 32 * u);
                v[u] = __ldcs(val + p + 32 * u);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = fma_rn(v[u], ldg_x<true>(x + c[u], xpol), acc);
        }
        for (; p < p1; p += 32) acc = fma_rn(__ldcs(val + p), ldg_x<true>(x + __ldcs(a.col + p), xpol), acc);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        if (lane == 0) {
            const int32_t orow = a.out[i];
            if (kCombine) {
                const int32_t k = a.slot[i];
                if (k >= 0) {
                    combine<T>(acc, k, orow, o);
                    continue;
                }
            }
            static_cast<T*>(o.y)[orow] = acc;
        }
    }
}

template <typename T, bool kCombine>
__global__ void __launch_bounds__(kThreads) spmv_vector_kernel(VecArgs a, SpmvOperands o) {
    vector_rows<T, kCombine>(a, o, (blockIdx.x * kThreads + threadIdx.x) >> 5, (gridDim.x * kThreads) >> 5);
}

struct StreamArgs {
    const int32_t* rowptr;
    const int32_t* col;
    const void* val;
    const int32_t* out;
    const int32_t* slot;
    const int32_t* tiles;   // [r0, r1) per tile, S-row indices
    int32_t ntiles;
    VecArgs v;              // rows > vector_threshold (nV = 0: none / launched apart)
    int32_t l2pf;           // > 0: lane 0 prefetches tile t + l2pf*warps into L2
    unsigned* work;         // non-null: tiles handed out in batches from work[0] (work[1]: warps done)
    int32_t grab;           // tiles per batch
};

// CSR-stream (irregular row lengths).  Lane l of a warp takes entries
// l, l+32, .., l+224 of its tile: every col/val load is one coalesced 128-B
// (256-B) access and the 8 x gathers of a lane are independent, so they are
// all in flight at once -- the access order in which the gathers run at the
// measured random-gather rate (C4).  The products, each rounded,
// go to shared memory; lane j then sums row j's products in stored order from
// +0 (the oracle's loop), so y is bitwise O1 on every row.
template <typename T, bool kCombine, bool kIdentity>
#ifndef DSPMV_STREAM_MINB
#define DSPMV_STREAM_MINB 2   // 2 CTAs of 20 warps (48 registers); without a minimum ptxas takes 64 and fits one
#endif
__global__ void __launch_bounds__(kStreamCtaWarps * 32, DSPMV_STREAM_MINB) spmv_stream_kernel(StreamArgs a, SpmvOperands o) {
    __shared__ T prod[kStreamCtaWarps][kStreamTile];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const T* __restrict__ val = static_cast<const T*>(a.val);
    const T* __restrict__ x = resolve_x<T>(o);
    T* __restrict__ y = static_cast<T*>(o.y);
    T* pr = prod[w];
    // the long rows (> vector_threshold) first, a warp per row, so they do not
    // trail the tiles (and need no second launch)
    if (a.v.nV > 0) {
        if (a.v.slot) vector_rows<T, true>(a.v, o, blockIdx.x * kStreamCtaWarps + w, gridDim.x * kStreamCtaWarps);
        else vector_rows<T, false>(a.v, o, blockIdx.x * kStreamCtaWarps + w, gridDim.x * kStreamCtaWarps);
    }
    const uint64_t xpol = policy_evict_last();
#if defined(DSPMV_K1B_EF)
    const uint64_t mpol = policy_evict_first();
#endif
    // Tiles go out in batches of a.grab: batch gw first, then (dynamic,
    // a.work) the next free batch from an atomic counter -- fetched one batch
    // ahead so its latency hides -- or (static) batch gw + nw, ...
    const int gw = blockIdx.x * kStreamCtaWarps + w, nw = gridDim.x * kStreamCtaWarps;
    int bnext = a.work && lane == 0 ? int(atomicAdd(a.work, 1u)) + nw : 0;
    for (int bt = gw; bt * a.grab < a.ntiles;) {
        for (int t = bt * a.grab, te = min(a.ntiles, t + a.grab); t < te; ++t) {
            const int2 tr = __ldg(reinterpret_cast<const int2*>(a.tiles) + t);
            const int32_t p0 = __ldg(a.rowptr + tr.x), m = __ldg(a.rowptr + tr.y) - p0;
            if (a.l2pf != 0 && lane == 0) {   // a later tile of this warp: HBM -> L2 (evict_first) while this one gathers
                const int tn = t + (a.l2pf > 0 ? a.l2pf : -a.l2pf) * gridDim.x * kStreamCtaWarps;
                if (tn < a.ntiles) {
                    const int2 trn = __ldg(reinterpret_cast<const int2*>(a.tiles) + tn);
                    const int32_t c0 = __ldg(a.rowptr + trn.x) & ~3, c1 = (__ldg(a.rowptr + trn.y) + 3) & ~3;
                    if (c1 > c0) {
                        const uint64_t pf = policy_evict_first();
                        if (a.l2pf > 0) bulk_prefetch_l2(val + c0, uint32_t(c1 - c0) * sizeof(T), pf);
                        bulk_prefetch_l2(a.col + c0, uint32_t(c1 - c0) * 4u, pf);   // l2pf < 0: col only
                    }
                }
            }
            int32_t c[kStreamTile / 32];
            T v[kStreamTile / 32], xv[kStreamTile / 32];
#pragma unroll
            for (int k = 0; k < kStreamTile / 32; ++k) {
                const int q = lane + 32 * k;
#if defined(DSPMV_K1B_EF)
                // experiment: the matrix stream with an explicit L2 evict_first policy
                c[k] = q < m ? ld_stream_ef(a.col + p0 + q, mpol) : 0;
                v[k] = q < m ? ld_stream_ef(val + p0 + q, mpol) : T(0);
#else
                c[k] = q < m ? __ldcs(a.col + p0 + q) : 0;
                v[k] = q < m ? __ldcs(val + p0 + q) : T(0);
#endif
            }
#pragma unroll
            for (int k = 0; k < kStreamTile / 32; ++k) {
#if defined(DSPMV_DIAG_GATHER) && DSPMV_DIAG_GATHER == 4
                xv[k] = T(c[k]);  // diagnostic build 4: no gathers (cost of the streaming + row sums)
#else
                xv[k] = lane + 32 * k < m ? ldg_x<true>(x + c[k], xpol) : T(0);
#endif
            }
            __syncwarp();  // keeps ptxas from pairing each gather with its multiply: all 8 stay in flight
#if defined(DSPMV_DIAG_GATHER) && DSPMV_DIAG_GATHER == 5
            // diagnostic build 5: no shared memory at all (each lane sums its 8
            // products and stores one value per row slot): gathers + streaming only
            {
                T acc5 = T(0);
#pragma unroll
                for (int k = 0; k < kStreamTile / 32; ++k) acc5 = add_rn(acc5, mul_rn(v[k], xv[k]));
                if (tr.x + lane < tr.y) __stcs(y + (kIdentity ? tr.x + lane : a.out[tr.x + lane]), acc5);
                continue;
            }
#endif
#pragma unroll
            for (int k = 0; k < kStreamTile / 32; ++k) pr[lane + 32 * k] = mul_rn(v[k], xv[k]);
            __syncwarp();
            for (int32_t r = tr.x + lane; r < tr.y; r += 32) {
#if defined(DSPMV_DIAG_GATHER) && DSPMV_DIAG_GATHER == 3
                // diagnostic build 3: no row sums (cost of the gather phase alone)
                const T acc = pr[r - tr.x];
#else
                const int32_t e0 = __ldg(a.rowptr + r) - p0, e1 = __ldg(a.rowptr + r + 1) - p0;
                T acc = T(0);
                for (int32_t q = e0; q < e1; ++q) acc = add_rn(acc, pr[q]);
#endif
                const int32_t orow = kIdentity ? r : a.out[r];
                if (kCombine) {
                    const int32_t k = a.slot[r];
                    if (k >= 0) {
                        combine<T>(acc, k, orow, o);
                        continue;
                    }
                }
                __stcs(y + orow, acc);
            }
            __syncwarp();
        }
        if (a.work) {
            bt = __shfl_sync(0xffffffffu, bnext, 0);
            if (lane == 0) bnext = int(atomicAdd(a.work, 1u)) + nw;
        } else {
            bt += nw;
        }
    }
    if (a.work && lane == 0) {
        // the last warp out resets the counters for the next launch (stream
        // order publishes them); every fetch of this warp completed first
        if (bnext < 0) __trap();
        __threadfence();
        if (atomicAdd(a.work + 1, 1u) == unsigned(nw) - 1u) {
            atomicExch(a.work, 0u);
            atomicExch(a.work + 1, 0u);
        }
    }
}


// Sliced CSR (DSPMV_SKERNEL_SELL, irregular row lengths).  Warp s takes slice
// s: lane l owns row sl_srow[32s + l] and walks its sl_len entries in CSR
// order, acc = acc + v*x from +0 with every product and sum rounded (the
// oracle's loop), so y is bitwise O1 with no shared-memory pass.  The
// slice's rows are sorted longest first, so the lanes still active at entry
// k are 0..m_k-1 (m_k = popc of a ballot) and entry k of the slice is m_k
// consecutive values: every col/val load is coalesced, and the U gathers of
// a lane are independent, all in flight together.
struct SellArgs {
    const int32_t* chunk;  // per work chunk: first slice (nchunks + 1)
    const int32_t* base;   // per slice: first entry (nslices + 1)
    const int32_t* srow;   // per lane: S-row index, -1 = empty lane
    const uint16_t* len;   // per lane: nnz of the row
    const int32_t* col;
    const void* val;
    const int32_t* out;
    const int32_t* slot;
    int32_t nchunks;
    VecArgs v;             // rows > vector_threshold (nV = 0: none / launched apart)
    int32_t l2pf;          // > 0: lane 0 prefetches chunk c + l2pf*warps into L2
    unsigned* work;        // non-null: chunks handed out from work[0] (work[1]: warps done)
};

#ifndef DSPMV_SELL_MINB
#define DSPMV_SELL_MINB 6   // 48 resident warps at 40 registers (measured best, profiles/r2_c4_sell.txt)
#endif
template <typename T, bool kCombine, bool kIdentity, int U, bool kNoL1 = true>
__global__ void __launch_bounds__(kSellCtaWarps * 32, DSPMV_SELL_MINB) spmv_sell_kernel(SellArgs a, SpmvOperands o) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const T* __restrict__ val = static_cast<const T*>(a.val);
    const T* __restrict__ x = resolve_x<T>(o);
    T* __restrict__ y = static_cast<T*>(o.y);
    const int gw = blockIdx.x * kSellCtaWarps + w, nw = gridDim.x * kSellCtaWarps;
    if (a.v.nV > 0) {   // the long rows first, a warp per row, so they do not trail
        if (a.v.slot) vector_rows<T, true>(a.v, o, gw, nw);
        else vector_rows<T, false>(a.v, o, gw, nw);
    }
    const uint64_t xpol = policy_evict_last();
    // Per chunk, slice s+1's lane metadata is loaded while slice s gathers, and
    // its output row / combine slot at the end of slice s, so neither sits on
    // the next slice's dependent chain (metadata -> col -> x).
    // chunk gw first, then (a.work) the next free chunk from an atomic
    // counter, fetched one chunk ahead, or (static) chunk gw + nw, ...
    int cnext = a.work && lane == 0 ? int(atomicAdd(a.work, 1u)) + nw : 0;
    for (int c = gw; c < a.nchunks;) {
        int s = __ldg(a.chunk + c);
        const int se = __ldg(a.chunk + c + 1);
        if (a.l2pf != 0 && lane == 0) {   // a later chunk of this warp: HBM -> L2 (evict_first) while this one gathers
            const int cn = c + (a.l2pf > 0 ? a.l2pf : -a.l2pf) * nw;
            if (cn < a.nchunks) {
                const int32_t e0 = __ldg(a.base + __ldg(a.chunk + cn)) & ~3;
                const int32_t e1 = (__ldg(a.base + __ldg(a.chunk + cn + 1)) + 3) & ~3;
                if (e1 > e0) {
                    const uint64_t pf = policy_evict_first();
                    if (a.l2pf > 0) bulk_prefetch_l2(val + e0, uint32_t(e1 - e0) * sizeof(T), pf);
                    bulk_prefetch_l2(a.col + e0, uint32_t(e1 - e0) * 4u, pf);   // l2pf < 0: col only
                }
            }
        }
        int32_t sr = __ldg(a.srow + 32 * s + lane);
        int len = __ldg(a.len + 32 * s + lane);
        int32_t off = __ldg(a.base + s);
        int32_t orow = sr < 0 ? -1 : kIdentity ? sr : __ldg(a.out + sr);
        int32_t kslot = kCombine && sr >= 0 ? __ldg(a.slot + sr) : -1;
        for (; s < se; ++s) {
            const bool more = s + 1 < se;
            const int32_t sr_n = more ? __ldg(a.srow + 32 * (s + 1) + lane) : -1;
            const int len_n = more ? __ldg(a.len + 32 * (s + 1) + lane) : 0;
            const int32_t off_n = more ? __ldg(a.base + s + 1) : 0;
            const int width = __shfl_sync(0xffffffffu, len, 0);
            T acc = T(0);
            for (int k0 = 0; k0 < width; k0 += U) {
                int32_t cc[U];
                T v[U], xv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const bool act = k0 + u < len;
                    const int32_t q = off + lane;
                    off += __popc(__ballot_sync(0xffffffffu, act));
                    cc[u] = act ? __ldcs(a.col + q) : 0;
                    v[u] = act ? __ldcs(val + q) : T(0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) xv[u] = k0 + u < len ? ldg_x<kNoL1>(x + cc[u], xpol) : T(0);
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (k0 + u < len) acc = add_rn(acc, mul_rn(v[u], xv[u]));
            }
            if (orow >= 0) {
                if (kCombine && kslot >= 0) combine<T>(acc, kslot, orow, o);
                else __stcs(y + orow, acc);
            }
            orow = sr_n < 0 ? -1 : kIdentity ? sr_n : __ldg(a.out + sr_n);
            kslot = kCombine && sr_n >= 0 ? __ldg(a.slot + sr_n) : -1;
            sr = sr_n;
            len = len_n;
            off = off_n;
        }
        if (a.work) {
            c = __shfl_sync(0xffffffffu, cnext, 0);
            if (lane == 0) cnext = int(atomicAdd(a.work, 1u)) + nw;
        } else {
            c += nw;
        }
    }
    if (a.work && lane == 0) {   // the last warp out resets the counters (as in spmv_stream_kernel)
        if (cnext < 0) __trap();
        __threadfence();
        if (atomicAdd(a.work + 1, 1u) == unsigned(nw) - 1u) {
            atomicExch(a.work, 0u);
            atomicExch(a.work + 1, 0u);
        }
    }
}


// CSR-stream with a TMA producer (irregular row lengths).  The same tiles as
// spmv_stream_kernel, grouped kStreamWarps to a block: one producer warp
// stages a whole block (col, val, rowptr slice; 1-D bulk copies with an L2
// evict_first hint) into a ring of kSTStages shared-memory slots, so the
// matrix stream never enters the LSU/L1TEX path the x gathers need
// (B300_MICROARCH: one in-order wavefront queue per SM).  Consumer warp w owns
// tile w of each block: its lanes read col from shared memory and keep 8 x
// gathers each in flight (lane-strided, as in spmv_stream_kernel), overwrite
// val in place with the rounded products, then lane j sums row j's products
// in stored order from +0 (the oracle's loop): y is bitwise O1.
template <typename T>
struct __align__(16) StStage {
    T val[kSTBlockNnz + kPad];
    int32_t col[kSTBlockNnz + kPad];
    int32_t rp[kSTBlockRows + kPad];
    int32_t hdr[kDescInts];
};
// Variants (measured on C4, K1c): ring slots, CTAs per SM, and
// whether a consumer warp issues the gathers of its next block before it
// sums the rows of the current one (the gather latency then overlaps the
// stored-order row sums instead of following them).
struct StVariant {
    int stages, min_ctas;
    bool pipe;
};
constexpr StVariant kStVariants[] = {{3, 2, false}, {2, 4, false}, {3, 2, true}, {2, 3, true}};
constexpr int kNumStVariants = 4;
template <typename T, int V>
constexpr int st_smem_bytes() {
    return kStVariants[V].stages * int(sizeof(StStage<T>)) + 2 * kStVariants[V].stages * 8;
}

struct StreamTmaArgs {
    const int32_t* rowptr;
    const int32_t* col;
    const void* val;
    const int32_t* desc;
    const int32_t* out;
    const int32_t* slot;
    int32_t nb;
    VecArgs v;              // rows > vector_threshold (nV = 0: none / launched apart)
};

// One consumer warp's tile of a staged block: tile rows [t0, t1), entries
// [e0, e1) of the stage (<= kStreamTile).
struct StTile {
    int32_t a0, ra0, t0, t1, e0, e1;
    bool combine;
    int32_t ro[2], rs[2];   // output row / combine slot of rows t0 + lane (+ 32), loaded early
};

template <typename T, bool kCombine, bool kIdentity>
__device__ __forceinline__ StTile st_tile(const StStage<T>& S, int warp, int lane, const int32_t* __restrict__ out,
                                          const int32_t* __restrict__ slot) {
    StTile t;
    t.a0 = S.hdr[2];
    t.ra0 = S.hdr[3];
    t.combine = kCombine && (S.hdr[4] & 1) != 0;
    t.t0 = S.hdr[5 + warp];
    t.t1 = S.hdr[6 + warp];
    t.e0 = S.rp[t.t0 - t.ra0] - t.a0;
    t.e1 = S.rp[t.t1 - t.ra0] - t.a0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int32_t r = t.t0 + lane + 32 * j;
        const bool ok = r < t.t1;
        t.ro[j] = kIdentity ? r : (ok ? __ldg(out + r) : 0);
        t.rs[j] = (t.combine && ok) ? __ldg(slot + r) : -1;
    }
    return t;
}

template <typename T, int K>
__device__ __forceinline__ void st_gather(const StStage<T>& S, const StTile& t, int lane, const T* __restrict__ x,
                                          uint64_t xpol, T (&xv)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int q = t.e0 + lane + 32 * k;
        xv[k] = q < t.e1 ? ldg_x<true>(x + S.col[q], xpol) : T(0);
    }
}

template <typename T, int K>
__device__ __forceinline__ void st_products(StStage<T>& S, const StTile& t, int lane, const T (&xv)[K]) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int q = t.e0 + lane + 32 * k;
        if (q < t.e1) S.val[q] = mul_rn(S.val[q], xv[k]);
    }
}

template <typename T>
__device__ __forceinline__ void st_rowsums(const StStage<T>& S, const StTile& t, int lane, T* __restrict__ y,
                                           const SpmvOperands& o) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int32_t r = t.t0 + lane + 32 * j;
        if (r >= t.t1) break;
        const int32_t q0 = S.rp[r - t.ra0] - t.a0, q1 = S.rp[r + 1 - t.ra0] - t.a0;
        T acc = T(0);
        for (int32_t q = q0; q < q1; ++q) acc = add_rn(acc, S.val[q]);
        if (t.rs[j] >= 0) {
            combine<T>(acc, t.rs[j], t.ro[j], o);
            continue;
        }
        __stcs(y + t.ro[j], acc);
    }
}

template <typename T, bool kCombine, bool kIdentity, int V>
__global__ void __launch_bounds__((kStreamWarps + 1) * 32, kStVariants[V].min_ctas)
    spmv_stream_tma_kernel(StreamTmaArgs a, SpmvOperands o) {
    constexpr int NS = kStVariants[V].stages;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    StStage<T>* st = reinterpret_cast<StStage<T>*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + NS * sizeof(StStage<T>));
    uint64_t* empty = full + NS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kStreamWarps);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == kStreamWarps) {
        // ------------------------------------------------ producer warp
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int it = 0;
            for (int b = blockIdx.x; b < a.nb; b += gridDim.x, ++it) {
                const int s = it % NS;
                const int u = it / NS;
                if (u > 0) mbar_wait(&empty[s], (u - 1) & 1);
                const int4* d = reinterpret_cast<const int4*>(a.desc + size_t(b) * kDescInts);
                const int4 d0 = __ldg(d), d1 = __ldg(d + 1), d2 = __ldg(d + 2), d3 = __ldg(d + 3);
                if (o.xflag) wait_xflag(o.xflag + d3.w, o.epoch);
                const int32_t r0 = d0.x, r1 = d0.y, p0 = d0.z, p1 = d0.w;
                const int32_t a0 = p0 & ~3, a1 = (p1 + 3) & ~3;
                const int32_t ra0 = r0 & ~3, ra1 = (r1 + 1 + 3) & ~3;
                StStage<T>& S = st[s];
                reinterpret_cast<int4*>(S.hdr)[0] = make_int4(r0, r1, a0, ra0);
                reinterpret_cast<int4*>(S.hdr)[1] = d1;
                reinterpret_cast<int4*>(S.hdr)[2] = d2;
                reinterpret_cast<int4*>(S.hdr)[3] = d3;
                const uint32_t nz = uint32_t(a1 - a0);
                const uint32_t bv = nz * sizeof(T), bc = nz * 4u, br = uint32_t(ra1 - ra0) * 4u;
                fence_proxy_async();
                mbar_arrive_expect_tx(&full[s], bv + bc + br);
                if (nz) {
                    bulk_g2s(S.val, static_cast<const T*>(a.val) + a0, bv, &full[s], pol);
                    bulk_g2s(S.col, a.col + a0, bc, &full[s], pol);
                }
                bulk_g2s(S.rp, a.rowptr + ra0, br, &full[s], pol);
            }
        }
        return;
    }

    // ------------------------------------------------------ consumer warps
    if (a.v.nV > 0) {  // the long rows first, a warp per row (no second launch)
        if (a.v.slot) vector_rows<T, true>(a.v, o, blockIdx.x * kStreamWarps + warp, gridDim.x * kStreamWarps);
        else vector_rows<T, false>(a.v, o, blockIdx.x * kStreamWarps + warp, gridDim.x * kStreamWarps);
    }
    const T* __restrict__ x = resolve_x<T>(o);
    T* __restrict__ y = static_cast<T*>(o.y);
    const uint64_t xpol = policy_evict_last();
    constexpr int K = kStreamTile / 32;
    if constexpr (!kStVariants[V].pipe) {
        int it = 0;
        for (int b = blockIdx.x; b < a.nb; b += gridDim.x, ++it) {
            const int s = it % NS;
            mbar_wait(&full[s], (it / NS) & 1);
            StStage<T>& S = st[s];
            const StTile t = st_tile<T, kCombine, kIdentity>(S, warp, lane, a.out, a.slot);
            T xv[K];
            st_gather<T, K>(S, t, lane, x, xpol, xv);
            __syncwarp();
            st_products<T, K>(S, t, lane, xv);
            __syncwarp();
            st_rowsums<T>(S, t, lane, y, o);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
    } else {
        // software pipeline: block b's gathers were issued during block
        // (b - grid)'s row sums
        int it = 0, b = blockIdx.x;
        T xv[K];
        StTile t{};
        if (b < a.nb) {
            mbar_wait(&full[0], 0);
            t = st_tile<T, kCombine, kIdentity>(st[0], warp, lane, a.out, a.slot);
            st_gather<T, K>(st[0], t, lane, x, xpol, xv);
        }
        while (b < a.nb) {
            const int s = it % NS;
            StStage<T>& S = st[s];
            __syncwarp();
            st_products<T, K>(S, t, lane, xv);
            __syncwarp();
            const StTile cur = t;
            const int bn = b + gridDim.x;
            if (bn < a.nb) {   // next block's gathers in flight during this block's row sums
                const int sn = (it + 1) % NS;
                mbar_wait(&full[sn], ((it + 1) / NS) & 1);
                t = st_tile<T, kCombine, kIdentity>(st[sn], warp, lane, a.out, a.slot);
                st_gather<T, K>(st[sn], t, lane, x, xpol, xv);
            }
            st_rowsums<T>(S, cur, lane, y, o);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            b = bn;
            ++it;
        }
    }
}

template <typename T>
__global__ void combine_end_kernel(const T* __restrict__ a, const T* __restrict__ b, const int32_t* __restrict__ rows,
                                   T* __restrict__ y, int64_t n) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x)
        y[rows[k]] = add_rn(a[k], b[k]);
}

template <typename T>
__global__ void pack_kernel(const T* __restrict__ x, const int32_t* __restrict__ map, T* __restrict__ out,
                            int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = __ldg(x + __ldg(map + i));
}

// Fused Pack + put over peer memory (NEXT-3 (ii)): each entry of
// the send list is gathered from x and stored straight into the destination
// rank's receive buffer; after a system-scope fence the last CTA to finish
// publishes the epoch flag of this rank on every destination.
template <typename T>
__global__ void pack_put_kernel(PutArgs a) {
    const T* __restrict__ x = static_cast<const T*>(a.x);
    const unsigned epoch = *a.epoch;
    void* const* dst = a.seg_dst + (epoch & 1u) * a.seg_stride;
    for (int64_t k = a.k0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < a.n;
         k += int64_t(gridDim.x) * blockDim.x) {
        int j = 0;  // nseg = destinations (<= P); empty segments only carry a flag
        while (j + 1 < a.nseg && a.seg_begin[j + 1] <= k) ++j;
        static_cast<T*>(dst[j])[k - a.seg_begin[j]] = __ldg(x + __ldg(a.pack_map + k));
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> c(*a.counter);
        if (c.fetch_add(1u, cuda::memory_order_acq_rel) == gridDim.x - 1) {
            c.store(0u, cuda::memory_order_relaxed);          // ready for the next apply
            __threadfence_system();
            for (int j = 0; j < a.nseg; ++j) {
                cuda::atomic_ref<unsigned, cuda::thread_scope_system> f(*a.seg_flag[j]);
                f.store(epoch, cuda::memory_order_release);
            }
        }
    }
}

template <typename T>
__global__ void copy_parity_kernel(const T* __restrict__ recv, size_t parity_elems, const unsigned* __restrict__ ep,
                                   T* __restrict__ dst, int64_t n) {
    const T* __restrict__ src = recv + ((*ep) & 1u) * parity_elems;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = __ldcs(src + i);
}

struct WaitPeers {
    int p[kMaxWaitPeers];
};

__global__ void wait_flags_kernel(const unsigned* flags, WaitPeers peers, int n, const unsigned* ep, unsigned ep_val) {
    const unsigned want = ep ? *ep : ep_val;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        cuda::atomic_ref<const unsigned, cuda::thread_scope_system> f(flags[peers.p[i]]);
        while (int(f.load(cuda::memory_order_acquire) - want) < 0) {
            __nanosleep(128);
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 30ull * 1000000000ull) __trap();   // a peer never published: fail, do not hang
        }
    }
    __syncthreads();
    __threadfence_system();
}

__global__ void epoch_bump_kernel(unsigned* ep) { *ep += 1u; }

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16,
                            const unsigned char* __restrict__ s8, unsigned char* __restrict__ d8,
                            int64_t tail_from, int64_t tail_to) {
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t i = tid; i < n16; i += stride) dst[i] = __ldcs(src + i);
    for (int64_t i = tail_from + tid; i < tail_to; i += stride) d8[i] = s8[i];
}

// Element-wise copy for segments not 16-B aligned (per-destination Unpack).
template <typename T>
__global__ void copy_elems_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = __ldcs(src + i);
}

// Read 2x L2 of scratch (leaves L2 clean and holding none of the SpMV data);
// one conditional store per thread keeps the loads alive.
__global__ void flush_kernel(const uint4* __restrict__ buf, int64_t n16, unsigned salt, unsigned* sink) {
    unsigned acc = 0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x) {
        const uint4 v = __ldcg(buf + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == salt) sink[0] = acc;
}

// SM count of the current device, cached per device (plans on several
// devices in one process size their grids for their own device)
std::atomic<int> g_num_sms[64];

int num_sms() {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int n = g_num_sms[dev].load(std::memory_order_relaxed);
    if (n <= 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        g_num_sms[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

template <typename T, int CFG, bool C, bool I, bool H = false>
cudaError_t prep_block_kernel() {
    static std::atomic<bool> done[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    const int smem = Cfg<CFG>::template smem_bytes<T>();
    cudaError_t e = cudaFuncSetAttribute(spmv_block_kernel<T, CFG, C, I, H>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(spmv_block_kernel<T, CFG, C, I, H>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess && dev < 64) done[dev].store(true, std::memory_order_release);
    return e;
}

template <typename T, int CFG, bool C, bool I>
cudaError_t launch_block(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, int32_t b0, int32_t b1) {
    BlockArgs a{L.s_rowptr, L.s_col, L.s_val, L.s_desc, L.s_out, L.s_slot, b0, b1, L.l2pf};
    const int grid = std::min(L.grid_s, b1 - b0);
    cudaError_t e;
    if (o.xflag) {   // x streamed in: the coherent-load instantiation
        e = prep_block_kernel<T, CFG, C, I, true>();
        if (e != cudaSuccess) return e;
        spmv_block_kernel<T, CFG, C, I, true>
            <<<grid, Cfg<CFG>::kThreadsPerCta, Cfg<CFG>::template smem_bytes<T>(), s>>>(a, o);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError();
    }
    e = prep_block_kernel<T, CFG, C, I>();
    if (e != cudaSuccess) return e;
    spmv_block_kernel<T, CFG, C, I, false>
        <<<grid, Cfg<CFG>::kThreadsPerCta, Cfg<CFG>::template smem_bytes<T>(), s>>>(a, o);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

template <typename T, int CFG>
cudaError_t launch_block_cfg(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, int32_t b0, int32_t b1) {
    const bool c = L.s_slot != nullptr, id = L.s_out == nullptr;
    if (c && id) return launch_block<T, CFG, true, true>(L, o, s, b0, b1);
    if (c) return launch_block<T, CFG, true, false>(L, o, s, b0, b1);
    if (id) return launch_block<T, CFG, false, true>(L, o, s, b0, b1);
    return launch_block<T, CFG, false, false>(L, o, s, b0, b1);
}

template <typename T>
cudaError_t launch_block_any(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, int32_t b0, int32_t b1) {
    switch (L.cfg) {
        case 0: return launch_block_cfg<T, 0>(L, o, s, b0, b1);
        case 1: return launch_block_cfg<T, 1>(L, o, s, b0, b1);
        case 2: return launch_block_cfg<T, 2>(L, o, s, b0, b1);
        case 3: return launch_block_cfg<T, 3>(L, o, s, b0, b1);
        case 4: return launch_block_cfg<T, 4>(L, o, s, b0, b1);
        case 5: return launch_block_cfg<T, 5>(L, o, s, b0, b1);
        case 6: return launch_block_cfg<T, 6>(L, o, s, b0, b1);
        case 7: return launch_block_cfg<T, 7>(L, o, s, b0, b1);
        default: return cudaErrorInvalidValue;
    }
}
static_assert(kNumBlockCfgs == 8, "update launch_block_any / occupancy dispatch");

// Experiment (DSPMV_X_PERSIST=<hit ratio>): an L2 access-policy window
// marking the x operand persisting for the CSR-stream kernels.  The
// persisting carve-out itself is set at plan time (set_x_persist_limit).
double x_persist_fraction() {
    static const double f = [] {
        const char* ev = std::getenv("DSPMV_X_PERSIST");
        return ev ? std::atof(ev) : 0.0;
    }();
    return f;
}
void x_window(cudaLaunchAttribute& at, const void* x, int64_t bytes) {
    at.id = cudaLaunchAttributeAccessPolicyWindow;
    at.val.accessPolicyWindow.base_ptr = const_cast<void*>(x);
    at.val.accessPolicyWindow.num_bytes = size_t(bytes);
    at.val.accessPolicyWindow.hitRatio = float(x_persist_fraction());
    at.val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at.val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
}

template <typename T>
cudaError_t launch_stream(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, bool vec) {
    StreamArgs a{L.s_rowptr, L.s_col, L.s_val, L.s_out, L.s_slot, L.s_tiles, L.ntiles,
                 VecArgs{L.v_rowptr, L.v_col, L.v_val, L.v_out, L.v_slot, vec ? L.nV : 0, L.v_ordered}, L.st_l2pf,
                 L.st_dynamic ? L.d_work : nullptr, L.st_grab};
    const bool c = L.s_slot != nullptr, id = L.s_out == nullptr;
    const dim3 grid(L.grid_t), block(kStreamCtaWarps * 32);
    if (x_persist_fraction() > 0 && L.x_bytes > 0) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        x_window(at[0], o.x, L.x_bytes);
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e;
        if (c && id) e = cudaLaunchKernelEx(&cfg, spmv_stream_kernel<T, true, true>, a, o);
        else if (c) e = cudaLaunchKernelEx(&cfg, spmv_stream_kernel<T, true, false>, a, o);
        else if (id) e = cudaLaunchKernelEx(&cfg, spmv_stream_kernel<T, false, true>, a, o);
        else e = cudaLaunchKernelEx(&cfg, spmv_stream_kernel<T, false, false>, a, o);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    if (c && id) spmv_stream_kernel<T, true, true><<<grid, block, 0, s>>>(a, o);
    else if (c) spmv_stream_kernel<T, true, false><<<grid, block, 0, s>>>(a, o);
    else if (id) spmv_stream_kernel<T, false, true><<<grid, block, 0, s>>>(a, o);
    else spmv_stream_kernel<T, false, false><<<grid, block, 0, s>>>(a, o);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

template <typename T, int U, bool kNoL1>
cudaError_t launch_sell_u(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, bool vec) {
    SellArgs a{L.sl_chunk, L.sl_base, L.sl_srow, L.sl_len, L.sl_col, L.sl_val, L.s_out, L.s_slot, L.nchunks,
               VecArgs{L.v_rowptr, L.v_col, L.v_val, L.v_out, L.v_slot, vec ? L.nV : 0, L.v_ordered}, L.st_l2pf,
               L.st_dynamic ? L.d_work : nullptr};
    const bool c = L.s_slot != nullptr, id = L.s_out == nullptr;
    const dim3 grid(L.grid_sl), block(kSellCtaWarps * 32);
    if (x_persist_fraction() > 0 && L.x_bytes > 0) {   // experiment DSPMV_X_PERSIST
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        x_window(at[0], o.x, L.x_bytes);
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e;
        if (c && id) e = cudaLaunchKernelEx(&cfg, spmv_sell_kernel<T, true, true, U, kNoL1>, a, o);
        else if (c) e = cudaLaunchKernelEx(&cfg, spmv_sell_kernel<T, true, false, U, kNoL1>, a, o);
        else if (id) e = cudaLaunchKernelEx(&cfg, spmv_sell_kernel<T, false, true, U, kNoL1>, a, o);
        else e = cudaLaunchKernelEx(&cfg, spmv_sell_kernel<T, false, false, U, kNoL1>, a, o);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    if (c && id) spmv_sell_kernel<T, true, true, U, kNoL1><<<grid, block, 0, s>>>(a, o);
    else if (c) spmv_sell_kernel<T, true, false, U, kNoL1><<<grid, block, 0, s>>>(a, o);
    else if (id) spmv_sell_kernel<T, false, true, U, kNoL1><<<grid, block, 0, s>>>(a, o);
    else spmv_sell_kernel<T, false, false, U, kNoL1><<<grid, block, 0, s>>>(a, o);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_sell(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, bool vec) {
    if (L.sell_l1) {   // uniform (banded) rows: neighbouring rows share x lines in L1
        switch (L.sell_unroll) {
            case 4: return launch_sell_u<T, 4, false>(L, o, s, vec);
            case 16: return launch_sell_u<T, 16, false>(L, o, s, vec);
            default: return launch_sell_u<T, 8, false>(L, o, s, vec);
        }
    }
    switch (L.sell_unroll) {
        case 4: return launch_sell_u<T, 4, true>(L, o, s, vec);
        case 16: return launch_sell_u<T, 16, true>(L, o, s, vec);
        default: return launch_sell_u<T, 8, true>(L, o, s, vec);
    }
}

int st_variant() {   // DSPMV_STMA_VARIANT (sweeps); default kDefaultStVariant
    static const int v = [] {
        const char* ev = std::getenv("DSPMV_STMA_VARIANT");
        const int k = ev ? std::atoi(ev) : kDefaultStVariant;
        return (k >= 0 && k < kNumStVariants) ? k : kDefaultStVariant;
    }();
    return v;
}

template <typename T, bool C, bool I, int V>
cudaError_t prep_stream_tma() {
    static std::atomic<bool> done[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(spmv_stream_tma_kernel<T, C, I, V>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, st_smem_bytes<T, V>());
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(spmv_stream_tma_kernel<T, C, I, V>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess && dev < 64) done[dev].store(true, std::memory_order_release);
    return e;
}

template <typename T, bool C, bool I, int V>
cudaError_t launch_stream_tma_v(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, bool vec) {
    cudaError_t e = prep_stream_tma<T, C, I, V>();
    if (e != cudaSuccess) return e;
    StreamTmaArgs a{L.s_rowptr, L.s_col, L.s_val, L.s_tdesc, L.s_out, L.s_slot, L.ntblocks,
                    VecArgs{L.v_rowptr, L.v_col, L.v_val, L.v_out, L.v_slot, vec ? L.nV : 0, L.v_ordered}};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(L.grid_tt);
    cfg.blockDim = dim3((kStreamWarps + 1) * 32);
    cfg.dynamicSmemBytes = st_smem_bytes<T, V>();
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (x_persist_fraction() > 0 && L.x_bytes > 0) {
        x_window(at[0], o.x, L.x_bytes);
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    e = cudaLaunchKernelEx(&cfg, spmv_stream_tma_kernel<T, C, I, V>, a, o);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <typename T, bool C, bool I>
cudaError_t launch_stream_tma_ci(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, bool vec) {
    switch (L.st_variant) {
        case 0: return launch_stream_tma_v<T, C, I, 0>(L, o, s, vec);
        case 1: return launch_stream_tma_v<T, C, I, 1>(L, o, s, vec);
        case 2: return launch_stream_tma_v<T, C, I, 2>(L, o, s, vec);
        default: return launch_stream_tma_v<T, C, I, 3>(L, o, s, vec);
    }
}
static_assert(kNumStVariants == 4, "update launch_stream_tma_ci / occupancy dispatch");

template <typename T>
cudaError_t launch_stream_tma(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, bool vec) {
    const bool c = L.s_slot != nullptr, id = L.s_out == nullptr;
    if (c && id) return launch_stream_tma_ci<T, true, true>(L, o, s, vec);
    if (c) return launch_stream_tma_ci<T, true, false>(L, o, s, vec);
    if (id) return launch_stream_tma_ci<T, false, true>(L, o, s, vec);
    return launch_stream_tma_ci<T, false, false>(L, o, s, vec);
}

template <typename T, int V>
int stma_occupancy() {
    int n = 0;
    if (prep_stream_tma<T, false, true, V>() == cudaSuccess)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, spmv_stream_tma_kernel<T, false, true, V>,
                                                      (kStreamWarps + 1) * 32, st_smem_bytes<T, V>());
    return n > 0 ? n : 1;
}

template <typename T>
cudaError_t launch_all(const DevLayout& L, const SpmvOperands& o, cudaStream_t s, int32_t b0, int32_t b1, bool vec) {
    cudaError_t e = cudaSuccess;
    if (L.stream) {  // CSR-stream S group: all tiles (b0 / b1 ignored) and the long rows, one launch
        if (b1 > b0 && (L.sell ? L.nslices > 0 : L.ntiles > 0)) {
            e = L.sell         ? launch_sell<T>(L, o, s, vec)
                : L.stream_tma ? launch_stream_tma<T>(L, o, s, vec)
                               : launch_stream<T>(L, o, s, vec);
            if (e != cudaSuccess) return e;
            vec = false;
        }
    } else if (b1 > b0) {
        e = launch_block_any<T>(L, o, s, b0, b1);
        if (e != cudaSuccess) return e;
    }
    if (vec && L.nV > 0) {
        VecArgs a{L.v_rowptr, L.v_col, L.v_val, L.v_out, L.v_slot, L.nV, L.v_ordered};
        if (L.v_slot) spmv_vector_kernel<T, true><<<L.grid_v, kThreads, 0, s>>>(a, o);
        else spmv_vector_kernel<T, false><<<L.grid_v, kThreads, 0, s>>>(a, o);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
    }
    return e;
}

template <typename T, int CFG>
int occupancy() {
    int n = 0;
    if (prep_block_kernel<T, CFG, true, false>() != cudaSuccess) return 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, spmv_block_kernel<T, CFG, true, false, false>,
                                                  Cfg<CFG>::kThreadsPerCta, Cfg<CFG>::template smem_bytes<T>());
    return n > 0 ? n : 1;
}

template <typename T>
int occupancy_any(int cfg) {
    switch (cfg) {
        case 0: return occupancy<T, 0>();
        case 1: return occupancy<T, 1>();
        case 2: return occupancy<T, 2>();
        case 3: return occupancy<T, 3>();
        case 4: return occupancy<T, 4>();
        case 5: return occupancy<T, 5>();
        case 6: return occupancy<T, 6>();
        case 7: return occupancy<T, 7>();
        default: return 1;
    }
}

}  // namespace

int prof_read(unsigned long long* out, int n, bool reset) {
#ifdef DSPMV_PROFILE
    unsigned long long h[8];
    if (cudaMemcpyFromSymbol(h, g_prof, sizeof(h)) != cudaSuccess) return -1;
    for (int i = 0; i < n && i < 8; ++i) out[i] = h[i];
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    }
    return 8;
#else
    (void)out; (void)n; (void)reset;
    return 0;
#endif
}

int stream_kernel_ctas_per_sm(int dtype) {
    int n = 0;
    if (dtype == DSPMV_F32)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, spmv_stream_kernel<float, false, true>, kStreamCtaWarps * 32, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, spmv_stream_kernel<double, false, true>, kStreamCtaWarps * 32, 0);
    return n > 0 ? n : 1;
}

template <typename T, int U>
int sell_occupancy() {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, spmv_sell_kernel<T, false, false, U>, kSellCtaWarps * 32, 0);
    return n > 0 ? n : 1;
}

int sell_kernel_ctas_per_sm(int dtype, int unroll) {
    const bool f = dtype == DSPMV_F32;
    switch (unroll) {
        case 4: return f ? sell_occupancy<float, 4>() : sell_occupancy<double, 4>();
        case 16: return f ? sell_occupancy<float, 16>() : sell_occupancy<double, 16>();
        default: return f ? sell_occupancy<float, 8>() : sell_occupancy<double, 8>();
    }
}

int sell_unroll() {   // kSellUnroll, or DSPMV_SELL_UNROLL (sweeps; plan time)
    const char* ev = std::getenv("DSPMV_SELL_UNROLL");
    const int v = ev ? std::atoi(ev) : kSellUnroll;
    return v == 4 || v == 16 ? v : 8;
}

int stream_tma_kernel_ctas_per_sm(int dtype, int variant) {
    if (dtype == DSPMV_F32) {
        switch (variant) {
            case 0: return stma_occupancy<float, 0>();
            case 1: return stma_occupancy<float, 1>();
            case 2: return stma_occupancy<float, 2>();
            default: return stma_occupancy<float, 3>();
        }
    }
    switch (variant) {
        case 0: return stma_occupancy<double, 0>();
        case 1: return stma_occupancy<double, 1>();
        case 2: return stma_occupancy<double, 2>();
        default: return stma_occupancy<double, 3>();
    }
}

int stream_tma_variant() { return st_variant(); }

void set_x_persist_limit() {
    if (x_persist_fraction() <= 0) return;
    int dev = 0, maxp = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(maxp));
}

int block_kernel_ctas_per_sm(int dtype, int cfg) {
    return dtype == DSPMV_F32 ? occupancy_any<float>(cfg) : occupancy_any<double>(cfg);
}

int device_sm_count() { return num_sms(); }

cudaError_t launch_spmv(const DevLayout& L, int dtype, const SpmvOperands& o, cudaStream_t s) {
    return launch_spmv_part(L, dtype, o, s, 0, L.nb, true);
}

cudaError_t launch_spmv_part(const DevLayout& L, int dtype, const SpmvOperands& o, cudaStream_t s, int32_t b0,
                             int32_t b1, bool vec) {
    return dtype == DSPMV_F32 ? launch_all<float>(L, o, s, b0, b1, vec) : launch_all<double>(L, o, s, b0, b1, vec);
}

cudaError_t launch_pack(int dtype, const void* x, const int32_t* map, void* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
    if (dtype == DSPMV_F32)
        pack_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), map, static_cast<float*>(out), n);
    else
        pack_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(x), map, static_cast<double*>(out), n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_combine_end(int dtype, const void* partL, const void* partR, const int32_t* rows, void* y,
                               int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
    if (dtype == DSPMV_F32)
        combine_end_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(partL), static_cast<const float*>(partR),
                                                       rows, static_cast<float*>(y), n);
    else
        combine_end_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(partL),
                                                        static_cast<const double*>(partR), rows,
                                                        static_cast<double*>(y), n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_pack_put(int dtype, const PutArgs& a, cudaStream_t s) {
    if (a.nseg <= 0) return cudaSuccess;
    const int grid =
        int(std::max<int64_t>(1, std::min<int64_t>((a.n - a.k0 + 255) / 256, int64_t(num_sms()) * 4)));
    if (dtype == DSPMV_F32) pack_put_kernel<float><<<grid, 256, 0, s>>>(a);
    else pack_put_kernel<double><<<grid, 256, 0, s>>>(a);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_copy_parity(int dtype, const void* recv, size_t parity_bytes, const unsigned* epoch, void* dst,
                               int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 4));
    if (dtype == DSPMV_F32)
        copy_parity_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(recv), parity_bytes / 4, epoch,
                                                       static_cast<float*>(dst), n);
    else
        copy_parity_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(recv), parity_bytes / 8, epoch,
                                                        static_cast<double*>(dst), n);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_wait_flags(const unsigned* flags, const int* peers, int n, const unsigned* epoch,
                              cudaStream_t s, unsigned epoch_val) {
    if (n <= 0) return cudaSuccess;
    if (n > kMaxWaitPeers) return cudaErrorInvalidValue;
    WaitPeers w{};
    for (int i = 0; i < n; ++i) w.p[i] = peers[i];
    wait_flags_kernel<<<1, 32, 0, s>>>(flags, w, n, epoch, epoch_val);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_epoch_bump(unsigned* epoch, cudaStream_t s) {
    epoch_bump_kernel<<<1, 1, 0, s>>>(epoch);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_copy(int dtype, const void* src, void* dst, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) {
        const int grid = int(std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8));
        if (dtype == DSPMV_F32)
            copy_elems_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(src), static_cast<float*>(dst), n);
        else
            copy_elems_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(src), static_cast<double*>(dst), n);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError();
    }
    const int64_t bytes = n * (dtype == DSPMV_F32 ? 4 : 8);
    const int64_t n16 = bytes / 16;
    const int grid = int(std::min<int64_t>((n16 + 255) / 256 + 1, int64_t(num_sms()) * 8));
    copy_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint4*>(dst), n16,
                                     static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst),
                                     n16 * 16, bytes);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

cudaError_t launch_flush(void* buf, size_t bytes, cudaStream_t s) {
    static unsigned salt = 0x9e3779b9u;
    const int64_t n16 = int64_t(bytes / 16) - 1;  // last 16 B: the sink
    flush_kernel<<<num_sms() * 4, 512, 0, s>>>(static_cast<const uint4*>(buf), n16, salt++,
                                               reinterpret_cast<unsigned*>(static_cast<uint4*>(buf) + n16));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}

}  // namespace dspmv
