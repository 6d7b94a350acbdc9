// Random fp64 gathers from a 64 MB vector on B200: the LSU path (the gather
// K1b uses: ld.global.nc.L1::no_allocate + L2 evict_last) against the TMA
// unit's tile::gather4 (cp.async.bulk.tensor.2d ... tile::gather4: 4 rows of
// a 2-D tensor per instruction, issued per thread, landing in shared memory).
// x is viewed as rows of 2 doubles (16 B, the smallest TMA box), so one
// gather4 fetches 4 random x pairs.  Question: does the TMA path sustain more
// random 8-byte gathers per second than the LSU's ~1 wavefront/clock/SM?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o ub scripts/ubench_tma_gather4.cu -lcuda
//   ./ub [gathers_millions=134] [x_MB=64]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);            \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ unsigned hash32(unsigned a) {
    a ^= a >> 16;
    a *= 0x7feb352dU;
    a ^= a >> 15;
    a *= 0x846ca68bU;
    a ^= a >> 16;
    return a;
}

__global__ void fill_idx(int* idx, long long m, int n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        idx[i] = int(hash32(unsigned(i) * 2654435761u + 12345u) % unsigned(n));
}

__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// LSU: 8 independent gathers per thread in flight, like K1b
__global__ void __launch_bounds__(256) lsu_gather(const double* __restrict__ x, const int* __restrict__ idx, long long m,
                                                  double* out) {
    const uint64_t pol = pol_last();
    double acc = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += 8 * stride) {
        int c[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) c[k] = i + k * stride < m ? __ldcs(idx + i + k * stride) : 0;
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[k]) : "l"(x + c[k]), "l"(pol));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 12345.678) out[0] = acc;
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// TMA gather4: each warp owns a ring of S stages; a stage = 32 gather4 ops
// (one per lane) = 128 gathers = 2 KB; lane 0 arms the stage's mbarrier.
// (the TMA destination must be 128-B aligned: each lane's 64 B land in a 128-B slot)
template <int S, bool kTile = false>
__global__ void __launch_bounds__(128) tma_gather(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                  long long m, double* out, int bw) {
    extern __shared__ __align__(128) unsigned char dsm_raw[];
    // the dynamic shared-memory base is not guaranteed 128-B aligned: align by hand
    unsigned char* dsm = dsm_raw + ((128 - (sa(dsm_raw) & 127)) & 127);
    double (*buf)[S][32 * 16] = reinterpret_cast<double (*)[S][32 * 16]>(dsm);
    uint64_t (*bar)[S] = reinterpret_cast<uint64_t (*)[S]>(dsm + sizeof(double) * 4 * S * 32 * 16);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[w][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t pol = pol_last();
    const long long per_stage = 128;   // gathers per warp per stage
    const long long nwarps = (long long)gridDim.x * 4;
    const long long gw = blockIdx.x * 4 + w;
    double acc = 0;
    long long it = 0;
    int cc[S][4];
    // chunk j of this warp: gathers [(gw + j*nwarps) * 128, +128)
    auto issue = [&](long long j, int s) {
        const long long base = (gw + j * nwarps) * per_stage + lane * 4;
        int r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int c = base + k < m ? __ldcs(idx + base + k) : 0;
            cc[s][k] = c;
            r[k] = c / bw;
        }
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[w][s])),
                         "r"(kTile ? 32 * 8 * bw : 32 * 32 * bw)
                         : "memory");
        __syncwarp();
        if constexpr (kTile) {   // control: one plain 2-D tile load (one row) per lane
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4}], [%2];" ::"r"(sa(&buf[w][s][lane * 16])),
                "l"(&tm), "r"(sa(&bar[w][s])), "r"(0), "r"(r[0])
                : "memory");
            return;
        }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(sa(&buf[w][s][lane * 8])),
            "l"(&tm), "r"(sa(&bar[w][s])), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "l"(pol)
            : "memory");
    };
    long long nchunks = 0;
    {
        const long long total = (m + per_stage - 1) / per_stage;
        nchunks = gw < total ? (total - gw + nwarps - 1) / nwarps : 0;
    }
    for (long long j = 0; j < nchunks && j < S; ++j) issue(j, int(j));
    for (long long j = 0; j < nchunks; ++j, ++it) {
        const int s = int(j % S);
        const unsigned par = unsigned((j / S) & 1);
        unsigned ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(ok) : "r"(sa(&bar[w][s])), "r"(par) : "memory");
#pragma unroll
        for (int k = 0; k < (kTile ? 1 : 4); ++k) acc += buf[w][s][lane * 16 + k * bw + (cc[s][k] % bw)];
        __syncwarp();
        if (j + S < nchunks) issue(j + S, s);
    }
    if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
    const long long m = (argc > 1 ? atoll(argv[1]) : 134) * 1000000LL;
    const long long xmb = argc > 2 ? atoll(argv[2]) : 64;
    const int bw = argc > 3 ? atoi(argv[3]) : 2;      // box width (doubles per gathered row)
    const int bh = argc > 4 ? atoi(argv[4]) : 1;      // box height in the tensor map
    const int mode = argc > 5 ? atoi(argv[5]) : 2;    // 0: lsu only, 1: tma only, 2: both
    const int n = int(xmb * 1024 * 1024 / 8);
    double* x;
    int* idx;
    double* out;
    CK(cudaMalloc(&x, size_t(n) * 8));
    CK(cudaMalloc(&idx, size_t(m) * 4));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(x, 0, size_t(n) * 8));
    fill_idx<<<1024, 256>>>(idx, m, n);
    CK(cudaDeviceSynchronize());
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));

    // tensor map: x as [n/2 rows][2 doubles]
    typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t dims[2] = {cuuint64_t(bw), cuuint64_t(n / bw)};
    cuuint64_t strides[1] = {cuuint64_t(bw) * 8};
    cuuint32_t box[2] = {cuuint32_t(bw), cuuint32_t(bh)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncFn)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("cuTensorMapEncodeTiled failed %d\n", int(r));
        return 1;
    }
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](const char* name, auto launch) {
        launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(e0));
            launch();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf("%-28s x %4lld MB  %lld M gathers  %.3f ms  %.1f G gathers/s\n", name, xmb, m / 1000000, best,
               double(m) / (best * 1e-3) / 1e9);
    };
    printf("box %d x %d\n", bw, bh);
    for (int ctas : {4, 8}) {
        if (mode == 1) break;
        char nm[64];
        snprintf(nm, sizeof nm, "lsu nc.noL1 %d CTA/SM", ctas);
        timeit(nm, [&] { lsu_gather<<<sms * ctas, 256>>>(x, idx, m, out); });
    }
    auto run_tma = [&](auto kern, int S, int ctas) {
        const size_t smem = sizeof(double) * 4 * S * 32 * 16 + 8 * 4 * S + 128;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        char nm[64];
        snprintf(nm, sizeof nm, "tma gather4 S=%d %d CTA/SM", S, ctas);
        timeit(nm, [&] { kern<<<sms * ctas, 128, smem>>>(tm, idx, m, out, bw); });
    };
    if (mode == 3) {
        run_tma(tma_gather<4, true>, 4, 2);
        return 0;
    }
    for (int ctas : {1, 2, 3}) {
        if (mode == 0) break;
        run_tma(tma_gather<2>, 2, ctas);
        run_tma(tma_gather<4>, 4, ctas);
    }
    return 0;
}
