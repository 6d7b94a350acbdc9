// (gather warps per CTA and CTAs per SM vary; 1 x 31 matches ubench_gather_scope's 1024-thread CTAs)
// Do C4's random x gathers slow down when a TMA bulk stream of the matrix
// runs beside them?  Grid of 2 CTAs/SM; each CTA = 1 streamer warp (lane 0
// issues 12 KB cp.async.bulk chunks of a 1.78 GB buffer, L2 evict_first,
// through a 3-slot shared-memory ring) + 8 gather warps (C4's col pattern
// from a file, ld.global.nc.L1::no_allocate.L2::cache_hint evict_last, 8 in
// flight per thread).  Modes: gathers only, stream only, both.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_gather_stream.cu -o ugst
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int CHUNK = 12 * 1024, RING = 3;

__global__ void __launch_bounds__(1024) both_kernel(const double* __restrict__ x, const int* __restrict__ idx,
                                                             long n_idx, const char* __restrict__ mat, long mat_bytes,
                                                             int do_gather, int do_stream, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + RING * CHUNK);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int GW = blockDim.x / 32 - 1;  // gather warps; the last warp streams
    if (threadIdx.x == 0) {
        for (int s = 0; s < RING; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (warp == GW) {
        if (!do_stream || lane) return;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        const long nch = mat_bytes / CHUNK;
        int it = 0;
        for (long c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
            const int s = it % RING;
            if (it >= RING) {  // wait for this slot's previous chunk
                const uint32_t par = ((it / RING) - 1) & 1;
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(ok) : "r"(sa(&bar[s])), "r"(par));
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(CHUNK));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                         ::"r"(sa(sm + s * CHUNK)), "l"(mat + c * CHUNK), "r"(CHUNK), "r"(sa(&bar[s])), "l"(pol) : "memory");
        }
        // drain
        for (int k = 0; k < RING && k < it; ++k) {
            const int j = it - 1 - k, s = j % RING;
            const uint32_t par = (j / RING) & 1;
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok) : "r"(sa(&bar[s])), "r"(par));
        }
        return;
    }
    if (!do_gather) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    double acc = 0;
    const long stride = (long)gridDim.x * GW * 32;
    long i = (long)blockIdx.x * GW * 32 + threadIdx.x;
    for (; i + 7 * stride < n_idx; i += 8 * stride) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[k]) : "l"(x + idx[i + k * stride]), "l"(pol));
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 12345.0) out[0] = acc;
}

__global__ void flush_l2(const uint4* buf, long n16, unsigned* sink) {
    unsigned acc = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(buf + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345u) sink[0] = acc;
}

int main(int argc, char** argv) {
    if (argc < 2) { printf("usage: ugst col.bin\n"); return 1; }
    FILE* f = fopen(argv[1], "rb");
    fseek(f, 0, SEEK_END); const long m = ftell(f) / 4; fseek(f, 0, SEEK_SET);
    std::vector<int> hc(m);
    if (fread(hc.data(), 4, m, f) != size_t(m)) return 1;
    fclose(f);
    const long n = 1L << 23, mat_bytes = 1776L << 20, fbytes = 512L << 20;
    double *x, *out; int* idx; char* mat; uint4* fb;
    CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&idx, m * 4));
    CK(cudaMalloc(&mat, mat_bytes)); CK(cudaMalloc(&fb, fbytes));
    CK(cudaMemset(x, 0, n * 8)); CK(cudaMemset(mat, 1, mat_bytes)); CK(cudaMemset(fb, 1, fbytes));
    CK(cudaMemcpy(idx, hc.data(), m * 4, cudaMemcpyHostToDevice));
    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int smem = RING * CHUNK + 64;
    CK(cudaFuncSetAttribute(both_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[3] = {"gathers only", "stream only ", "both        "};
    const int cfgs[][2] = {{1, 31}, {1, 15}, {1, 11}, {1, 7}, {2, 15}, {2, 11}, {2, 8}, {3, 10}, {4, 7}, {6, 4}, {8, 3}};
    const int nm = argc > 2 ? 1 : 3;  // argv[2]: gathers only
    for (auto& cf : cfgs) for (int mode = 0; mode < nm; ++mode) {
        const int ctas = cf[0], GW = cf[1];
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            flush_l2<<<sms * 4, 512>>>(fb, fbytes / 16, reinterpret_cast<unsigned*>(out));
            cudaEventRecord(a);
            if (argc > 3) {  // argv[3]: grid = sms*ctas CTAs but only sms*ctas/2 launched... (unused)
            }
            both_kernel<<<sms * ctas, 32 * (GW + 1), smem>>>(x, idx, m, mat, mat_bytes, mode != 1, mode != 0, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
        }
        CK(cudaGetLastError());
        cudaEventElapsedTime(&ms, a, b);
        printf("%d CTAs/SM (%2d gather warps/SM)  %s  %8.3f ms   gathers %6.1f G/s   stream %6.1f GB/s\n", ctas, ctas * GW,
               names[mode], ms, mode != 1 ? m / ms / 1e6 : 0.0, mode != 0 ? mat_bytes / ms / 1e6 : 0.0);
    }
    return 0;
}
