// Pure-read HBM bandwidth on B200 (the roofline of the read-dominated SpMV
// stream, beside MEASURED_PEAKS.json's copy figure): 128-bit LDG streaming
// with a grid-stride loop, and 1-D TMA bulk copies into a shared-memory ring
// (the row-block kernel's producer pattern), over a buffer far larger than L2.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o urb scripts/ubench_read_bw.cu
//   ./urb [GB=6]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);            \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__global__ void __launch_bounds__(512) ldg_read(const uint4* __restrict__ p, long long n16, unsigned* sink) {
    unsigned acc = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
        acc ^= a.x ^ b.y ^ c.z ^ d.w;
    }
    for (; i < n16; i += stride) acc ^= __ldcs(p + i).x;
    if (acc == 0x12345678u) sink[0] = acc;
}

__device__ __forceinline__ uint32_t sa(const void* q) { return static_cast<uint32_t>(__cvta_generic_to_shared(q)); }

// one elected thread per CTA streams CHUNK-byte pieces into S ring slots;
// the other warps only release slots (no compute): the TMA read ceiling
template <int S, int CHUNK>
__global__ void __launch_bounds__(64) tma_read(const char* __restrict__ p, long long bytes, unsigned* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* base = sm + ((128 - (sa(sm) & 127)) & 127);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + S * CHUNK);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long nchunks = bytes / CHUNK;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    long long it = 0;
    unsigned acc = 0;
    for (long long c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = int(it % S);
        if (it >= S) {   // wait for the copy issued S iterations ago
            unsigned ok = 0;
            const unsigned par = unsigned(((it - S) / S) & 1);
            while (!ok)
                asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
                             : "=r"(ok) : "r"(sa(&full[s])), "r"(par) : "memory");
            acc ^= base[s * CHUNK];
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(CHUNK) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
            ::"r"(sa(base + s * CHUNK)), "l"(p + c * CHUNK), "r"(CHUNK), "r"(sa(&full[s])), "l"(pol) : "memory");
    }
    for (long long j = it > S ? it - S : 0; j < it; ++j) {
        unsigned ok = 0;
        const int s = int(j % S);
        const unsigned par = unsigned((j / S) & 1);
        while (!ok)
            asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q; }"
                         : "=r"(ok) : "r"(sa(&full[s])), "r"(par) : "memory");
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

int main(int argc, char** argv) {
    const double gb = argc > 1 ? atof(argv[1]) : 6.0;
    const long long bytes = (long long)(gb * 1e9) / 65536 * 65536;
    char* p;
    unsigned* sink;
    CK(cudaMalloc(&p, bytes));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(p, 1, bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto timeit = [&](const char* name, auto launch) {
        launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            CK(cudaEventRecord(a));
            launch();
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = ms < best ? ms : best;
        }
        printf("%-36s %.2f GB  %.3f ms  %.1f GB/s\n", name, bytes / 1e9, best, bytes / (best * 1e-3) / 1e9);
    };
    for (int ctas : {2, 4}) {
        char nm[64];
        snprintf(nm, sizeof nm, "ldg.128 %d x 512 thr/SM", ctas);
        timeit(nm, [&] { ldg_read<<<sms * ctas, 512>>>(reinterpret_cast<const uint4*>(p), bytes / 16, sink); });
    }
    auto tma = [&](auto kern, int S, int chunk, int ctas) {
        const int smem = S * chunk + 8 * S + 128;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        char nm[64];
        snprintf(nm, sizeof nm, "tma bulk %dx%dKB, %d CTA/SM", S, chunk / 1024, ctas);
        timeit(nm, [&] { kern<<<sms * ctas, 64, smem>>>(p, bytes, sink); });
    };
    tma(tma_read<4, 16384>, 4, 16384, 2);
    tma(tma_read<4, 16384>, 4, 16384, 3);
    tma(tma_read<8, 8192>, 8, 8192, 2);
    tma(tma_read<6, 32768>, 6, 32768, 1);
    return 0;
}
