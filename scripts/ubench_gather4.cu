// Microbenchmark: random gathers of 8-byte x values (64 MB vector, random
// indices) through (a) LDG (ld.global.nc, L1::no_allocate) from many warps and
// (b) TMA tile::gather4 (x viewed as [n/2][2] doubles, 16-B rows) issued by one
// warp per CTA into a shared-memory ring.  Reports gathered elements / s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_gather4.cu -o ubench_gather4
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void ldg_kernel(const double* __restrict__ x, const int* __restrict__ idx, long n_idx, double* out) {
    double acc = 0;
    const long stride = (long)gridDim.x * blockDim.x;
    long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n_idx; i += 8 * stride) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double* p = x + idx[i + k * stride];
            asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[k]) : "l"(p));
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc += v[k];
    }
    if (acc == 12345.0) out[0] = acc;
}

constexpr int RING = 4;           // slots (each 1024 gathers x 32 B)
constexpr int PER_SLOT = 256;      // gather4 per slot per warp-lane batch -> 1024 elements

__global__ void __launch_bounds__(64) g4_kernel(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                long n_idx, double* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    double4* buf = reinterpret_cast<double4*>(sm);                       // RING * 1024 * 32 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + RING * 1024 * 32);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int s = 0; s < RING; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const long chunks = n_idx / 1024;
    double acc = 0;
    if (warp == 0) {
        int it = 0;
        for (long c = blockIdx.x; c < chunks; c += gridDim.x, ++it) {
            const int s = it % RING;
            if (it >= RING) {  // wait until consumer (warp 1) drained this slot: simple phase tracking
                uint32_t ok = 0;
                const uint32_t par = ((it / RING) - 1) & 1;
                // consumer signals by flipping a flag in smem; keep it simple: reuse bar of slot after consume
                while (!ok) {
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                                 : "=r"(ok) : "r"(sa(&bar[s])), "r"(par ^ 1 ^ 1));
                }
            }
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(1024 * 32));
            __syncwarp();
            const int* ix = idx + c * 1024;
            for (int g = lane; g < PER_SLOT; g += 32) {
                const int r0 = ix[4 * g] >> 2, r1 = ix[4 * g + 1] >> 2, r2 = ix[4 * g + 2] >> 2, r3 = ix[4 * g + 3] >> 2;
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(&buf[s * 1024 + 4 * g])),
                    "l"(&tm), "r"(sa(&bar[s])), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                    : "memory");
            }
        }
    } else {
        int it = 0;
        for (long c = blockIdx.x; c < chunks; c += gridDim.x, ++it) {
            const int s = it % RING;
            const uint32_t par = (it / RING) & 1;
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok) : "r"(sa(&bar[s])), "r"(par));
            for (int e = lane; e < 1024; e += 32) acc += buf[s * 1024 + e].x;
            __syncwarp();
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

int main(int argc, char** argv) {
    const long n = 1L << 23;            // 8M doubles = 64 MB
    const long n_idx = 1L << 27;        // 134M gathers
    std::vector<int> h(n_idx);
    uint64_t z = 12345;
    for (long i = 0; i < n_idx; ++i) {
        z ^= z << 13; z ^= z >> 7; z ^= z << 17;
        h[i] = (int)(z % n);
    }
    double *x, *out;
    int* idx;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&out, 8));
    CK(cudaMalloc(&idx, n_idx * 4));
    CK(cudaMemset(x, 0, n * 8));
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    // LDG
    for (int warps : {8, 16, 32}) {
        const int grid = sms * (warps * 32 / 256);
        ldg_kernel<<<grid, 256>>>(x, idx, n_idx, out);
        cudaEventRecord(a);
        ldg_kernel<<<grid, 256>>>(x, idx, n_idx, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("LDG   %2d warps/SM: %.3f ms  %.1f G gathers/s\n", warps, ms, n_idx / ms / 1e6);
    }
    // TMA gather4
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap tm;
    cuuint64_t gdim[2] = {4, (cuuint64_t)(n / 4)};
    cuuint64_t gstr[1] = {32};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
    }
    const int smem = RING * 1024 * 32 + RING * 8;
    CK(cudaFuncSetAttribute(g4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int ctas : {1}) {  // one CTA per SM (ring uses ~128 KB)
        g4_kernel<<<sms * ctas, 64, smem>>>(tm, idx, n_idx, out);
        CK(cudaGetLastError());
        cudaEventRecord(a);
        g4_kernel<<<sms * ctas, 64, smem>>>(tm, idx, n_idx, out);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        printf("TMA g4 %d CTA/SM: %.3f ms  %.1f G gathers/s\n", ctas, ms, n_idx / ms / 1e6);
    }
    return 0;
}
