// Where does the random-gather ceiling of C4's y_L come from?  134M random
// 8-byte LDG gathers (8 in flight per thread, one 1024-thread CTA per SM) while varying
// (a) the gathered vector's size (L1-resident .. beyond L2), (b) the number of
// SMs the grid occupies (per-SM limit vs a global L2 limit), (c) the load's
// L1 / L2 cache policy (PTX qualifiers).
// With a file argument: the gather pattern is read from it (int32 ids into a
// 2^23-double x; e.g. C4's col array), with and without an L2 flush.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_gather_scope.cu -o ubench_gather_scope
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

// MODE 0: ld.global.nc.L1::no_allocate   1: ld.global.nc (L1 allocate)
//      2: ld.global.nc.L1::no_allocate.L2::cache_hint(evict_last)
//      3: ld.global.nc.L2::cache_hint(evict_last)   4: ld.global (coherent path)
//      5: ld.global.nc.L1::evict_last
template <int MODE>
__global__ void ldg_kernel(const double* __restrict__ x, const int* __restrict__ idx, long n_idx, int mask, double* out) {
    double acc = 0;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const long stride = (long)gridDim.x * blockDim.x;
    long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n_idx; i += 8 * stride) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const double* p = x + (idx[i + k * stride] & mask);
            if (MODE == 0) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[k]) : "l"(p));
            else if (MODE == 1) asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v[k]) : "l"(p));
            else if (MODE == 2) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[k]) : "l"(p), "l"(pol));
            else if (MODE == 3) asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[k]) : "l"(p), "l"(pol));
            else if (MODE == 4) asm volatile("ld.global.f64 %0, [%1];" : "=d"(v[k]) : "l"(p));
            else asm volatile("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v[k]) : "l"(p));
        }
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
    if (argc > 1) {  // gather pattern from a file of int32 column ids (e.g. C4's CSR col array), x of 2^23 doubles
        FILE* f = fopen(argv[1], "rb");
        if (!f) { printf("cannot open %s\n", argv[1]); return 1; }
        fseek(f, 0, SEEK_END); const long bytes = ftell(f); fseek(f, 0, SEEK_SET);
        const long m = bytes / 4;
        std::vector<int> hc(m);
        if (fread(hc.data(), 4, m, f) != size_t(m)) return 1;
        fclose(f);
        const long n = 1L << 23;
        double *x, *out; int* idx; uint4* fb;
        const long fbytes = 512L << 20;
        CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&idx, m * 4)); CK(cudaMalloc(&fb, fbytes));
        CK(cudaMemset(x, 0, n * 8)); CK(cudaMemset(fb, 1, fbytes));
        CK(cudaMemcpy(idx, hc.data(), m * 4, cudaMemcpyHostToDevice));
        int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        CK(cudaFuncSetAttribute(ldg_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        CK(cudaFuncSetAttribute(ldg_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        CK(cudaFuncSetAttribute(ldg_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        CK(cudaFuncSetAttribute(ldg_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024));
        const char* names[4] = {"nc.L1noalloc", "nc", "nc.L1noalloc.L2hint", "nc.L2hint"};
        for (int mode = 0; mode < 4; ++mode)
            for (int flush = 0; flush < 2; ++flush)
                for (int threads : {256, 512, 1024}) {
                    float ms = 0;
                    for (int rep = 0; rep < 3; ++rep) {
                        if (flush) flush_l2<<<sms * 4, 512>>>(fb, fbytes / 16, reinterpret_cast<unsigned*>(out));
                        cudaEventRecord(a);
                        switch (mode) {
                            case 0: ldg_kernel<0><<<sms, threads, 120 * 1024>>>(x, idx, m, int(n - 1), out); break;
                            case 1: ldg_kernel<1><<<sms, threads, 120 * 1024>>>(x, idx, m, int(n - 1), out); break;
                            case 2: ldg_kernel<2><<<sms, threads, 120 * 1024>>>(x, idx, m, int(n - 1), out); break;
                            default: ldg_kernel<3><<<sms, threads, 120 * 1024>>>(x, idx, m, int(n - 1), out); break;
                        }
                        cudaEventRecord(b);
                        CK(cudaEventSynchronize(b));
                    }
                    CK(cudaGetLastError());
                    cudaEventElapsedTime(&ms, a, b);
                    printf("file-pattern %ld gathers  warps/SM %2d  %-20s L2 %s  %8.3f ms  %6.1f G gathers/s\n", m,
                           threads / 32, names[mode], flush ? "flushed" : "warm   ", ms, m / ms / 1e6);
                }
        return 0;
    }
    const long nmax = 1L << 25;         // 32M doubles = 256 MB
    const long n_idx = 1L << 27;        // 134M gathers
    std::vector<int> h(n_idx);
    uint64_t z = 12345;
    for (long i = 0; i < n_idx; ++i) { z ^= z << 13; z ^= z >> 7; z ^= z << 17; h[i] = (int)(z % nmax); }
    double *x, *out; int* idx;
    CK(cudaMalloc(&x, nmax * 8)); CK(cudaMalloc(&out, 8)); CK(cudaMalloc(&idx, n_idx * 4));
    CK(cudaMemset(x, 0, nmax * 8));
    CK(cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice));
    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms = 0;
    const char* names[6] = {"nc.L1noalloc", "nc", "nc.L1noalloc.L2hint", "nc.L2hint", "ld.global", "nc.L1evlast"};
    auto run = [&](const char* tag, long n, int nsm, int mode) {
        const int grid = nsm;  // one 1024-thread CTA per SM (120 KB smem forces 1 CTA/SM)
        const int mask = int(n - 1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            switch (mode) {
                case 0: ldg_kernel<0><<<grid, 1024, 120 * 1024>>>(x, idx, n_idx, mask, out); break;
                case 1: ldg_kernel<1><<<grid, 1024, 120 * 1024>>>(x, idx, n_idx, mask, out); break;
                case 2: ldg_kernel<2><<<grid, 1024, 120 * 1024>>>(x, idx, n_idx, mask, out); break;
                case 3: ldg_kernel<3><<<grid, 1024, 120 * 1024>>>(x, idx, n_idx, mask, out); break;
                case 4: ldg_kernel<4><<<grid, 1024, 120 * 1024>>>(x, idx, n_idx, mask, out); break;
                default: ldg_kernel<5><<<grid, 1024, 120 * 1024>>>(x, idx, n_idx, mask, out); break;
            }
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
        }
        CK(cudaGetLastError());
        cudaEventElapsedTime(&ms, a, b);
        printf("%-5s x %7.2f MB  SMs %3d  %-20s %8.3f ms  %6.1f G gathers/s  %.3f per SM-clock@1.965GHz\n", tag,
               n * 8 / 1e6, nsm, names[mode], ms, n_idx / ms / 1e6, n_idx / (ms * 1e-3) / (nsm * 1.965e9));
    };
#define SETSMEM(M) CK(cudaFuncSetAttribute(ldg_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024))
    SETSMEM(0); SETSMEM(1); SETSMEM(2); SETSMEM(3); SETSMEM(4); SETSMEM(5);
    for (int mode = 0; mode < 6; ++mode)
        for (long n : {1L << 18, 1L << 21, 1L << 23, 1L << 24}) run("size", n, sms, mode);
    for (int mode : {0, 1, 3})
        for (int nsm : {sms / 2, sms / 4}) run("sms", 1L << 23, nsm, mode);
    // order check: the first configuration again at the end
    run("again", 1L << 23, sms, 0);
    run("again", 1L << 23, sms, 1);
    return 0;
}
