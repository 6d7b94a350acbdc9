// Kernel stores into mapped pinned host memory (the zero-copy y of
// dspmv_apply_host) on B200: achieved GB/s by store width, alone and while a
// copy engine moves the same number of bytes host->device (x of the next
// chunk).  Question: is the e2e leg bound by SM-issued PCIe writes?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o uz scripts/ubench_zerocopy.cu
//   ./uz [MB=134]
#include <cuda_runtime.h>

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

template <int W>   // bytes per thread per store: 8, 16, 32
__global__ void store_kernel(double* __restrict__ out, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    constexpr int E = W / 8;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i * E < n; i += stride) {
        if constexpr (E == 1) {
            __stcs(out + i, double(i));
        } else if constexpr (E == 2) {
            __stcs(reinterpret_cast<double2*>(out) + i, make_double2(double(i), 1.0));
        } else {
            double2* p = reinterpret_cast<double2*>(out) + 2 * i;
            __stcs(p, make_double2(double(i), 1.0));
            __stcs(p + 1, make_double2(2.0, 3.0));
        }
    }
}

int main(int argc, char** argv) {
    const long long mb = argc > 1 ? atoll(argv[1]) : 134;
    const size_t bytes = size_t(mb) << 20;
    const long long n = bytes / 8;
    double *h_y, *d_y_map, *h_x, *d_x;
    CK(cudaHostAlloc(&h_y, bytes, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(&d_y_map, h_y, 0));
    CK(cudaHostAlloc(&h_x, bytes, cudaHostAllocDefault));
    CK(cudaMalloc(&d_x, bytes));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    auto run = [&](const char* name, auto launch, bool with_h2d) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(a, s1));
            CK(cudaStreamWaitEvent(s2, a, 0));
            if (with_h2d) CK(cudaMemcpyAsync(d_x, h_x, bytes, cudaMemcpyHostToDevice, s2));
            launch();
            CK(cudaGetLastError());
            cudaEvent_t c;
            CK(cudaEventCreate(&c));
            CK(cudaEventRecord(c, s2));
            CK(cudaStreamWaitEvent(s1, c, 0));
            CK(cudaEventRecord(b, s1));
            CK(cudaEventSynchronize(b));
            CK(cudaEventDestroy(c));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = ms < best ? ms : best;
        }
        printf("%-40s %lld MB  %.3f ms  %.1f GB/s (kernel bytes)\n", name, mb, best, bytes / (best * 1e-3) / 1e9);
    };
    for (int h2d = 0; h2d < 2; ++h2d) {
        char nm[80];
        snprintf(nm, sizeof nm, "zero-copy st 8B/thread%s", h2d ? " + concurrent H2D" : "");
        run(nm, [&] { store_kernel<8><<<sms * 8, 256, 0, s1>>>(d_y_map, n); }, h2d);
        snprintf(nm, sizeof nm, "zero-copy st 16B/thread%s", h2d ? " + concurrent H2D" : "");
        run(nm, [&] { store_kernel<16><<<sms * 8, 256, 0, s1>>>(d_y_map, n); }, h2d);
        snprintf(nm, sizeof nm, "zero-copy st 32B/thread%s", h2d ? " + concurrent H2D" : "");
        run(nm, [&] { store_kernel<32><<<sms * 8, 256, 0, s1>>>(d_y_map, n); }, h2d);
    }
    run("H2D copy alone", [&] {}, true);
    return 0;
}
