// Cost of external event-record nodes around a kernel inside a CUDA graph:
// START..END of a captured [rec START] -> [rec t0]? -> kernel -> [rec t1]? -> [rec END]
// vs the kernel's own duration, with an L2-flush kernel queued before each launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_graph_events.cu -o uge
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, long n) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void flush_k(const uint4* buf, long n16, unsigned* sink) {
    unsigned acc = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(buf + i); acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x1234567u) sink[0] = acc;
}

int main() {
    const long n = (110L << 20) / 32;  // 110 MB copied: ~34 us at ~6.5 TB/s (read + write)
    double4 *a, *b; uint4* fb; unsigned* sink;
    const long fbytes = 256L << 20;
    CK(cudaMalloc(&a, n * 32)); CK(cudaMalloc(&b, n * 32)); CK(cudaMalloc(&fb, fbytes)); CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(a, 0, n * 32)); CK(cudaMemset(fb, 0, fbytes));
    cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, t0, t1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&t0)); CK(cudaEventCreate(&t1));
    cudaStream_t s2; CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t f0, f1; CK(cudaEventCreateWithFlags(&f0, cudaEventDisableTiming)); CK(cudaEventCreateWithFlags(&f1, cudaEventDisableTiming));
    for (int variant = 0; variant < 7; ++variant) {
        // 0: no graph (stream launches); 1: graph [START, kernel, END]; 2: graph [START, t0, kernel, t1, END];
        // 3: graph [START, kernel, t1, END]; 4: stream launches with t0/t1 records;
        // 5: stream, t0/t1 + fork/join of an empty second stream; 6: graph of variant 5
        cudaGraphExec_t ge = nullptr;
        if (variant == 6) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            CK(cudaEventRecordWithFlags(e0, s, cudaEventRecordExternal));
            CK(cudaEventRecord(f0, s)); CK(cudaStreamWaitEvent(s2, f0, 0));
            CK(cudaEventRecordWithFlags(t0, s, cudaEventRecordExternal));
            copy_k<<<148 * 8, 256, 0, s>>>(a, b, n);
            CK(cudaEventRecordWithFlags(t1, s, cudaEventRecordExternal));
            CK(cudaEventRecord(f1, s2)); CK(cudaStreamWaitEvent(s, f1, 0));
            CK(cudaEventRecordWithFlags(e1, s, cudaEventRecordExternal));
            CK(cudaStreamEndCapture(s, &g));
            CK(cudaGraphInstantiate(&ge, g, 0));
        } else if (variant > 0 && variant < 4) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            CK(cudaEventRecordWithFlags(e0, s, cudaEventRecordExternal));
            if (variant == 2) CK(cudaEventRecordWithFlags(t0, s, cudaEventRecordExternal));
            copy_k<<<148 * 8, 256, 0, s>>>(a, b, n);
            if (variant >= 2) CK(cudaEventRecordWithFlags(t1, s, cudaEventRecordExternal));
            CK(cudaEventRecordWithFlags(e1, s, cudaEventRecordExternal));
            CK(cudaStreamEndCapture(s, &g));
            CK(cudaGraphInstantiate(&ge, g, 0));
        }
        std::vector<float> st, kt;
        for (int it = 0; it < 220; ++it) {
            flush_k<<<148 * 4, 512, 0, s>>>(fb, fbytes / 16, sink);
            if (variant == 0) {
                CK(cudaEventRecord(e0, s));
                copy_k<<<148 * 8, 256, 0, s>>>(a, b, n);
                CK(cudaEventRecord(e1, s));
            } else if (variant == 4 || variant == 5) {
                CK(cudaEventRecord(e0, s));
                if (variant == 5) { CK(cudaEventRecord(f0, s)); CK(cudaStreamWaitEvent(s2, f0, 0)); }
                CK(cudaEventRecord(t0, s));
                copy_k<<<148 * 8, 256, 0, s>>>(a, b, n);
                CK(cudaEventRecord(t1, s));
                if (variant == 5) { CK(cudaEventRecord(f1, s2)); CK(cudaStreamWaitEvent(s, f1, 0)); }
                CK(cudaEventRecord(e1, s));
            } else {
                CK(cudaGraphLaunch(ge, s));
            }
            CK(cudaEventSynchronize(e1));
            float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
            if (it >= 20) st.push_back(ms * 1e3f);
            if (variant == 2 || variant >= 4) { CK(cudaEventElapsedTime(&ms, t0, t1)); if (it >= 20) kt.push_back(ms * 1e3f); }
        }
        std::sort(st.begin(), st.end());
        printf("variant %d: START..END median %.2f us", variant, st[st.size() / 2]);
        if (!kt.empty()) { std::sort(kt.begin(), kt.end()); printf("   t0..t1 median %.2f us", kt[kt.size() / 2]); }
        printf("\n");
    }
    return 0;
}
