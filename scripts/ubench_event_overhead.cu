// Microbenchmark: what a START/END CUDA-event pair around one ~30 us kernel
// adds, (a) recorded on a stream around a plain launch, (b) as external
// event-record nodes inside a captured CUDA graph, (c) on the stream around a
// graph launch.  The kernel stamps %globaltimer at entry/exit of CTA 0, so
// overhead = event interval - kernel interval.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 ubench_event_overhead.cu -o ubench_event_overhead
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void spin(unsigned long long ns, unsigned long long* stamp) {
    const unsigned long long t0 = gt();
    if (threadIdx.x == 0 && blockIdx.x == 0) stamp[0] = t0;
    while (gt() - t0 < ns) {}
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) stamp[1] = gt();
}
int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    unsigned long long* d;
    cudaMalloc(&d, 16);
    unsigned long long h[2];
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const unsigned long long ns = 30000;
    auto report = [&](const char* name, auto body) {
        std::vector<float> ov, tot;
        for (int i = 0; i < 220; ++i) {
            body();
            cudaStreamSynchronize(s);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            if (i >= 20) {
                tot.push_back(ms * 1e3f);
                ov.push_back(ms * 1e3f - (h[1] - h[0]) * 1e-3f);
            }
        }
        std::sort(ov.begin(), ov.end());
        std::sort(tot.begin(), tot.end());
        printf("%-44s interval median %6.2f us, overhead median %5.2f us (p10 %5.2f, p90 %5.2f)\n", name,
               tot[tot.size() / 2], ov[ov.size() / 2], ov[ov.size() / 10], ov[ov.size() * 9 / 10]);
    };
    report("stream: record, launch, record", [&] {
        cudaEventRecord(a, s);
        spin<<<148, 128, 0, s>>>(ns, d);
        cudaEventRecord(b, s);
    });
    // graph with external event nodes
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaEventRecordWithFlags(a, s, cudaEventRecordExternal);
    spin<<<148, 128, 0, s>>>(ns, d);
    cudaEventRecordWithFlags(b, s, cudaEventRecordExternal);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    report("graph: ext-record node, kernel, ext-record", [&] { cudaGraphLaunch(ge, s); });
    // graph of only the kernel, events on the stream
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    spin<<<148, 128, 0, s>>>(ns, d);
    cudaStreamEndCapture(s, &g2);
    cudaGraphInstantiate(&ge2, g2, 0);
    report("stream: record, graph launch, record", [&] {
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge2, s);
        cudaEventRecord(b, s);
    });
    // same, after a preceding busy kernel (host runs ahead: launch latency hidden)
    report("stream: spin, record, graph launch, record", [&] {
        spin<<<148, 128, 0, s>>>(ns, d + 0);
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge2, s);
        cudaEventRecord(b, s);
    });
    report("stream: spin, record, launch, record", [&] {
        spin<<<148, 128, 0, s>>>(ns, d + 0);
        cudaEventRecord(a, s);
        spin<<<148, 128, 0, s>>>(ns, d);
        cudaEventRecord(b, s);
    });
    report("graph after spin: ext node, kernel, ext node", [&] {
        spin<<<148, 128, 0, s>>>(ns, d + 0);
        cudaGraphLaunch(ge, s);
    });
    return 0;
}
