// Plain CSR y = A x on C4's matrix without shared-memory staging, to compare
// with the TMA-staged y_L kernel: L lanes per row (L = 1, 2, 4), each lane
// loading its own col/val entries from global memory and keeping CH gathers
// in flight; rows of a warp are consecutive.  Matrix from files written by
// scripts/diag_c4_naive.sh (rowptr int32, col int32, val f64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ubench_csr_naive.cu -o ucsr
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <class T> std::vector<T> rd(const char* p) {
    FILE* f = fopen(p, "rb"); fseek(f, 0, SEEK_END); long b = ftell(f); fseek(f, 0, SEEK_SET);
    std::vector<T> v(b / sizeof(T)); if (fread(v.data(), 1, b, f) != size_t(b)) exit(1); fclose(f); return v;
}

template <int L, int CH>
__global__ void __launch_bounds__(256) csr_kernel(const int* __restrict__ rp, const int* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ x,
                                                  double* __restrict__ y, int n) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const int lane = threadIdx.x & 31, sub = lane & (L - 1);
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (int rb = gw * (32 / L); rb < n; rb += nw * (32 / L)) {
        const int r = rb + lane / L;
        double acc = 0.0;
        if (r < n) {
            const int e0 = __ldcs(rp + r), e1 = __ldcs(rp + r + 1);
            for (int q = e0 + sub; q < e1; q += CH * L) {
                int c[CH]; double v[CH], xv[CH];
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    const int qq = min(q + k * L, e1 - 1);
                    c[k] = __ldcs(col + qq); v[k] = q + k * L < e1 ? __ldcs(val + qq) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < CH; ++k)
                    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(xv[k]) : "l"(x + c[k]), "l"(pol));
#pragma unroll
                for (int k = 0; k < CH; ++k) acc += v[k] * xv[k];
            }
        }
#pragma unroll
        for (int off = L / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (r < n && sub == 0) __stcs(y + r, acc);
    }
}

__global__ void flush_l2(const uint4* buf, long n16, unsigned* sink) {
    unsigned acc = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n16; i += (long)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(buf + i); acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345u) sink[0] = acc;
}

int main() {
    auto hrp = rd<int>("/tmp/c4rp.bin"); auto hcol = rd<int>("/tmp/c4col.bin"); auto hval = rd<double>("/tmp/c4val.bin");
    const int n = int(hrp.size()) - 1; const long nnz = long(hcol.size());
    int *rp, *col; double *val, *x, *y; uint4* fb; unsigned* sink;
    const long fbytes = 512L << 20;
    CK(cudaMalloc(&rp, hrp.size() * 4)); CK(cudaMalloc(&col, nnz * 4)); CK(cudaMalloc(&val, nnz * 8));
    CK(cudaMalloc(&x, n * 8L)); CK(cudaMalloc(&y, n * 8L)); CK(cudaMalloc(&fb, fbytes)); CK(cudaMalloc(&sink, 64));
    CK(cudaMemcpy(rp, hrp.data(), hrp.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(col, hcol.data(), nnz * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(val, hval.data(), nnz * 8, cudaMemcpyHostToDevice));
    CK(cudaMemset(x, 0, n * 8L)); CK(cudaMemset(fb, 1, fbytes));
    int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern) {
        for (int bps : {4, 8}) {
            std::vector<float> t;
            for (int rep = 0; rep < 7; ++rep) {
                flush_l2<<<sms * 4, 512>>>(fb, fbytes / 16, sink);
                cudaEventRecord(a);
                kern<<<sms * bps, 256>>>(rp, col, val, x, y, n);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                float ms; cudaEventElapsedTime(&ms, a, b); t.push_back(ms);
            }
            CK(cudaGetLastError());
            std::sort(t.begin(), t.end());
            const double bytes = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n;
            printf("%-22s %d CTAs/SM (%2d warps/SM): %.3f ms  %.0f GB/s  %.1f G gathers/s\n", name, bps, bps * 8, t[3],
                   bytes / t[3] / 1e6, nnz / t[3] / 1e6);
        }
    };
    run("1 lane/row, 8 in flight", csr_kernel<1, 8>);
    run("1 lane/row, 16 in flight", csr_kernel<1, 16>);
    run("2 lanes/row, 8 in flight", csr_kernel<2, 8>);
    run("4 lanes/row, 4 in flight", csr_kernel<4, 4>);
    run("4 lanes/row, 8 in flight", csr_kernel<4, 8>);
    return 0;
}
