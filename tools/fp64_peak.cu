// FP64 throughput microbenchmarks for the roofline denominator:
//   k_dfma  - scalar DFMA, 8 independent chains per thread
//   k_dmma  - FP64 tensor core: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4 on sm_100a), 4 independent
//             accumulators per warp
// Built as a shared library (extern "C" entry points called from tools/fp64_peak.py); every
// launch is timed with CUDA events on the default stream.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = 1e-3 * (threadIdx.x + j);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == 12345.678) out[threadIdx.x] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) k_dmma(double* out, int iters, double a, double b) {
    const int lane = threadIdx.x & 31;
    double av = a + 1e-9 * lane, bv = b - 1e-9 * lane;
    double c[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) c[j][0] = c[j][1] = 1e-3 * (lane + j);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[j][0]), "+d"(c[j][1])
                             : "d"(av), "d"(bv));
        }
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

extern "C" {
// kind 0 = DFMA, 1 = DMMA.  Returns milliseconds of one launch of `blocks` x 256 threads, or < 0.
double fp64_run(int kind, int blocks, int iters) {
    double* out = nullptr;
    if (cudaMalloc(&out, 256 * sizeof(double)) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    if (kind == 0)
        k_dfma<<<blocks, 256>>>(out, iters, 0.9999999, 1e-7);
    else
        k_dmma<<<blocks, 256>>>(out, iters, 0.25, 1e-7);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = -1.f;
    if (err == cudaSuccess && cudaGetLastError() == cudaSuccess) cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return ms;
}
// flops of one launch
double fp64_flops(int kind, int blocks, int iters) {
    const double threads = (double)blocks * 256;
    if (kind == 0) return threads * iters * 8 * 8 * 2.0;            // 64 DFMA per iteration
    return threads / 32.0 * iters * 8 * 4 * (2.0 * 8 * 8 * 4);     // 32 MMA m8n8k4 per iteration per warp
}
}
