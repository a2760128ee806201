// Microbenchmark of the column-per-thread chunk append (dh2_cq.cu): cycles per reflection step
// at k = 125 for 1..CTAS resident CTAs per SM.  build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -std=c++17 -I paper_1809_04384_b200/csrc tools/cq_bench.cu -o /tmp/cq_bench
#include <cstdio>
#include <vector>
#include "dh2_cq.cu"

namespace dh2 {
template <int NB, int NC, int CT, int CH>
__global__ void __launch_bounds__(128 / NC, CT) k_cq_bench(double2* scr, const double2* in, int k, int nch) {
    __shared__ CqRefl<NB> sh;
    double2 b[NC][NB];
    double2* Rs = scr + (size_t)blockIdx.x * k * CQ_KP;
    for (int q = 0; q < nch; ++q) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int i = 0; i < NB; ++i)
                b[c][i] = in[((size_t)(q % 8) * NB + i) * 128 + cq_col<NC>(c)];
        cq_append<NB, NC, CH>(b, Rs, k, q == 0, sh);
    }
}
// dependent-chain latencies (one thread): DFMA, DADD, rsqrt, sqrt, division, __drcp_rn, LDS+STS
__global__ void k_lat(double* out, double x0, long long* cyc) {
    double x = x0, y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) x = fma(x, y, 1e-9);
    long long t1 = clock64();
    for (int i = 0; i < 256; ++i) x = x + 1e-9;
    long long t2 = clock64();
    for (int i = 0; i < 64; ++i) x = rsqrt(x) + 1.0;
    long long t3 = clock64();
    for (int i = 0; i < 64; ++i) x = sqrt(x) + 1.0;
    long long t4 = clock64();
    for (int i = 0; i < 64; ++i) x = 3.0 / x + 1.0;
    long long t5 = clock64();
    for (int i = 0; i < 64; ++i) x = __drcp_rn(x) + 1.0;
    long long t6 = clock64();
    out[0] = x;
    cyc[0] = (t1 - t0) / 256;
    cyc[1] = (t2 - t1) / 256;
    cyc[2] = (t3 - t2) / 64;
    cyc[3] = (t4 - t3) / 64;
    cyc[4] = (t5 - t4) / 64;
    cyc[5] = (t6 - t5) / 64;
}
}  // namespace dh2
using namespace dh2;

template <int NB, int NC, int CT, int CH>
void run(const char* name, double2* scr, double2* in, int nsm, int k, int nch) {
    for (int per = 1; per <= CT; ++per) {
        int grid = nsm * per;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k_cq_bench<NB, NC, CT, CH><<<grid, 128 / NC>>>(scr, in, k, 2);
        cudaEventRecord(a);
        k_cq_bench<NB, NC, CT, CH><<<grid, 128 / NC>>>(scr, in, k, nch);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        int clk;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        double steps = (double)nch * k;
        double cyc = ms * 1e-3 * clk * 1e3 / steps;  // cycles per step per CTA
        // useful complex FMAs per step per CTA: 2 NB (dot + update) x active columns (avg k/2)
        double flops = (double)grid * nch * NB * (double)k * k * 8.0;  // 2 x NB x k^2/2 x 8
        printf("%-14s CH=%d NB=%2d NC=%d CTAs/SM=%d: %7.1f cycles/step/CTA, %6.1f per SM-step, %.2f TF/s (%s)\n", name, CH, NB, NC,
               per, cyc, cyc / per, flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int k = 125, nch = 64;
    double2 *scr, *in;
    cudaMalloc(&scr, (size_t)nsm * 8 * k * CQ_KP * sizeof(double2));
    std::vector<double2> h(8 * 32 * 128);
    unsigned s = 12345;
    for (auto& v : h) {
        s = s * 1664525u + 1013904223u;
        v.x = (s >> 8) / 16777216.0 - 0.5;
        s = s * 1664525u + 1013904223u;
        v.y = (s >> 8) / 16777216.0 - 0.5;
    }
    cudaMalloc(&in, h.size() * sizeof(double2));
    cudaMemcpy(in, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice);
    {
        double* o;
        long long* c;
        cudaMalloc(&o, 8);
        cudaMalloc(&c, 6 * 8);
        k_lat<<<1, 1>>>(o, 1.5, c);
        long long h[6];
        cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
        fflush(stdout); printf("latency (cycles): DFMA %lld, DADD %lld, rsqrt+add %lld, sqrt+add %lld, div+add %lld, drcp+add %lld\n", h[0], h[1],
               h[2], h[3], h[4], h[5]);
    }
    run<16, 1, 4, 2>("owner", scr, in, nsm, k, nch);
    run<24, 1, 3, 2>("owner", scr, in, nsm, k, nch);
    run<32, 1, 2, 2>("owner", scr, in, nsm, k, nch);
    run<8, 1, 4, 2>("owner", scr, in, nsm, k, nch);
    return 0;
}
