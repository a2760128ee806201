// Test-only harness: runs the device building blocks of dh2_device.cuh on batches of small
// matrices (one CTA per matrix) so tests can compare them with numpy.  Not part of libdh2.so.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../paper_1809_04384_b200/csrc/dh2_device.cuh"

using namespace dh2;

// op: 0 = cta_qr (R), 1 = cta_qrcp (R, piv), 2 = qrcp_auto (R, piv), 3 = cta_jacobi_rows on the
// rows of the input, 4 = jacobi_rows_auto on the rows of the input, 5/6 = 1/2 with the rank stop,
// 7/8 = qrcp_np_auto (no column exchanges) without / with the rank stop.
__global__ void k_devtest(int op, const double2* in, double2* out, int* iout, double* dout, int M, int N, int ld) {
    extern __shared__ double2 smem[];
    __shared__ double2 sh[4];
    __shared__ int s_piv, flag;
    double2* A = smem;
    double* nrm = reinterpret_cast<double*>(A + (size_t)ld * N);
    int* piv = reinterpret_cast<int*>(nrm + 2 * N + M);
    const double2* X = in + (size_t)blockIdx.x * M * N;
    for (int idx = threadIdx.x; idx < M * N; idx += blockDim.x) A[idx % M + (idx / M) * ld] = X[idx];
    __syncthreads();
    int res = 0;
    if (op == 0) cta_qr(A, ld, M, N, sh);
    if (op == 1) res = cta_qrcp(A, ld, M, N, piv, nrm, sh, &s_piv, 0.0);
    if (op == 2) res = qrcp_auto(A, ld, M, N, piv, nrm, sh, &s_piv, 0.0);
    if (op == 3) res = cta_jacobi_rows(A, ld, M, N, nrm, &flag);
    if (op == 4) res = jacobi_rows_auto(A, ld, M, N, nrm, &flag);
    if (op == 5) res = cta_qrcp(A, ld, M, N, piv, nrm, sh, &s_piv, 1e-26);
    if (op == 6) res = qrcp_auto(A, ld, M, N, piv, nrm, sh, &s_piv, 1e-26);
    if (op == 7) res = qrcp_np_auto(A, ld, M, N, piv, nrm, 0.0);
    if (op == 8) res = qrcp_np_auto(A, ld, M, N, piv, nrm, 1e-26);
    __syncthreads();
    double2* Y = out + (size_t)blockIdx.x * M * N;
    for (int idx = threadIdx.x; idx < M * N; idx += blockDim.x) Y[idx] = A[idx % M + (idx / M) * ld];
    if (threadIdx.x == 0) iout[(size_t)blockIdx.x * (N + 1)] = res;
    for (int c = threadIdx.x; c < N; c += blockDim.x) iout[(size_t)blockIdx.x * (N + 1) + 1 + c] = (op == 1 || op == 2 || op >= 5) ? piv[c] : 0;
    for (int c = threadIdx.x; c < M; c += blockDim.x) dout[(size_t)blockIdx.x * M + c] = (op == 3 || op == 4) ? nrm[c] : 0.0;
}

extern "C" int devtest_run(int op, const double* in, double* out, int* iout, double* dout, int batch, int M, int N,
                           int threads) {
    int ld = (M | 1);
    size_t sm = (size_t)ld * N * sizeof(double2) + (size_t)(2 * N + M) * sizeof(double) + (size_t)(N + M) * sizeof(int) + 64;
    double2 *din, *dout2;
    int* di;
    double* dd;
    size_t nb = (size_t)batch * M * N * sizeof(double2);
    if (cudaMalloc(&din, nb) || cudaMalloc(&dout2, nb) || cudaMalloc(&di, (size_t)batch * (N + 1) * sizeof(int)) ||
        cudaMalloc(&dd, (size_t)batch * M * sizeof(double)))
        return -1;
    cudaMemcpy(din, in, nb, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_devtest, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_devtest<<<batch, threads, sm>>>(op, din, dout2, di, dd, M, N, ld);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out, dout2, nb, cudaMemcpyDeviceToHost);
    cudaMemcpy(iout, di, (size_t)batch * (N + 1) * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(dout, dd, (size_t)batch * M * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(din);
    cudaFree(dout2);
    cudaFree(di);
    cudaFree(dd);
    return e == cudaSuccess ? 0 : -2;
}

// out (nb x k) = w * X (nb x k) * op(S): X and S column-major, conj_s/strided as in the library.
__global__ void k_devgemm(const double2* X, const double2* S, double2* out, int nb, int k, int conj_s, int strided) {
    chunk_gemm_S_dmma(X, nb, 0, nb, S, conj_s != 0, strided != 0, 0.5, k, out, nb);
}
extern "C" int devtest_gemm(const double* X, const double* S, double* out, int nb, int k, int conj_s, int strided) {
    double2 *dx, *ds, *dout;
    cudaMalloc(&dx, (size_t)nb * k * 16);
    cudaMalloc(&ds, (size_t)k * k * 16);
    cudaMalloc(&dout, (size_t)nb * k * 16);
    cudaMemcpy(dx, X, (size_t)nb * k * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, S, (size_t)k * k * 16, cudaMemcpyHostToDevice);
    k_devgemm<<<1, 256>>>(dx, ds, dout, nb, k, conj_s, strided);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out, dout, (size_t)nb * k * 16, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(ds);
    cudaFree(dout);
    return e == cudaSuccess ? 0 : -2;
}

// R factor of A (M x N, column-major) by 32-row chunks appended into an N x N triangle:
// mode 0 = cta_qr_append (dense R), 1 = cta_qr_append_wy (dense), 2 / 3 = the same on the packed R.
__global__ void k_devappend(int mode, const double2* A, double2* Rout, int M, int N) {
    extern __shared__ double2 smem[];
    __shared__ WyPanel wp;
    __shared__ double s_tau[128];
    __shared__ double2 s_u0[128];
    __shared__ int s_step;
    const bool pk = mode == 2 || mode == 3 || mode == 5;
    const int ldr = N | 1, ldb = 33;
    double2* R = smem;
    const size_t relems = pk ? (size_t)N * (N + 1) / 2 : (size_t)ldr * N;
    double2* B = R + relems;
    for (size_t i = threadIdx.x; i < relems; i += blockDim.x) R[i] = cmk(0.0, 0.0);
    for (int r0 = 0; r0 < M; r0 += 32) {
        const int nb = min(32, M - r0);
        __syncthreads();
        for (int idx = threadIdx.x; idx < nb * N; idx += blockDim.x) B[idx % nb + (idx / nb) * ldb] = A[r0 + idx % nb + (size_t)(idx / nb) * M];
        __syncthreads();
        if (mode == 0) cta_qr_append<false, 2>(R, ldr, B, ldb, nb, N);
        if (mode == 1) cta_qr_append_wy<false>(R, ldr, B, ldb, nb, N, &wp);
        if (mode == 2) cta_qr_append<true, 2>(R, ldr, B, ldb, nb, N);
        if (mode == 3) cta_qr_append_wy<true>(R, ldr, B, ldb, nb, N, &wp);
        if (mode == 4) cta_qr_append_flag<false, 4, 8>(R, ldr, B, ldb, nb, N, s_tau, s_u0, &s_step);
        if (mode == 5) cta_qr_append_flag<true, 4, 8>(R, ldr, B, ldb, nb, N, s_tau, s_u0, &s_step);
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < N * N; idx += blockDim.x) {
        const int i = idx % N, c = idx / N;
        Rout[idx] = i > c ? cmk(0.0, 0.0) : R[pk ? ridx<true>(i, c, ldr) : ridx<false>(i, c, ldr)];
    }
}
extern "C" int devtest_append(int mode, const double* A, double* R, int M, int N, int threads) {
    double2 *da, *dr;
    cudaMalloc(&da, (size_t)M * N * 16);
    cudaMalloc(&dr, (size_t)N * N * 16);
    cudaMemcpy(da, A, (size_t)M * N * 16, cudaMemcpyHostToDevice);
    const bool pk = mode == 2 || mode == 3 || mode == 5;
    const size_t relems = pk ? (size_t)N * (N + 1) / 2 : (size_t)(N | 1) * N;
    const size_t sm = (relems + (size_t)33 * N) * 16;
    cudaFuncSetAttribute(k_devappend, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    k_devappend<<<1, threads, sm>>>(mode, da, dr, M, N);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaMemcpy(R, dr, (size_t)N * N * 16, cudaMemcpyDeviceToHost);
    cudaFree(da);
    cudaFree(dr);
    return e == cudaSuccess ? 0 : -2;
}
