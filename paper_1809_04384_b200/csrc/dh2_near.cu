// Nearfield of the Galerkin matrix (NEXT-4; Section 5): the inadmissible
// leaves b = (t, s) in L- are stored densely,
//     g_ij = int_{tau_i} int_{tau_j} exp(i kappa |x-y|) / (4 pi |x-y|) dy dx,
// with piecewise-constant basis functions.  As in the paper: Sauter-Erichsen-Schwab quadrature of
// order n_q = 5 for triangles that are identical or share an edge or a vertex, and Gauss quadrature
// with Duffy transformation of order n_q = 3 otherwise.
//
// Reference triangle T = {0 <= u2 <= u1 <= 1}, chi(u) = P0 + u1 (P1 - P0) + u2 (P2 - P1), Jacobian
// 2|tau|.  Regular pairs: Duffy map (s, t) -> (s, s t) (Jacobian s), n_q^2 points per triangle,
// precomputed once per triangle (k_near_points) and combined n_q^2 x n_q^2 per entry
// (k_near_regular: one CTA per block, one thread per entry, touching entries skipped).  Touching
// pairs: the relative-coordinate transformations of T x T onto [0,1]^4 (identical 6 regions,
// common edge 5, common vertex 2), whose factor xi^3 cancels the singularity; the host lists these
// entries with the vertex orders that put the shared vertices first, and k_near_singular gives one
// warp to each (its lanes split the regions x n_q^4 points; warp-shuffle reduction).
//
// Bound: FP64 ALU (sqrt, sincos, division per kernel evaluation; nothing is read twice from HBM).
// The matvec (k_mv_near) reads every stored coefficient once: HBM bound, 16 B per coefficient.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "dh2_shard.h"

namespace dh2 {

namespace {

constexpr int NQ_MAX = 8;
__constant__ double c_gx[NQ_MAX], c_gw[NQ_MAX];  // Gauss-Legendre on [0,1] (singular order)
__constant__ double c_rx[NQ_MAX], c_rw[NQ_MAX];  // Gauss-Legendre on [0,1] (regular order)

// n-point Gauss-Legendre rule on [0,1]: Newton on P_n from the Chebyshev-like initial guesses.
void gauss01(int n, double* x, double* w) {
    for (int i = 0; i < n; ++i) {
        double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = 0.0;
            for (int j = 1; j <= n; ++j) {
                const double p2 = p1;
                p1 = p0;
                p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
            }
            dp = n * (z * p0 - p1) / (z * z - 1.0);
            const double dz = p0 / dp;
            z -= dz;
            if (std::fabs(dz) < 1e-16) break;
        }
        x[n - 1 - i] = 0.5 * (z + 1.0);  // ascending
        w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);  // (2/((1-z^2) P'^2)) / 2
    }
}

struct Tri {
    double3 p0, e1, e2;  // chi(u) = p0 + u1 e1 + u2 e2 (e1 = P1 - P0, e2 = P2 - P1)
};

__device__ __forceinline__ double3 ld3(const double* xyz, int64_t v) {
    return make_double3(xyz[3 * v], xyz[3 * v + 1], xyz[3 * v + 2]);
}
__device__ __forceinline__ double3 sub3(double3 a, double3 b) { return make_double3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ double area3(double3 a, double3 b) {  // |a x b| / 2
    const double cx = a.y * b.z - a.z * b.y, cy = a.z * b.x - a.x * b.z, cz = a.x * b.y - a.y * b.x;
    return 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
}

// Duffy-Gauss points of every triangle (cluster order): (x, y, z, w_p * 2|tau|).
__global__ void k_near_points(const double* __restrict__ xyz, const int64_t* __restrict__ tri,
                              const int64_t* __restrict__ perm, int n, int nq, double4* __restrict__ pts) {
    const int q2 = nq * nq;
    const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (id >= (int64_t)n * q2) return;
    const int pos = (int)(id / q2), q = (int)(id % q2), a = q / nq, b = q % nq;
    const int64_t i = perm[pos];
    const double3 P0 = ld3(xyz, tri[3 * i]), P1 = ld3(xyz, tri[3 * i + 1]), P2 = ld3(xyz, tri[3 * i + 2]);
    const double3 e1 = sub3(P1, P0), e2 = sub3(P2, P1);
    const double s = c_rx[a], t = c_rx[b];
    const double u1 = s, u2 = s * t;
    const double w = c_rw[a] * c_rw[b] * s * 2.0 * area3(sub3(P1, P0), sub3(P2, P0));
    pts[id] = make_double4(P0.x + u1 * e1.x + u2 * e2.x, P0.y + u1 * e1.y + u2 * e2.y, P0.z + u1 * e1.z + u2 * e2.z, w);
}

__device__ __forceinline__ void acc_g(double2& acc, double3 x, double3 y, double w, double kappa) {
    const double dx = x.x - y.x, dy = x.y - y.y, dz = x.z - y.z;
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    double sn, cs;
    sincos(kappa * r, &sn, &cs);
    const double f = w / r;
    acc.x += f * cs;
    acc.y += f * sn;
}

// Regular entries of the own blocks: one CTA per block, one thread per entry (column-major).
// Q2 = n_q^2 at compile time (9: the paper's order 3, loops unrolled), 0 = run-time q2.
template <int Q2>
__global__ void __launch_bounds__(256) k_near_regular(const double4* __restrict__ pts, const int64_t* __restrict__ tri,
                                                      const int64_t* __restrict__ perm, const int64_t* __restrict__ c_begin,
                                                      const int* __restrict__ c_size, const int* __restrict__ bt,
                                                      const int* __restrict__ bs, const int64_t* __restrict__ off, int q2_rt,
                                                      double kappa, double2* __restrict__ val) {
    const int q2 = Q2 ? Q2 : q2_rt;
    const int b = blockIdx.x, t = bt[b], s = bs[b];
    const int nt = c_size[t], ns = c_size[s];
    const int64_t bt0 = c_begin[t], bs0 = c_begin[s];
    double2* out = val + off[b];
    const double inv4pi = 0.25 / M_PI;
    for (int e = threadIdx.x; e < nt * ns; e += blockDim.x) {
        const int a = e % nt, c = e / nt;
        const int64_t pi = bt0 + a, pj = bs0 + c;
        const int64_t i = perm[pi], j = perm[pj];
        const int64_t i0 = tri[3 * i], i1 = tri[3 * i + 1], i2 = tri[3 * i + 2];
        const int64_t j0 = tri[3 * j], j1 = tri[3 * j + 1], j2 = tri[3 * j + 2];
        const bool touch = i0 == j0 || i0 == j1 || i0 == j2 || i1 == j0 || i1 == j1 || i1 == j2 || i2 == j0 ||
                           i2 == j1 || i2 == j2;
        if (touch) continue;  // (k_near_singular writes it)
        const double4* X = pts + pi * q2;
        const double4* Y = pts + pj * q2;
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int p = 0; p < q2; ++p) {
            const double4 xp = X[p];
            double2 row = make_double2(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < (Q2 ? Q2 : q2); ++q) {
                const double4 yq = Y[q];
                acc_g(row, make_double3(xp.x, xp.y, xp.z), make_double3(yq.x, yq.y, yq.z), yq.w, kappa);
            }
            acc.x += xp.w * row.x;
            acc.y += xp.w * row.y;
        }
        out[e] = make_double2(acc.x * inv4pi, acc.y * inv4pi);
    }
}

// One touching entry: value offset, triangles (original ids), case (0 identical, 1 edge, 2 vertex)
// and the vertex orders (2 bits per vertex, i then j).
struct SingItem {
    int64_t off;
    int i, j;
    int code;  // case | oi0<<2 | oi1<<4 | oi2<<6 | oj0<<8 | oj1<<10 | oj2<<12
};

__device__ __forceinline__ Tri make_tri(const double* xyz, const int64_t* tri, int i, int o0, int o1, int o2) {
    const double3 P0 = ld3(xyz, tri[3 * (int64_t)i + o0]), P1 = ld3(xyz, tri[3 * (int64_t)i + o1]),
                  P2 = ld3(xyz, tri[3 * (int64_t)i + o2]);
    Tri T;
    T.p0 = P0;
    T.e1 = sub3(P1, P0);
    T.e2 = sub3(P2, P1);
    return T;
}
__device__ __forceinline__ double3 chi(const Tri& T, double u1, double u2) {
    return make_double3(T.p0.x + u1 * T.e1.x + u2 * T.e2.x, T.p0.y + u1 * T.e1.y + u2 * T.e2.y,
                        T.p0.z + u1 * T.e1.z + u2 * T.e2.z);
}

// Sauter-Schwab sub-region r of `cas` at (xi, e1, e2, e3): (u1, u2), (v1, v2) and the weight.
__device__ __forceinline__ double ss_region(int cas, int r, double xi, double e1, double e2, double e3, double& u1,
                                            double& u2, double& v1, double& v2) {
    if (cas == 0) {  // identical, weight xi^3 e1^2 e2
        switch (r) {
            case 0: u1 = xi; u2 = xi * (1 - e1 + e1 * e2); v1 = xi * (1 - e1 * e2 * e3); v2 = xi * (1 - e1); break;
            case 1: u1 = xi * (1 - e1 * e2 * e3); u2 = xi * (1 - e1); v1 = xi; v2 = xi * (1 - e1 + e1 * e2); break;
            case 2: u1 = xi; u2 = xi * e1 * (1 - e2 + e2 * e3); v1 = xi * (1 - e1 * e2); v2 = xi * e1 * (1 - e2); break;
            case 3: u1 = xi * (1 - e1 * e2); u2 = xi * e1 * (1 - e2); v1 = xi; v2 = xi * e1 * (1 - e2 + e2 * e3); break;
            case 4: u1 = xi * (1 - e1 * e2 * e3); u2 = xi * e1 * (1 - e2 * e3); v1 = xi; v2 = xi * e1 * (1 - e2); break;
            default: u1 = xi; u2 = xi * e1 * (1 - e2); v1 = xi * (1 - e1 * e2 * e3); v2 = xi * e1 * (1 - e2 * e3); break;
        }
        return xi * xi * xi * e1 * e1 * e2;
    }
    if (cas == 1) {  // common edge (u2 = 0 in both), weights xi^3 e1^2 (r = 0), xi^3 e1^2 e2
        switch (r) {
            case 0: u1 = xi; u2 = xi * e1 * e3; v1 = xi * (1 - e1 * e2); v2 = xi * e1 * (1 - e2);
                return xi * xi * xi * e1 * e1;
            case 1: u1 = xi; u2 = xi * e1; v1 = xi * (1 - e1 * e2 * e3); v2 = xi * e1 * e2 * (1 - e3); break;
            case 2: u1 = xi * (1 - e1 * e2); u2 = xi * e1 * (1 - e2); v1 = xi; v2 = xi * e1 * e2 * e3; break;
            case 3: u1 = xi * (1 - e1 * e2 * e3); u2 = xi * e1 * e2 * (1 - e3); v1 = xi; v2 = xi * e1; break;
            default: u1 = xi * (1 - e1 * e2 * e3); u2 = xi * e1 * (1 - e2 * e3); v1 = xi; v2 = xi * e1 * e2; break;
        }
        return xi * xi * xi * e1 * e1 * e2;
    }
    // common vertex (u = 0 in both), weight xi^3 e2
    if (r == 0) {
        u1 = xi; u2 = xi * e1; v1 = xi * e2; v2 = xi * e2 * e3;
    } else {
        u1 = xi * e2; u2 = xi * e2 * e3; v1 = xi; v2 = xi * e1;
    }
    return xi * xi * xi * e2;
}

// NQ: the singular order as a compile-time constant (the point index decomposes by constant
// divisions); a generic-order instance (NQ = 0) serves the other orders.
template <int NQ>
__global__ void __launch_bounds__(256, 3) k_near_singular(const double* __restrict__ xyz, const int64_t* __restrict__ tri,
                                                          const SingItem* __restrict__ items, int64_t nitems, int nq_rt,
                                                          double kappa, double2* __restrict__ val) {
    const int nq = NQ ? NQ : nq_rt;
    // the rule in shared memory: lanes index it at different points (constant memory would
    // serialise the divergent addresses)
    __shared__ double sgx[NQ_MAX], sgw[NQ_MAX];
    if (threadIdx.x < NQ_MAX) {
        sgx[threadIdx.x] = c_gx[threadIdx.x];
        sgw[threadIdx.x] = c_gw[threadIdx.x];
    }
    __syncthreads();
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= nitems) return;
    const SingItem it = items[w];
    const int cas = it.code & 3;
    const Tri X = make_tri(xyz, tri, it.i, (it.code >> 2) & 3, (it.code >> 4) & 3, (it.code >> 6) & 3);
    const Tri Y = make_tri(xyz, tri, it.j, (it.code >> 8) & 3, (it.code >> 10) & 3, (it.code >> 12) & 3);
    const int nreg = cas == 0 ? 6 : cas == 1 ? 5 : 2;
    const int q3 = nq * nq * nq, q4 = q3 * nq;
    double2 acc = make_double2(0.0, 0.0);
    for (int r = 0; r < nreg; ++r)  // (region uniform across the warp)
        for (int q = lane; q < q4; q += 32) {
            const int a = q / q3, b = (q / (nq * nq)) % nq, c = (q / nq) % nq, d = q % nq;
            double u1, u2, v1, v2;
            const double wr = ss_region(cas, r, sgx[a], sgx[b], sgx[c], sgx[d], u1, u2, v1, v2);
            acc_g(acc, chi(X, u1, u2), chi(Y, v1, v2), wr * (sgw[a] * sgw[b]) * (sgw[c] * sgw[d]), kappa);
        }
    for (int o = 16; o; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) {
        const double jac = 4.0 * area3(X.e1, sub3(chi(X, 1.0, 1.0), X.p0)) * area3(Y.e1, sub3(chi(Y, 1.0, 1.0), Y.p0));
        const double f = jac * 0.25 / M_PI;
        val[it.off] = make_double2(acc.x * f, acc.y * f);
    }
}

// y_p[t] += sum over the row group's blocks N_b x_p[s] (cluster order); one CTA per row leaf,
// R rows x 256/R column slices per pass (R = 32 when every leaf has <= 32 triangles), reduction of
// the slices in shared memory.
template <int R>
__global__ void __launch_bounds__(256) k_mv_near(const int64_t* __restrict__ c_begin, const int* __restrict__ c_size,
                                                 const int* __restrict__ gord, const int* __restrict__ gptr, const int* __restrict__ bt,
                                                 const int* __restrict__ bs, const int64_t* __restrict__ off,
                                                 const double2* __restrict__ val, const double2* __restrict__ xp,
                                                 double2* __restrict__ yp) {
    constexpr int NS = 256 / R;
    __shared__ double2 red[NS][R];
    const int g0 = gptr[gord[blockIdx.x]], g1 = gptr[gord[blockIdx.x] + 1];
    const int t = bt[g0], nt = c_size[t];
    const int lr = threadIdx.x % R, sl = threadIdx.x / R;
    for (int a0 = 0; a0 < nt; a0 += R) {
        const int a = a0 + lr;
        double2 acc = make_double2(0.0, 0.0);
        if (a < nt)
            for (int b = g0; b < g1; ++b) {
                const int s = bs[b], ns = c_size[s];
                const double2* N = val + off[b];
                const double2* x = xp + c_begin[s];
                for (int c = sl; c < ns; c += NS) {
                    const double2 v = __ldg(N + (int64_t)c * nt + a), xv = __ldg(x + c);
                    acc.x += v.x * xv.x - v.y * xv.y;
                    acc.y += v.x * xv.y + v.y * xv.x;
                }
            }
        red[sl][lr] = acc;
        __syncthreads();
        if (sl == 0 && a < nt) {
            double2 y = yp[c_begin[t] + a];
            for (int k = 0; k < NS; ++k) {
                y.x += red[k][lr].x;
                y.y += red[k][lr].y;
            }
            yp[c_begin[t] + a] = y;
        }
        __syncthreads();
    }
}


// TMA form of the nearfield matvec: the row group's blocks N_b (contiguous, column-major, 16-byte
// aligned) are streamed through a ring of NEAR_ST shared-memory stages by 1-D bulk copies
// (cp.async.bulk, completion on an mbarrier per stage), NEAR_CE coefficients (16 KB) per stage, issued
// NEAR_ST - 1 chunks ahead by thread 0; the 256 threads multiply from shared memory (R rows x 256/R
// column slices).  One __syncthreads per chunk hands the consumed stage back to the producer.
constexpr int NEAR_ST = 4, NEAR_CE = 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@p bra D;\nbra W;\nD:\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}

struct NearCursor {  // walks the chunks (block b, first column c0) of a row group in order
    int b, c0;
    __device__ __forceinline__ void next(int cw, int ns) {
        c0 += cw;
        if (c0 >= ns) {
            c0 = 0;
            ++b;
        }
    }
};

template <int R>
__global__ void __launch_bounds__(256) k_mv_near_tma(const int64_t* __restrict__ c_begin, const int* __restrict__ c_size,
                                                     const int* __restrict__ gord, const int* __restrict__ gptr, const int* __restrict__ bt,
                                                     const int* __restrict__ bs, const int64_t* __restrict__ off,
                                                     const double2* __restrict__ val, const double2* __restrict__ xp,
                                                     double2* __restrict__ yp) {
    constexpr int NS = 256 / R;
    extern __shared__ __align__(128) unsigned char near_smem[];
    double2* ring = reinterpret_cast<double2*>(near_smem);                          // NEAR_ST x NEAR_CE
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)NEAR_ST * NEAR_CE);  // NEAR_ST barriers
    __shared__ double2 red[NS][R];
    const int g0 = gptr[gord[blockIdx.x]], g1 = gptr[gord[blockIdx.x] + 1];
    const int t = bt[g0], nt = c_size[t];  // nt <= R (checked by the host)
    const int cwmax = NEAR_CE / nt;        // columns per chunk
    const int lr = threadIdx.x % R, sl = threadIdx.x / R;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NEAR_ST; ++i) mbar_init(full + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    NearCursor pc{g0, 0};  // producer (thread 0 only)
    int issued = 0;
    auto issue = [&]() {
        if (pc.b >= g1) return;
        const int ns = c_size[bs[pc.b]];
        const int cw = min(cwmax, ns - pc.c0);
        const int st = issued % NEAR_ST;
        bulk_g2s(ring + (size_t)st * NEAR_CE, val + off[pc.b] + (int64_t)pc.c0 * nt, (uint32_t)(cw * nt) * 16u, full + st);
        ++issued;
        pc.next(cw, ns);
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < NEAR_ST - 1; ++i) issue();
    double2 acc = make_double2(0.0, 0.0);
    NearCursor cc{g0, 0};
    for (int i = 0; cc.b < g1; ++i) {
        if (threadIdx.x == 0) issue();  // into the stage consumed in iteration i - 1
        const int s = bs[cc.b], ns = c_size[s];
        const int cw = min(cwmax, ns - cc.c0);
        const int st = i % NEAR_ST;
        mbar_wait(full + st, (uint32_t)(i / NEAR_ST) & 1u);
        if (lr < nt) {
            const double2* N = ring + (size_t)st * NEAR_CE;
            const double2* x = xp + c_begin[s] + cc.c0;
#pragma unroll 4
            for (int c = sl; c < cw; c += NS) {
                const double2 v = N[c * nt + lr], xv = __ldg(x + c);
                acc.x += v.x * xv.x - v.y * xv.y;
                acc.y += v.x * xv.y + v.y * xv.x;
            }
        }
        cc.next(cw, ns);
        __syncthreads();
    }
    red[sl][lr] = acc;
    __syncthreads();
    if (sl == 0 && lr < nt) {
        double2 y = yp[c_begin[t] + lr];
        for (int k = 0; k < NS; ++k) {
            y.x += red[k][lr].x;
            y.y += red[k][lr].y;
        }
        yp[c_begin[t] + lr] = y;
    }
}

}  // namespace

void near_assemble(Shard* C, int nq_sing, int nq_reg) {
    if (nq_sing < 1 || nq_sing > NQ_MAX || nq_reg < 1 || nq_reg > NQ_MAX)
        throw std::invalid_argument("nearfield quadrature orders must be in 1.." + std::to_string(NQ_MAX));
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    const int64_t n = C->n;
    auto& N = C->near;
    N.on = false;
    N.nq_sing = nq_sing;
    N.nq_reg = nq_reg;
    // own blocks (row leaf t owned by this shard), in the structure's (t, s) order
    N.t.clear();
    N.s.clear();
    N.max_rows = 0;
    N.off.clear();
    std::vector<int> gptr;
    int64_t acc = 0;
    for (auto& ts : C->st.near) {
        const int t = (int)ts.first, sc = (int)ts.second;
        if (C->world > 1 && C->owner[t] != C->rank) continue;
        if (N.t.empty() || N.t.back() != t) gptr.push_back((int)N.t.size());
        N.t.push_back(t);
        N.s.push_back(sc);
        N.max_rows = std::max(N.max_rows, (int)T.size(t));
        N.off.push_back(acc);
        acc += T.size(t) * T.size(sc);
    }
    gptr.push_back((int)N.t.size());
    N.nblk = (int)N.t.size();
    N.ngroups = (int)gptr.size() - 1;
    N.values = acc;
    // touching entries: vertex -> triangles adjacency of the (replicated) mesh
    std::vector<int64_t> tri(3 * n);
    CK(cudaMemcpyAsync(tri.data(), C->d_tri.p, tri.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int64_t nv = 0;
    for (int64_t v : tri) nv = std::max(nv, v + 1);
    std::vector<int64_t> vptr(nv + 1, 0), vtri(3 * n);
    for (int64_t v : tri) ++vptr[v + 1];
    for (int64_t v = 0; v < nv; ++v) vptr[v + 1] += vptr[v];
    {
        std::vector<int64_t> fill(vptr.begin(), vptr.end() - 1);
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k) vtri[fill[tri[3 * i + k]]++] = i;
    }
    std::vector<int64_t> ipos(n);
    for (int64_t p = 0; p < n; ++p) ipos[T.perm[p]] = p;
    std::vector<SingItem> items;
    std::vector<int64_t> nb;
    int64_t expected = 0;
    std::vector<char> seen(n, 0);
    for (int b = 0; b < N.nblk; ++b) {
        const int t = N.t[b], sc = N.s[b];
        const int64_t t0 = T.begin[t], nt = T.size(t), s0 = T.begin[sc], ns = T.size(sc);
        for (int64_t a = 0; a < nt; ++a) {
            const int64_t i = T.perm[t0 + a];
            nb.clear();
            for (int k = 0; k < 3; ++k)
                for (int64_t q = vptr[tri[3 * i + k]]; q < vptr[tri[3 * i + k] + 1]; ++q) nb.push_back(vtri[q]);
            std::sort(nb.begin(), nb.end());
            nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
            if (!seen[i]) {  // once per row triangle: with mixed levels a row lies in several row clusters
                seen[i] = 1;
                expected += (int64_t)nb.size();
            }
            for (int64_t j : nb) {
                const int64_t pj = ipos[j];
                if (pj < s0 || pj >= s0 + ns) continue;
                // case and vertex orders: the shared vertices first, in the order of i (as the oracle)
                const int64_t* ti = &tri[3 * i];
                const int64_t* tj = &tri[3 * j];
                int pos_j[3], ncom = 0, ci[3], cj[3];
                for (int u = 0; u < 3; ++u) {
                    pos_j[u] = -1;
                    for (int v = 0; v < 3; ++v)
                        if (ti[u] == tj[v]) pos_j[u] = v;
                    if (pos_j[u] >= 0) {
                        ci[ncom] = u;
                        cj[ncom] = pos_j[u];
                        ++ncom;
                    }
                }
                int cas, oi[3], oj[3];
                if (ncom == 3) {
                    cas = 0;
                    for (int u = 0; u < 3; ++u) oi[u] = u, oj[u] = pos_j[u];
                } else if (ncom == 2) {
                    cas = 1;
                    oi[0] = ci[0], oi[1] = ci[1], oi[2] = 3 - ci[0] - ci[1];
                    oj[0] = cj[0], oj[1] = cj[1], oj[2] = 3 - cj[0] - cj[1];
                } else {
                    cas = 2;
                    for (int u = 0; u < 3; ++u) oi[u] = (ci[0] + u) % 3, oj[u] = (cj[0] + u) % 3;
                }
                SingItem it;
                it.off = N.off[b] + a + (pj - s0) * nt;
                it.i = (int)i;
                it.j = (int)j;
                it.code = cas | oi[0] << 2 | oi[1] << 4 | oi[2] << 6 | oj[0] << 8 | oj[1] << 10 | oj[2] << 12;
                items.push_back(it);
            }
        }
    }
    if ((int64_t)items.size() != expected)
        throw std::runtime_error("nearfield: " + std::to_string(items.size()) + " touching entries in the inadmissible leaves, " +
                                 std::to_string(expected) + " touching pairs in the mesh");
    N.nsing = (int64_t)items.size();
    N.evals = (double)(N.values - N.nsing) * nq_reg * nq_reg * nq_reg * nq_reg;
    for (const SingItem& it : items) {
        const int cas = it.code & 3;
        N.evals += (cas == 0 ? 6.0 : cas == 1 ? 5.0 : 2.0) * nq_sing * nq_sing * nq_sing * nq_sing;
    }
    // quadrature rules
    double gx[NQ_MAX], gw[NQ_MAX], rx[NQ_MAX], rw[NQ_MAX];
    gauss01(nq_sing, gx, gw);
    gauss01(nq_reg, rx, rw);
    CK(cudaMemcpyToSymbolAsync(c_gx, gx, sizeof(double) * nq_sing, 0, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyToSymbolAsync(c_gw, gw, sizeof(double) * nq_sing, 0, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyToSymbolAsync(c_rx, rx, sizeof(double) * nq_reg, 0, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyToSymbolAsync(c_rw, rw, sizeof(double) * nq_reg, 0, cudaMemcpyHostToDevice, s));
    N.d_t.upload(N.t, s);
    N.d_s.upload(N.s, s);
    N.d_off.upload(N.off, s);
    N.d_gptr.upload(gptr, s);
    {   // with mixed levels a row triangle lies in row clusters of several levels (a cluster and a descendant
        // leaf): the matvec adds one level per launch, in level order, so that no two CTAs update the same rows
        std::vector<int> gord(N.ngroups);
        for (int g = 0; g < N.ngroups; ++g) gord[g] = g;
        std::stable_sort(gord.begin(), gord.end(),
                         [&](int a, int b) { return T.level[N.t[gptr[a]]] < T.level[N.t[gptr[b]]]; });
        N.glev_ptr.assign(1, 0);
        for (int i = 1; i <= N.ngroups; ++i)
            if (i == N.ngroups || T.level[N.t[gptr[gord[i]]]] != T.level[N.t[gptr[gord[i - 1]]]]) N.glev_ptr.push_back(i);
        N.d_gord.upload(gord, s);
    }
    N.d_val.alloc((size_t)std::max<int64_t>(N.values, 1));
    const int q2 = nq_reg * nq_reg;
    N.d_pts.alloc((size_t)n * q2);
    DevBuf<SingItem> d_items;
    d_items.upload(items, s);
    const PlanD& P = C->P;
    C->timed("nearfield", 1, [&] {
        const int64_t tot = n * q2;
        k_near_points<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(P.xyz, P.tri, P.perm, (int)n, nq_reg, N.d_pts.p);
    });
    if (N.nblk)
        C->timed("nearfield", 1, [&] {
            if (q2 == 9)
                k_near_regular<9><<<N.nblk, 256, 0, s>>>(N.d_pts.p, P.tri, P.perm, C->d_c_begin.p, C->d_c_size.p, N.d_t.p,
                                                         N.d_s.p, N.d_off.p, q2, P.kappa, N.d_val.p);
            else
                k_near_regular<0><<<N.nblk, 256, 0, s>>>(N.d_pts.p, P.tri, P.perm, C->d_c_begin.p, C->d_c_size.p, N.d_t.p,
                                                         N.d_s.p, N.d_off.p, q2, P.kappa, N.d_val.p);
        });
    if (N.nsing)
        C->timed("nearfield", 1, [&] {
            const unsigned grid = (unsigned)((N.nsing * 32 + 255) / 256);
            if (nq_sing == 5)
                k_near_singular<5><<<grid, 256, 0, s>>>(P.xyz, P.tri, d_items.p, N.nsing, nq_sing, P.kappa, N.d_val.p);
            else
                k_near_singular<0><<<grid, 256, 0, s>>>(P.xyz, P.tri, d_items.p, N.nsing, nq_sing, P.kappa, N.d_val.p);
        });
    CK(cudaStreamSynchronize(s));
    N.d_pts.free();
    N.on = true;
}

void near_matvec(Shard* C) {
    auto& N = C->near;
    if (!N.on || !N.ngroups) return;
    C->kstat["matvec_near"].bytes += 16.0 * (double)N.values;  // every coefficient read once
    constexpr size_t smem = (size_t)NEAR_ST * NEAR_CE * sizeof(double2) + NEAR_ST * sizeof(uint64_t);
    const bool tma = C->near_tma && N.max_rows <= 64;
    if (tma) {
        CK(cudaFuncSetAttribute(k_mv_near_tma<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaFuncSetAttribute(k_mv_near_tma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    const int nlev = (int)N.glev_ptr.size() - 1;
    C->timed("matvec_near", nlev, [&] {
        for (int i = 0; i < nlev; ++i) {  // one launch per tree level of the row clusters (one, unless levels are mixed)
            const int* gord = N.d_gord.p + N.glev_ptr[i];
            const int ng = N.glev_ptr[i + 1] - N.glev_ptr[i];
            if (tma && N.max_rows <= 32)
                k_mv_near_tma<32><<<ng, 256, smem, C->stream>>>(C->d_c_begin.p, C->d_c_size.p, gord, N.d_gptr.p, N.d_t.p, N.d_s.p,
                                                                N.d_off.p, N.d_val.p, C->d_xp.p, C->d_yp.p);
            else if (tma)
                k_mv_near_tma<64><<<ng, 256, smem, C->stream>>>(C->d_c_begin.p, C->d_c_size.p, gord, N.d_gptr.p, N.d_t.p, N.d_s.p,
                                                                N.d_off.p, N.d_val.p, C->d_xp.p, C->d_yp.p);
            else if (N.max_rows <= 32)
                k_mv_near<32><<<ng, 256, 0, C->stream>>>(C->d_c_begin.p, C->d_c_size.p, gord, N.d_gptr.p, N.d_t.p, N.d_s.p,
                                                         N.d_off.p, N.d_val.p, C->d_xp.p, C->d_yp.p);
            else
                k_mv_near<64><<<ng, 256, 0, C->stream>>>(C->d_c_begin.p, C->d_c_size.p, gord, N.d_gptr.p, N.d_t.p, N.d_s.p,
                                                         N.d_off.p, N.d_val.p, C->d_xp.p, C->d_yp.p);
        }
    });
}

}  // namespace dh2
