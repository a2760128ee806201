// Device-side building blocks for the DH^2 recompression kernels (sm_100a).
// Complex float64 is double2 (re, im); all matrices are column-major.
#pragma once
#include <cuda_runtime.h>
#include <cuda/atomic>
#include <stdint.h>

namespace dh2 {

constexpr int MMAX = 5;  // maximal Chebyshev order per axis supported by the grid tables
// Householder reflectors are formed only for columns with sum of squares above HH_TINY: below it
// tau = 1/(xn (xn + |alpha|)) can overflow (xn < 1e-154), and the column (norm < 1e-150) is
// numerically zero at every scale of this problem; it is left in place (beta = alpha).
constexpr double HH_TINY = 1e-300;

struct GridD {
    double mid[3];
    double half[3];
    double nodes[3][MMAX];
    int flat[3];
};

// ------------------------------------------------------------------ complex helpers
__device__ __forceinline__ double2 cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) { return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cconj(double2 a) { return cmk(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return cmk(a.x * s, a.y * s); }
__device__ __forceinline__ double cabs2(double2 a) { return a.x * a.x + a.y * a.y; }
// acc += a * b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_cj(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(-a.y, b.x, acc.y);
}
// acc += a * conj(b)
__device__ __forceinline__ void cfma_bj(double2& acc, double2 a, double2 b) {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(a.y, b.y, acc.x);
    acc.y = fma(a.y, b.x, acc.y);
    acc.y = fma(-a.x, b.y, acc.y);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
    v.x = warp_sum(v.x);
    v.y = warp_sum(v.y);
    return v;
}

// Lane groups: G consecutive lanes (G a power of two, 2..32) cooperate on one vector so a
// warp works on 32/G independent vectors at once; shuffles use the group's own mask.
struct LaneGroup {
    int G, gl, gid, ng;
    unsigned mask;
};
__device__ __forceinline__ LaneGroup lane_group(int G) {
    LaneGroup g;
    g.G = G;
    g.gl = threadIdx.x & (G - 1);
    g.gid = threadIdx.x / G;
    g.ng = blockDim.x / G;
    const int lane = threadIdx.x & 31;
    g.mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    return g;
}
// smallest power of two >= ceil(len / per_lane), clamped to [lo, 32]
__device__ __forceinline__ int group_size_for(int len, int per_lane, int lo) {
    int need = (len + per_lane - 1) / per_lane;
    int G = lo;
    while (G < need && G < 32) G <<= 1;
    return G;
}
__device__ __forceinline__ double group_sum(double v, const LaneGroup& g) {
    for (int o = g.G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(g.mask, v, o);
    return v;
}
__device__ __forceinline__ double2 group_sum2(double2 v, const LaneGroup& g) {
    for (int o = g.G >> 1; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(g.mask, v.x, o);
        v.y += __shfl_xor_sync(g.mask, v.y, o);
    }
    return v;
}

// Lagrange basis of the Chebyshev points of the first kind on one axis, evaluated at x
// (P:245-248): L_j(xhat) = prod_{i != j} (xhat - z_i)/(z_j - z_i), xhat = (x - mid)/half.
// A collapsed (flat) axis has L_j = delta_{j0} (DESIGN reading Q7).
__device__ __forceinline__ void lagrange_axis(const GridD& g, int a, int m, const double* z, const double* inv_den,
                                              double x, double* L) {
    if (g.flat[a]) {
        for (int j = 0; j < m; ++j) L[j] = (j == 0) ? 1.0 : 0.0;
        return;
    }
    double xh = (x - g.mid[a]) / g.half[a];
    for (int j = 0; j < m; ++j) {
        double v = inv_den[j];
        for (int i = 0; i < m; ++i)
            if (i != j) v *= (xh - z[i]);
        L[j] = v;
    }
}

// ------------------------------------------------------------------ asynchronous staging
// dst (nb x k, ld ldd, shared) <- src rows [i0, i0 + nb) of a column-major global matrix (ld lds)
// with 16-byte cp.async copies (many loads in flight per thread); the caller waits with
// cp_async_wait_all() and a barrier.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ inline void stage_rows(double2* dst, int ldd, const double2* src, int lds, int i0, int nb, int k) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int nu = warp; nu < k; nu += nw)
        for (int i = lane; i < nb; i += 32) cp_async16(dst + i + (size_t)nu * ldd, src + i0 + i + (size_t)nu * lds);
}

// ------------------------------------------------------------------ CTA-cooperative kernels

// In-place X <- X * E or X <- X * E^* for the Kronecker-structured transfer matrix
// E = Ez (x) Ey (x) Ex, nu = jx + m jy + m^2 jz (Eq. 10 with separable phase); X occupies
// rows [0, rows) of the column-major smem matrix X (leading dimension ld).  Ef holds the
// three m x m factors, Ef[a*m*m + jp*m + j] = E_a[j', j].  Each thread owns whole fibres.
template <int MM>
__device__ inline void kron_apply_t(double2* X, int ld, int rows, const double2* Ef, bool adjoint) {
    constexpr int m2 = MM * MM;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int stride = a == 0 ? 1 : (a == 1 ? MM : m2);
        const double2* F = Ef + a * m2;  // factor stays in shared memory (register budget)
        const int nfib = rows * m2;
        for (int fb = threadIdx.x; fb < nfib; fb += blockDim.x) {
            const int i = fb % rows;
            const int r = fb / rows;
            const int lo = r % stride, hi = r / stride;
            double2* xp = X + i + (lo + hi * stride * MM) * ld;
            double2 in[MM];
#pragma unroll
            for (int j = 0; j < MM; ++j) in[j] = xp[j * stride * ld];
#pragma unroll
            for (int j = 0; j < MM; ++j) {
                double2 acc = cmk(0.0, 0.0);
                if (!adjoint) {
#pragma unroll
                    for (int jp = 0; jp < MM; ++jp) cfma(acc, in[jp], F[jp * MM + j]);
                } else {
#pragma unroll
                    for (int jp = 0; jp < MM; ++jp) cfma_bj(acc, in[jp], F[j * MM + jp]);
                }
                xp[j * stride * ld] = acc;
            }
        }
        __syncthreads();
    }
}

__device__ inline void kron_apply_generic(double2* X, int ld, int rows, int m, const double2* Ef, bool adjoint);

__device__ inline void kron_apply(double2* X, int ld, int rows, int m, const double2* Ef, bool adjoint) {
    switch (m) {
        case 2: kron_apply_t<2>(X, ld, rows, Ef, adjoint); return;
        case 3: kron_apply_t<3>(X, ld, rows, Ef, adjoint); return;
        case 4: kron_apply_t<4>(X, ld, rows, Ef, adjoint); return;
        case 5: kron_apply_t<5>(X, ld, rows, Ef, adjoint); return;
        default: kron_apply_generic(X, ld, rows, m, Ef, adjoint); return;
    }
}

__device__ inline void kron_apply_generic(double2* X, int ld, int rows, int m, const double2* Ef, bool adjoint) {
    const int k = m * m * m;
    const int m2 = m * m;
    for (int a = 0; a < 3; ++a) {
        const int stride = a == 0 ? 1 : (a == 1 ? m : m2);
        const double2* F = Ef + a * m2;
        const int nfib = rows * m2;
        for (int f = threadIdx.x; f < nfib; f += blockDim.x) {
            int i = f % rows;
            int r = f / rows;  // index among the m^2 fibres of a row
            // base nu with the a-th digit zero
            int lowmask = stride;  // digits below a
            int lo = r % lowmask;
            int hi = r / lowmask;
            int base = lo + hi * stride * m;
            double2 in[MMAX], out[MMAX];
            for (int j = 0; j < m; ++j) in[j] = X[i + (size_t)(base + j * stride) * ld];
            for (int j = 0; j < m; ++j) {
                double2 acc = cmk(0.0, 0.0);
                if (!adjoint) {
                    for (int jp = 0; jp < m; ++jp) cfma(acc, in[jp], F[jp * m + j]);  // sum_j' X[j'] E[j', j]
                } else {
                    for (int jp = 0; jp < m; ++jp) cfma_bj(acc, in[jp], F[j * m + jp]);  // sum_j' X[j'] conj(E[j, j'])
                }
                out[j] = acc;
            }
            for (int j = 0; j < m; ++j) X[i + (size_t)(base + j * stride) * ld] = out[j];
        }
        (void)k;
        __syncthreads();
    }
}

// Householder QR (R factor only) of the M x N column-major smem matrix A in place
// ("skinny QR factorization").  On return the upper trapezoid of
// A[0:min(M,N), :] is R; entries below the diagonal hold Householder vectors and must be
// read as zero.  H_j = I - tau u u^*, u = x - beta e1, beta = -e^{i arg x0} |x|.
__device__ inline void cta_qr(double2* A, int lda, int M, int N, double2* sh /* >= 2 */) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int K = min(M, N);
    __syncthreads();
    for (int j = 0; j < K; ++j) {
        double2* colj = A + (size_t)j * lda;
        if (warp == 0) {
            double s = 0.0;
            for (int i = j + 1 + lane; i < M; i += 32) s += cabs2(colj[i]);
            s = warp_sum(s);
            if (lane == 0) {
                double2 alpha = colj[j];
                double tau = 0.0;
                double2 beta = alpha;
                if (s > HH_TINY) {  // tiny columns are left as they are (1/(xn (xn + aa)) would overflow)
                    double aa = sqrt(cabs2(alpha));
                    double xn = sqrt(s + aa * aa);
                    double2 ph = aa > 0.0 ? cscale(alpha, 1.0 / aa) : cmk(1.0, 0.0);
                    beta = cscale(ph, -xn);
                    colj[j] = cscale(ph, aa + xn);  // u0 = alpha - beta
                    tau = 1.0 / (xn * (xn + aa));   // 2 / (u^* u)
                }
                sh[0] = beta;
                sh[1] = cmk(tau, 0.0);
            }
        }
        __syncthreads();
        const double tau = sh[1].x;
        if (tau != 0.0) {
            const LaneGroup g = lane_group(group_size_for(M - j, 4, 4));
            for (int c = j + 1 + g.gid; c < N; c += g.ng) {
                double2* colc = A + (size_t)c * lda;
                double2 w = cmk(0.0, 0.0);
                for (int i = j + g.gl; i < M; i += g.G) cfma_cj(w, colj[i], colc[i]);
                w = group_sum2(w, g);
                w = cscale(w, tau);
                for (int i = j + g.gl; i < M; i += g.G) {
                    double2 u = colj[i];
                    colc[i] = csub(colc[i], cmul(u, w));
                }
            }
        }
        __syncthreads();
        if (tid == 0) colj[j] = sh[0];
        __syncthreads();
    }
}

// One-sided (Hestenes) Jacobi on the columns of the m x n smem matrix W (column-major,
// leading dimension ld): on return the columns are mutually orthogonal, W = U diag(s) J^*
// with J unitary, so the non-zero columns normalised are left singular vectors.
// Round-robin (circle) ordering, one warp per column pair.  Returns the number of sweeps.
__device__ inline int cta_jacobi(double2* W, int ld, int m, int n, int* flag) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    if (n <= 1) return 0;
    const int np = n + (n & 1);
    const double tol = fmax((double)m, 1.0) * 2.220446049250313e-16;
    int sweep = 0;
    for (; sweep < 60; ++sweep) {
        __syncthreads();
        if (tid == 0) *flag = 0;
        __syncthreads();
        for (int r = 0; r < np - 1; ++r) {
            for (int pi = warp; pi < np / 2; pi += nw) {
                int i0 = pi, i1 = np - 1 - pi;
                int p = i0 == 0 ? 0 : 1 + (i0 - 1 + r) % (np - 1);
                int q = i1 == 0 ? 0 : 1 + (i1 - 1 + r) % (np - 1);
                if (p >= n || q >= n) continue;
                double2* cp = W + (size_t)p * ld;
                double2* cq = W + (size_t)q * ld;
                double al = 0.0, be = 0.0;
                double2 ga = cmk(0.0, 0.0);
                for (int i = lane; i < m; i += 32) {
                    double2 a = cp[i], b = cq[i];
                    al += cabs2(a);
                    be += cabs2(b);
                    cfma_cj(ga, a, b);
                }
                al = warp_sum(al);
                be = warp_sum(be);
                ga = warp_sum2(ga);
                double g = sqrt(cabs2(ga));
                if (g > tol * sqrt(al * be) && al > 0.0 && be > 0.0) {
                    double zeta = (be - al) / (2.0 * g);
                    double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                    double c = 1.0 / sqrt(1.0 + t * t);
                    double s = c * t;
                    double2 e = cmk(ga.x / g, -ga.y / g);  // e^{-i phi}, gamma = g e^{i phi}
                    for (int i = lane; i < m; i += 32) {
                        double2 a = cp[i];
                        double2 b = cmul(e, cq[i]);
                        cp[i] = csub(cscale(a, c), cscale(b, s));
                        cq[i] = cadd(cscale(a, s), cscale(b, c));
                    }
                    if (lane == 0) *flag = 1;
                }
            }
            __syncthreads();
        }
        if (*flag == 0) break;
    }
    __syncthreads();
    return sweep;
}

// Householder QR with column pivoting (R factor + pivot order) of the M x N column-major
// smem matrix B, in place.  Pivot = remaining column of largest norm (first on ties); norms
// are recomputed exactly after every step (no downdating).  On return piv[j] = original
// column placed at position j, R = upper trapezoid of B[0:min(M,N), :] in pivoted order.
// If rank_rel2 > 0 the factorisation stops at the first step j whose trailing block has
// ||B[j:, j:]||_F^2 <= rank_rel2 * (largest column norm of B)^2 <= rank_rel2 * sigma_1(B)^2
// (numerical rank); returns the steps done.
__device__ inline int cta_qrcp(double2* B, int ldb, int M, int N, int* piv, double* nrm, double2* sh, int* s_piv,
                               double rank_rel2) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int K = min(M, N);
    for (int c = tid; c < N; c += blockDim.x) piv[c] = c;
    __syncthreads();
    for (int c = warp; c < N; c += nw) {
        double s = 0.0;
        for (int i = lane; i < M; i += 32) s += cabs2(B[i + (size_t)c * ldb]);
        s = warp_sum(s);
        if (lane == 0) nrm[c] = s;
    }
    __syncthreads();
    __shared__ double s_total;
    int j = 0;
    for (; j < K; ++j) {
        if (warp == 0) {
            double best = -1.0, rem = 0.0;
            int bi = j;
            for (int c = j + lane; c < N; c += 32) {
                double v = nrm[c];
                rem += v;
                if (v > best) { best = v; bi = c; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                double ob = __shfl_xor_sync(0xffffffffu, best, o);
                int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                rem += __shfl_xor_sync(0xffffffffu, rem, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            if (lane == 0) {
                if (j == 0) s_total = best;
                *s_piv = (rank_rel2 > 0.0 && j > 0 && rem <= rank_rel2 * s_total) ? -1 : bi;
            }
        }
        __syncthreads();
        const int pc = *s_piv;
        if (pc < 0) break;  // numerical rank reached (uniform across the CTA)
        if (pc != j) {
            for (int i = tid; i < M; i += blockDim.x) {
                double2 a = B[i + (size_t)j * ldb];
                B[i + (size_t)j * ldb] = B[i + (size_t)pc * ldb];
                B[i + (size_t)pc * ldb] = a;
            }
            if (tid == 0) {
                int t = piv[j]; piv[j] = piv[pc]; piv[pc] = t;
                double v = nrm[j]; nrm[j] = nrm[pc]; nrm[pc] = v;
            }
        }
        __syncthreads();
        double2* colj = B + (size_t)j * ldb;
        if (warp == 0) {
            double s = 0.0;
            for (int i = j + 1 + lane; i < M; i += 32) s += cabs2(colj[i]);
            s = warp_sum(s);
            if (lane == 0) {
                double2 alpha = colj[j];
                double tau = 0.0;
                double2 beta = alpha;
                if (s > HH_TINY) {  // tiny columns are left as they are (1/(xn (xn + aa)) would overflow)
                    double aa = sqrt(cabs2(alpha));
                    double xn = sqrt(s + aa * aa);
                    double2 ph = aa > 0.0 ? cscale(alpha, 1.0 / aa) : cmk(1.0, 0.0);
                    beta = cscale(ph, -xn);
                    colj[j] = cscale(ph, aa + xn);
                    tau = 1.0 / (xn * (xn + aa));
                }
                sh[0] = beta;
                sh[1] = cmk(tau, 0.0);
            }
        }
        __syncthreads();
        const double tau = sh[1].x;
        const LaneGroup g = lane_group(group_size_for(M - j, 4, 4));
        for (int c = j + 1 + g.gid; c < N; c += g.ng) {
            double2* colc = B + (size_t)c * ldb;
            if (tau != 0.0) {
                double2 w = cmk(0.0, 0.0);
                for (int i = j + g.gl; i < M; i += g.G) cfma_cj(w, colj[i], colc[i]);
                w = cscale(group_sum2(w, g), tau);
                for (int i = j + g.gl; i < M; i += g.G) colc[i] = csub(colc[i], cmul(colj[i], w));
            }
            double s = 0.0;
            for (int i = j + 1 + g.gl; i < M; i += g.G) s += cabs2(colc[i]);
            s = group_sum(s, g);
            if (g.gl == 0) nrm[c] = s;
        }
        __syncthreads();
        if (tid == 0) colj[j] = sh[0];
    }
    __syncthreads();
    return j;
}

// One-sided Jacobi on the vectors x_p = conj(R[p, 0:len]) (rows of the smem matrix R,
// column-major, leading dimension ldr), p < nv: on return the x_p are mutually orthogonal,
// i.e. the columns of R^* are U diag(s).  Round-robin ordering, one warp per pair, squared
// norms carried in nrm[] and updated by the exact rotation identities
// a' = a - t|g|, b' = b + t|g| (recomputed at every sweep).  Returns the sweeps done.
__device__ inline int cta_jacobi_rows(double2* R, int ldr, int nv, int len, double* nrm, int* flag) {
    const int tid = threadIdx.x;
    const LaneGroup g = lane_group(group_size_for(len, 4, 4));
    if (nv <= 1) {
        if (nv == 1 && g.gid == 0) {
            double s = 0.0;
            for (int i = g.gl; i < len; i += g.G) s += cabs2(R[(size_t)i * ldr]);
            s = group_sum(s, g);
            if (g.gl == 0) nrm[0] = s;
        }
        __syncthreads();
        return 0;
    }
    const int np = nv + (nv & 1);
    const int nr = np - 1;
    const double tol = fmax((double)len, 1.0) * 2.220446049250313e-16;
    const double tol2 = tol * tol;
    int sweep = 0;
    for (; sweep < 60; ++sweep) {
        for (int p = g.gid; p < nv; p += g.ng) {
            double s = 0.0;
            for (int i = g.gl; i < len; i += g.G) s += cabs2(R[p + (size_t)i * ldr]);
            s = group_sum(s, g);
            if (g.gl == 0) nrm[p] = s;
        }
        if (tid == 0) *flag = 0;
        __syncthreads();
        for (int r = 0; r < nr; ++r) {
            for (int pi = g.gid; pi < np / 2; pi += g.ng) {
                const int i1 = np - 1 - pi;
                int p = 0, q;
                if (pi != 0) { p = pi - 1 + r; if (p >= nr) p -= nr; ++p; }
                q = i1 - 1 + r; if (q >= nr) q -= nr; ++q;
                if (p >= nv || q >= nv) continue;
                const double al = nrm[p], be = nrm[q];
                double2 ga = cmk(0.0, 0.0);  // <x_p, x_q> = sum_i R[p,i] conj(R[q,i])
                for (int i = g.gl; i < len; i += g.G) cfma_bj(ga, R[p + (size_t)i * ldr], R[q + (size_t)i * ldr]);
                ga = group_sum2(ga, g);
                const double g2 = cabs2(ga);
                // rotate iff |gamma| > tol sqrt(al be)  (squared test, no square roots)
                if (g2 > tol2 * (al * be) && al > 0.0 && be > 0.0) {
                    const double ig = rsqrt(g2);  // 1/|gamma|
                    const double gm = g2 * ig;
                    const double zeta = 0.5 * (be - al) * ig;
                    const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
                    const double c = rsqrt(fma(t, t, 1.0));
                    const double sn = c * t;
                    // x_q <- e x_q with e = e^{-i phi}; on the rows of R (conjugated) the factor is gamma/|gamma|
                    const double2 ec = cmk(ga.x * ig, ga.y * ig);
                    for (int i = g.gl; i < len; i += g.G) {
                        const double2 a = R[p + (size_t)i * ldr];
                        const double2 b = cmul(ec, R[q + (size_t)i * ldr]);
                        R[p + (size_t)i * ldr] = csub(cscale(a, c), cscale(b, sn));
                        R[q + (size_t)i * ldr] = cadd(cscale(a, sn), cscale(b, c));
                    }
                    if (g.gl == 0) {
                        nrm[p] = al - t * gm;
                        nrm[q] = be + t * gm;
                        *flag = 1;
                    }
                }
            }
            __syncthreads();
        }
        if (*flag == 0) break;
        __syncthreads();
    }
    for (int p = g.gid; p < nv; p += g.ng) {
        double s = 0.0;
        for (int i = g.gl; i < len; i += g.G) s += cabs2(R[p + (size_t)i * ldr]);
        s = group_sum(s, g);
        if (g.gl == 0) nrm[p] = s;
    }
    __syncthreads();
    return sweep;
}


// ------------------------------------------------------------------ compile-time specialised
// One-sided Jacobi on the rows of R (see cta_jacobi_rows) for len <= G*E: every vector is
// held by a group of G lanes, E elements per lane, fully unrolled; the two vectors of a pair
// stay in registers between the inner product and the rotation.
template <int G, int E>
__device__ inline int jacobi_rows_t(double2* R, int ldr, int nv, int len, double* nrm, int* flag) {
    const int tid = threadIdx.x;
    const int gl = tid & (G - 1), gid = tid / G, ng = blockDim.x / G;
    const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((tid & 31) & ~(G - 1)));
    const int st = G * ldr;  // stride between a lane's elements
    __syncthreads();  // R was just written by the caller
    if (nv <= 1) {
        if (nv == 1 && gid == 0) {
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (gl + G * e < len) s += cabs2(R[(gl + G * e) * ldr]);
            for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
            if (gl == 0) nrm[0] = s;
        }
        __syncthreads();
        return 0;
    }
    const int np = nv + (nv & 1);
    const int nr = np - 1;
    const double tol = fmax((double)len, 1.0) * 2.220446049250313e-16;
    const double tol2 = tol * tol;
    int sweep = 0;
    for (; sweep < 60; ++sweep) {
        for (int p = gid; p < nv; p += ng) {
            const double2* rp = R + p + gl * ldr;
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (gl + G * e < len) s += cabs2(rp[e * st]);
            for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
            if (gl == 0) nrm[p] = s;
        }
        if (tid == 0) *flag = 0;
        __syncthreads();
        // absolute floor of the convergence test (DESIGN reading N3): |a_p^* a_q| <= 1e-28 sigma_1^2
        // counts as orthogonal -- it moves no singular value >= 1e-14 sigma_1 by more than 3e-13 sigma_1
        double mx = 0.0;
        for (int p = 0; p < nv; ++p) mx = fmax(mx, nrm[p]);
        const double floor2 = 1e-56 * mx * mx;
        for (int r = 0; r < nr; ++r) {
            // two pairs per iteration: independent dot products / rotations in flight
            for (int pi0 = gid; pi0 < np / 2; pi0 += 2 * ng) {
                int pp[2], qq[2];
                bool act[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pi = pi0 + h * ng;
                    act[h] = pi < np / 2;
                    const int i1 = np - 1 - pi;
                    int p = 0, q;
                    if (pi != 0) { p = pi - 1 + r; if (p >= nr) p -= nr; ++p; }
                    q = i1 - 1 + r; if (q >= nr) q -= nr; ++q;
                    act[h] = act[h] && p < nv && q < nv;
                    pp[h] = act[h] ? p : 0;
                    qq[h] = act[h] ? q : 0;
                }
                double2 a[2][E], b[2][E];
                double2 ga[2] = {cmk(0.0, 0.0), cmk(0.0, 0.0)};
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double2* rp = R + pp[h] + gl * ldr;
                    const double2* rq = R + qq[h] + gl * ldr;
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        if (act[h] && gl + G * e < len) {
                            a[h][e] = rp[e * st];
                            b[h][e] = rq[e * st];
                        } else {
                            a[h][e] = cmk(0.0, 0.0);
                            b[h][e] = cmk(0.0, 0.0);
                        }
                        cfma_bj(ga[h], a[h][e], b[h][e]);
                    }
                }
                for (int o = G >> 1; o > 0; o >>= 1) {
                    ga[0].x += __shfl_xor_sync(mask, ga[0].x, o);
                    ga[0].y += __shfl_xor_sync(mask, ga[0].y, o);
                    ga[1].x += __shfl_xor_sync(mask, ga[1].x, o);
                    ga[1].y += __shfl_xor_sync(mask, ga[1].y, o);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (!act[h]) continue;
                    const int p = pp[h], q = qq[h];
                    const double al = nrm[p], be = nrm[q];
                    const double g2 = cabs2(ga[h]);
                    if (g2 > fmax(tol2 * (al * be), floor2) && al > 0.0 && be > 0.0) {
                        // rotation by the smaller angle theta with tan(2 theta) = 2|g|/(be - al), from
                        // two dependent rsqrt only: with d = be - al, r = sqrt(d^2 + 4|g|^2),
                        // c^2 = (1 + |d|/r)/2 and t = tan(theta) = sign(d) |g| / (r c^2)
                        const double ig = rsqrt(g2);  // 1/|g| (independent chain)
                        const double gm = g2 * ig;
                        const double d = be - al;
                        const double ir = rsqrt(fma(d, d, 4.0 * g2));
                        const double c2 = fma(0.5 * fabs(d), ir, 0.5);
                        const double ic = rsqrt(c2);
                        const double c = c2 * ic;
                        const double t = (d >= 0.0 ? gm : -gm) * ir * (ic * ic);
                        const double sn = t * c;
                        const double2 ec = cmk(ga[h].x * ig, ga[h].y * ig);
                        double2* rp = R + p + gl * ldr;
                        double2* rq = R + q + gl * ldr;
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            if (gl + G * e < len) {
                                const double2 bb = cmul(ec, b[h][e]);
                                rp[e * st] = cmk(c * a[h][e].x - sn * bb.x, c * a[h][e].y - sn * bb.y);
                                rq[e * st] = cmk(sn * a[h][e].x + c * bb.x, sn * a[h][e].y + c * bb.y);
                            }
                        }
                        if (gl == 0) {
                            nrm[p] = al - t * gm;
                            nrm[q] = be + t * gm;
                            *flag = 1;
                        }
                    }
                }
            }
            __syncthreads();
        }
        if (*flag == 0) break;
        __syncthreads();
    }
    for (int p = gid; p < nv; p += ng) {
        const double2* rp = R + p + gl * ldr;
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (gl + G * e < len) s += cabs2(rp[e * st]);
        for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
        if (gl == 0) nrm[p] = s;
    }
    __syncthreads();
    return sweep;
}

// dispatch on the vector length (falls back to the generic version beyond 128)
__device__ inline int jacobi_rows_auto(double2* R, int ldr, int nv, int len, double* nrm, int* flag) {
    if (len <= 16) return jacobi_rows_t<4, 4>(R, ldr, nv, len, nrm, flag);
    if (len <= 32) return jacobi_rows_t<8, 4>(R, ldr, nv, len, nrm, flag);
    if (len <= 64) return jacobi_rows_t<16, 4>(R, ldr, nv, len, nrm, flag);
    if (len <= 128) return jacobi_rows_t<32, 4>(R, ldr, nv, len, nrm, flag);
    return cta_jacobi_rows(R, ldr, nv, len, nrm, flag);
}

// Pivoted QR (see cta_qrcp) for M <= G*E rows: column updates by groups of G lanes holding
// E elements each (unrolled, column values kept in registers for dot, update and norm).
template <int G, int E>
__device__ inline int qrcp_t(double2* B, int ldb, int M, int N, int* piv, double* nrm, double2* sh, int* s_piv,
                             double rank_rel2) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gl = tid & (G - 1), gid = tid / G, ng = blockDim.x / G;
    const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int K = min(M, N);
    __shared__ double s_total;
    __syncthreads();  // B was just written by the caller
    for (int c = tid; c < N; c += blockDim.x) piv[c] = c;
    for (int c = gid; c < N; c += ng) {
        const double2* bc = B + c * ldb + gl;
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (gl + G * e < M) s += cabs2(bc[G * e]);
        for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
        if (gl == 0) nrm[c] = s;
    }
    __syncthreads();
    int j = 0;
    for (; j < K; ++j) {
        if (warp == 0) {
            double best = -1.0, rem = 0.0;
            int bi = j;
            for (int c = j + lane; c < N; c += 32) {
                const double v = nrm[c];
                rem += v;
                if (v > best) { best = v; bi = c; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                rem += __shfl_xor_sync(0xffffffffu, rem, o);
                if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
            }
            const int pc = (rank_rel2 > 0.0 && j > 0 && rem <= rank_rel2 * s_total) ? -1 : bi;
            // swap columns j <-> pc (warp 0) and form the Householder vector of column j
            if (lane == 0) {
                if (j == 0) s_total = best;
                *s_piv = pc;
            }
            if (pc >= 0) {
                if (pc != j) {
                    for (int i = lane; i < M; i += 32) {
                        const double2 t = B[i + j * ldb];
                        B[i + j * ldb] = B[i + pc * ldb];
                        B[i + pc * ldb] = t;
                    }
                    if (lane == 0) {
                        const int t = piv[j]; piv[j] = piv[pc]; piv[pc] = t;
                        const double v = nrm[j]; nrm[j] = nrm[pc]; nrm[pc] = v;
                    }
                }
                __syncwarp();
                double2* colj = B + j * ldb;
                double s = 0.0;
                for (int i = j + 1 + lane; i < M; i += 32) s += cabs2(colj[i]);
                s = warp_sum(s);
                if (lane == 0) {
                    const double2 alpha = colj[j];
                    double tau = 0.0;
                    double2 beta = alpha;
                    if (s > HH_TINY) {  // tiny columns are left as they are (1/(xn (xn + aa)) would overflow)
                        const double aa = sqrt(cabs2(alpha));
                        const double xn = sqrt(s + aa * aa);
                        const double2 ph = aa > 0.0 ? cscale(alpha, 1.0 / aa) : cmk(1.0, 0.0);
                        beta = cscale(ph, -xn);
                        colj[j] = cscale(ph, aa + xn);
                        tau = 1.0 / (xn * (xn + aa));
                    }
                    sh[0] = beta;
                    sh[1] = cmk(tau, 0.0);
                }
            }
        }
        __syncthreads();
        if (*s_piv < 0) break;
        const double tau = sh[1].x;
        const double2* colj = B + j * ldb;
        double2 u[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = gl + G * e;
            u[e] = (i >= j && i < M) ? colj[i] : cmk(0.0, 0.0);
        }
        for (int c = j + 1 + gid; c < N; c += ng) {
            double2* bc = B + c * ldb;
            double2 x[E];
            double2 w = cmk(0.0, 0.0);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = gl + G * e;
                x[e] = (i < M) ? bc[i] : cmk(0.0, 0.0);
                cfma_cj(w, u[e], x[e]);
            }
            for (int o = G >> 1; o > 0; o >>= 1) {
                w.x += __shfl_xor_sync(mask, w.x, o);
                w.y += __shfl_xor_sync(mask, w.y, o);
            }
            w = cscale(w, tau);
            double s = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = gl + G * e;
                if (i >= j && i < M) {
                    x[e] = csub(x[e], cmul(u[e], w));
                    bc[i] = x[e];
                }
                if (i > j && i < M) s += cabs2(x[e]);
            }
            for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
            if (gl == 0) nrm[c] = s;
        }
        __syncthreads();
        if (tid == 0) B[j + j * ldb] = sh[0];
    }
    __syncthreads();
    return j;
}

__device__ inline int qrcp_auto(double2* B, int ldb, int M, int N, int* piv, double* nrm, double2* sh, int* s_piv,
                                double rank_rel2) {
    if (M <= 16) return qrcp_t<4, 4>(B, ldb, M, N, piv, nrm, sh, s_piv, rank_rel2);
    if (M <= 32) return qrcp_t<8, 4>(B, ldb, M, N, piv, nrm, sh, s_piv, rank_rel2);
    if (M <= 64) return qrcp_t<16, 4>(B, ldb, M, N, piv, nrm, sh, s_piv, rank_rel2);
    if (M <= 128) return qrcp_t<32, 4>(B, ldb, M, N, piv, nrm, sh, s_piv, rank_rel2);
    return cta_qrcp(B, ldb, M, N, piv, nrm, sh, s_piv, rank_rel2);
}


// Pivoted QR without column exchanges, for M <= G*E rows: step j picks the remaining physical
// column pc of largest norm (first on ties) and reflects rows j.. of every remaining column;
// piv[j] = pc, and column pc holds R[0..j, j] (logical order) above its Householder vector.
// Every warp selects the pivot and forms the reflector itself from the same shared data, so a
// step needs one barrier and no serial section; the column norms are double-buffered
// (nrm, nrm + N) because warps read step j's norms while others write step j+1's.
// Same R (up to the order of ties) as qrcp_t; stops at the numerical rank like qrcp_t.
// Requires nrm to hold 2 N doubles.  Returns the steps done.
template <int G, int E>
__device__ inline int qrcp_np_t(double2* B, int ldb, int M, int N, int* piv, double* nrm, double rank_rel2) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int gl = tid & (G - 1), gid = tid / G, ng = blockDim.x / G;
    const unsigned mask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int K = min(M, N);
    __syncthreads();  // B was just written by the caller
    for (int c = gid; c < N; c += ng) {
        const double2* bc = B + c * ldb + gl;
        double s = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (gl + G * e < M) s += cabs2(bc[G * e]);
        for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(mask, s, o);
        if (gl == 0) nrm[c] = s;
    }
    __syncthreads();
    double total = 0.0;
    int j = 0, prev_pc = -1;
    double2 prev_beta = cmk(0.0, 0.0);
    for (; j < K; ++j) {
        const double* ncur = nrm + (j & 1) * N;
        double* nnext = nrm + ((j + 1) & 1) * N;
        // pivot: every warp, identical reduction order
        double best = -1.0, rem = 0.0;
        int bi = N;
        for (int c = lane; c < N; c += 32) {
            const double v = ncur[c];
            if (v >= 0.0) {
                rem += v;
                if (v > best) { best = v; bi = c; }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            rem += __shfl_xor_sync(0xffffffffu, rem, o);
            if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (j == 0) total = rem;
        if (tid == 0 && prev_pc >= 0) B[j - 1 + prev_pc * ldb] = prev_beta;
        if (rank_rel2 > 0.0 && j > 0 && rem <= rank_rel2 * total) break;
        const int pc = bi;
        // reflector of column pc, rows j..M-1 (every warp)
        const double2* colp = B + pc * ldb;
        double sq = 0.0;
        for (int i = j + 1 + lane; i < M; i += 32) sq += cabs2(colp[i]);
        sq = warp_sum(sq);
        const double2 alpha = colp[j];
        double tau = 0.0;
        double2 beta = alpha, u0 = alpha;
        if (sq > HH_TINY) {  // see cta_qr_append
            const double aa = sqrt(cabs2(alpha));
            const double xn = sqrt(sq + aa * aa);
            const double2 ph = aa > 0.0 ? cscale(alpha, 1.0 / aa) : cmk(1.0, 0.0);
            beta = cscale(ph, -xn);
            u0 = cscale(ph, aa + xn);
            tau = 1.0 / (xn * (xn + aa));
        }
        double2 u[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = gl + G * e;
            u[e] = (i > j && i < M) ? colp[i] : (i == j ? u0 : cmk(0.0, 0.0));
        }
        for (int c = gid; c < N; c += ng) {
            if (c == pc || ncur[c] < 0.0) continue;
            double2* bc = B + c * ldb;
            double2 x[E];
            double2 w = cmk(0.0, 0.0);
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = gl + G * e;
                x[e] = (i < M) ? bc[i] : cmk(0.0, 0.0);
                cfma_cj(w, u[e], x[e]);
            }
            for (int o = G >> 1; o > 0; o >>= 1) {
                w.x += __shfl_xor_sync(mask, w.x, o);
                w.y += __shfl_xor_sync(mask, w.y, o);
            }
            w = cscale(w, tau);
            double s2 = 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = gl + G * e;
                if (i >= j && i < M) {
                    x[e] = csub(x[e], cmul(u[e], w));
                    bc[i] = x[e];
                }
                if (i > j && i < M) s2 += cabs2(x[e]);
            }
            for (int o = G >> 1; o > 0; o >>= 1) s2 += __shfl_xor_sync(mask, s2, o);
            if (gl == 0) nnext[c] = s2;
        }
        if (tid == 0) {
            nnext[pc] = -1.0;
            piv[j] = pc;
        }
        // columns finished earlier stay marked in the next buffer
        for (int c = tid; c < N; c += blockDim.x)
            if (ncur[c] < 0.0) nnext[c] = -1.0;
        prev_pc = pc;
        prev_beta = beta;
        __syncthreads();
    }
    if (tid == 0 && prev_pc >= 0 && j == K) B[K - 1 + prev_pc * ldb] = prev_beta;
    __syncthreads();
    return j;
}

__device__ inline int qrcp_np_auto(double2* B, int ldb, int M, int N, int* piv, double* nrm, double rank_rel2) {
    if (M <= 16) return qrcp_np_t<4, 4>(B, ldb, M, N, piv, nrm, rank_rel2);
    if (M <= 32) return qrcp_np_t<8, 4>(B, ldb, M, N, piv, nrm, rank_rel2);
    if (M <= 64) return qrcp_np_t<16, 4>(B, ldb, M, N, piv, nrm, rank_rel2);
    return qrcp_np_t<32, 4>(B, ldb, M, N, piv, nrm, rank_rel2);  // M <= 128
}

// ------------------------------------------------------------------ FP64 tensor cores (DMMA)
// D = A B + C for one 8x8x4 f64 tile (mma.sync m8n8k4; SASS DMMA).  Fragments: lane holds
// A[lane/4][lane%4], B[lane%4][lane/4], C/D[lane/4][2(lane%4)+{0,1}].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Complex 8x8 tile accumulator: (re, im) = (re, im) + a * b with 4 real DMMAs.
struct ZTile {
    double r0, r1, i0, i1;
};
__device__ __forceinline__ void ztile_mma(ZTile& t, double2 a, double2 b) {
    dmma884(t.r0, t.r1, a.x, b.x);
    dmma884(t.r0, t.r1, -a.y, b.y);
    dmma884(t.i0, t.i1, a.x, b.y);
    dmma884(t.i0, t.i1, a.y, b.x);
}

// out[i, nu] = w * sum_mu X[i0+i, mu] * op(S)[mu, nu] for i < nb, nu < k, on the FP64 tensor
// cores.  X: rx x k column-major (global or shared); op(S)[mu, nu] = Sg[nu + mu k] (conjugated
// if conj_s) or Sg[mu + nu k] if strided.  k is padded to a multiple of 32 with zero fragments
// (k = 125 for m = 5).  Each warp owns one 8-row tile and four 8-column tiles, reusing its A
// fragment across them.
template <bool FULL, bool UNROLL>
__device__ inline void chunk_gemm_S_dmma_t(const double2* X, int rx, int i0, int nb, const double2* Sg, bool conj_s,
                                           bool strided, double w, int k, double2* out, int ldo, bool conj_x) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nrt = (nb + 7) >> 3, nct4 = (k + 31) >> 5;
    const int ar = lane >> 2, ac = lane & 3;
    const double sgn = conj_s ? -1.0 : 1.0;
    const double sgx = conj_x ? -1.0 : 1.0;
    constexpr bool full = FULL;
    for (int task = warp; task < nrt * nct4; task += nw) {
        const int rt = task % nrt, cq = task / nrt;
        const int row = rt * 8 + ar;
        const bool rok = row < nb;
        ZTile t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = ZTile{0.0, 0.0, 0.0, 0.0};
        const double2* xa = X + i0 + row;
#pragma unroll(UNROLL ? 4 : 1)
        for (int mu = 0; mu < k; mu += 4) {
            const int mm = mu + ac;
            const bool mok = full || mm < k;
            double2 a = (rok && mok) ? xa[mm * rx] : cmk(0.0, 0.0);
            a.y *= sgx;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int nu = (cq * 4 + q) * 8 + ar;
                double2 b = cmk(0.0, 0.0);
                if (full || (mok && nu < k)) b = strided ? Sg[mm + nu * k] : Sg[nu + mm * k];
                b.y *= sgn;
                ztile_mma(t[q], a, b);
            }
        }
        const int orow = rt * 8 + ar;
        if (orow < nb) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int oc = (cq * 4 + q) * 8 + 2 * ac;
                if (full || oc < k) out[orow + oc * ldo] = cmk(w * t[q].r0, w * t[q].i0);
                if (full || oc + 1 < k) out[orow + (oc + 1) * ldo] = cmk(w * t[q].r1, w * t[q].i1);
            }
        }
    }
}

// UNROLL: unroll the k loop 4x (more loads in flight; more registers).  conj_x: X is stored
// conjugated (the column side read from the row basis pair at -c, adjoint symmetry).
template <bool UNROLL = false>
__device__ inline void chunk_gemm_S_dmma(const double2* X, int rx, int i0, int nb, const double2* Sg, bool conj_s,
                                         bool strided, double w, int k, double2* out, int ldo, bool conj_x = false) {
    if ((k & 31) == 0)
        chunk_gemm_S_dmma_t<true, UNROLL>(X, rx, i0, nb, Sg, conj_s, strided, w, k, out, ldo, conj_x);
    else
        chunk_gemm_S_dmma_t<false, UNROLL>(X, rx, i0, nb, Sg, conj_s, strided, w, k, out, ldo, conj_x);
}

// C = A B^H on the FP64 tensor cores: C[i, j] = sum_mu A[i, mu] conj(Bm[j, mu]) for i < na,
// j < nbm, mu < k (A: na x k, ld lda; Bm: nbm x k, ld ldbm; both column-major, global or shared).
// Tiles of 8 x 8 per warp task, k padded to a multiple of 4 with zero fragments.  STORE: write
// C (ld ldo); otherwise return this thread's share of ||C||_F^2 (padded entries are zero).
template <bool STORE, bool BCONJ = false>  // BCONJ: Bm is stored conjugated (C = A Bm^T of the stored data)
__device__ inline double dmma_abh(const double2* A, int lda, int na, const double2* Bm, int ldbm, int nbm, int k,
                                  double2* out, int ldo) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nrt = (na + 7) >> 3, nct = (nbm + 7) >> 3;
    const int ar = lane >> 2, ac = lane & 3;
    double part = 0.0;
    for (int task = warp; task < nrt * nct; task += nw) {
        const int rt = task % nrt, ct = task / nrt;
        const int row = rt * 8 + ar, col = ct * 8 + ar;
        const bool rok = row < na, cok = col < nbm;
        ZTile t{0.0, 0.0, 0.0, 0.0};
        const double2* ap = A + row;
        const double2* bp = Bm + col;
        int mu = 0;
#pragma unroll 4
        for (; mu + 4 <= k; mu += 4) {
            const int mm = mu + ac;
            const double2 a = rok ? ap[(size_t)mm * lda] : cmk(0.0, 0.0);
            const double2 b = cok ? (BCONJ ? bp[(size_t)mm * ldbm] : cconj(bp[(size_t)mm * ldbm])) : cmk(0.0, 0.0);
            ztile_mma(t, a, b);
        }
        if (mu < k) {
            const int mm = mu + ac;
            const double2 a = (rok && mm < k) ? ap[(size_t)mm * lda] : cmk(0.0, 0.0);
            const double2 b = (cok && mm < k) ? (BCONJ ? bp[(size_t)mm * ldbm] : cconj(bp[(size_t)mm * ldbm]))
                                              : cmk(0.0, 0.0);
            ztile_mma(t, a, b);
        }
        if constexpr (STORE) {
            const int oc = ct * 8 + 2 * ac;
            if (rok) {
                if (oc < nbm) out[row + (size_t)oc * ldo] = cmk(t.r0, t.i0);
                if (oc + 1 < nbm) out[row + (size_t)(oc + 1) * ldo] = cmk(t.r1, t.i1);
            }
        } else {
            part += (t.r0 * t.r0 + t.i0 * t.i0) + (t.r1 * t.r1 + t.i1 * t.i1);
        }
    }
    return part;
}

// C = A B^H as dmma_abh<true>, register-blocked: a warp task is an 8-row tile times 4 column
// tiles (32 columns), so each A fragment is loaded once for four DMMA chains (A re-read per 32
// instead of per 8 columns; four independent accumulations in flight).
__device__ inline void dmma_abh4(const double2* A, int lda, int na, const double2* Bm, int ldbm, int nbm, int k, double2* out,
                                 int ldo) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nrt = (na + 7) >> 3, ncq = (nbm + 31) >> 5;
    const int ar = lane >> 2, ac = lane & 3;
    for (int task = warp; task < nrt * ncq; task += nw) {
        const int rt = task % nrt, cq = task / nrt;
        const int row = rt * 8 + ar;
        const bool rok = row < na;
        ZTile t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = ZTile{0.0, 0.0, 0.0, 0.0};
        const double2* ap = A + row;
#pragma unroll 2
        for (int mu = 0; mu < k; mu += 4) {
            const int mm = mu + ac;
            const bool mok = mm < k;
            const double2 a = (rok && mok) ? ap[(size_t)mm * lda] : cmk(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int col = (cq * 4 + q) * 8 + ar;
                const double2 b = (mok && col < nbm) ? cconj(Bm[col + (size_t)mm * ldbm]) : cmk(0.0, 0.0);
                ztile_mma(t[q], a, b);
            }
        }
        if (rok) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int oc = (cq * 4 + q) * 8 + 2 * ac;
                if (oc < nbm) out[row + (size_t)oc * ldo] = cmk(t[q].r0, t[q].i0);
                if (oc + 1 < nbm) out[row + (size_t)(oc + 1) * ldo] = cmk(t[q].r1, t[q].i1);
            }
        }
    }
}

// ||A B^H||_F^2 share of this thread (as dmma_abh<false, BCONJ>), register-blocked as dmma_abh4
template <bool BCONJ>
__device__ inline double dmma_abh4_norm(const double2* A, int lda, int na, const double2* Bm, int ldbm, int nbm, int k) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int nrt = (na + 7) >> 3, ncq = (nbm + 31) >> 5;
    const int ar = lane >> 2, ac = lane & 3;
    double part = 0.0;
    for (int task = warp; task < nrt * ncq; task += nw) {
        const int rt = task % nrt, cq = task / nrt;
        const int row = rt * 8 + ar;
        const bool rok = row < na;
        ZTile t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = ZTile{0.0, 0.0, 0.0, 0.0};
        const double2* ap = A + row;
#pragma unroll 2
        for (int mu = 0; mu < k; mu += 4) {
            const int mm = mu + ac;
            const bool mok = mm < k;
            const double2 a = (rok && mok) ? ap[(size_t)mm * lda] : cmk(0.0, 0.0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int col = (cq * 4 + q) * 8 + ar;
                double2 b = cmk(0.0, 0.0);
                if (mok && col < nbm) {
                    b = Bm[col + (size_t)mm * ldbm];
                    if (!BCONJ) b = cconj(b);
                }
                ztile_mma(t[q], a, b);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) part += (t[q].r0 * t[q].r0 + t[q].i0 * t[q].i0) + (t[q].r1 * t[q].r1 + t[q].i1 * t[q].i1);
    }
    return part;
}

// Upper-triangular k x k factor R in shared memory: dense column-major (ld ldr) or packed by
// columns (R[i, c] at i + c(c+1)/2, 8 k(k+1) bytes; used when the dense square does not fit,
// e.g. k = 125: 126 KB packed instead of 250 KB).
template <bool PK>
__device__ __forceinline__ int ridx(int i, int c, int ldr) {
    return PK ? i + ((c * (c + 1)) >> 1) : i + c * ldr;
}
template <bool PK>
__host__ __device__ inline size_t r_elems(int k, int ldr) {
    return PK ? (size_t)k * (k + 1) / 2 : (size_t)ldr * k;
}

// Annihilate the nb x k chunk B (nb <= 16 E) into the k x k upper-triangular smem factor R:
// [R; B] = Q [R'; 0] by k structured Householder reflections, each touching row j of R and the
// nb rows of B only (the rows of R below j are zero in column j).  Lane groups of 16 own one
// column at a time, E rows of B per lane (rows gl + 16 e) plus row j of R on lane 0, two columns
// per iteration (independent reductions in flight).  One barrier per reflection: every warp forms
// the reflector itself from ||B(:, j)||^2, which group 0 -- it updates column j during step j-1 --
// publishes in shared memory (look-ahead: no reduction over B on the critical path); the new
// diagonal beta_j is stored one step later (nobody reads R[j, j] during step j+1).
template <bool PK, int E, int G = 16>  // G lanes per column group (16 or 8), E rows per lane: nb <= G E
__device__ inline void cta_qr_append(double2* R, int ldr, double2* B, int ldb, int nb, int k) {
    // reflector of the next step (double-buffered by step parity): tau, u0, beta, formed once by
    // group 0 right after it applied the current reflector to column j + 1 (look-ahead)
    __shared__ double2 s_u0[2], s_beta[2];
    __shared__ double s_tau[2];
    const int tid = threadIdx.x, lane = tid & 31;
    const int gl = tid & (G - 1), gid = tid / G, ng = blockDim.x / G;
    const unsigned mask = ((1u << G) - 1u) << (lane & ~(G - 1));
    __syncthreads();
    auto col_norm = [&](int c) {  // G-lane reduction of ||B(:, c)||^2 (group-uniform result)
        double v = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (gl + G * e < nb) v += cabs2(B[(size_t)c * ldb + gl + G * e]);
#pragma unroll
        for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
        return v;
    };
    // Householder reflector of column j from s = ||B(:, j)||^2 and alpha = R[j, j] (lane 0 of group 0)
    auto publish = [&](int j, double s) {
        const double2 alpha = R[ridx<PK>(j, j, ldr)];
        double tau = 0.0;
        double2 beta = alpha, u0 = cmk(0.0, 0.0);
        if (s > HH_TINY) {  // tiny columns are left as they are (1/(xn (xn + aa)) would overflow)
            const double aa = sqrt(cabs2(alpha));
            const double xn = sqrt(s + aa * aa);
            const double2 ph = aa > 0.0 ? cscale(alpha, 1.0 / aa) : cmk(1.0, 0.0);
            beta = cscale(ph, -xn);
            u0 = cscale(ph, aa + xn);
            tau = 1.0 / (xn * (xn + aa));
        }
        s_tau[j & 1] = tau;
        s_u0[j & 1] = u0;
        s_beta[j & 1] = beta;
    };
    if (gid == 0 && k > 0) {
        const double v = col_norm(0);
        if (gl == 0) publish(0, v);
    }
    __syncthreads();
    for (int j = 0; j < k; ++j) {
        const double2* bj = B + j * ldb;
        const double tau = s_tau[j & 1];
        const double2 u0 = s_u0[j & 1];
        if (tid == 0) R[ridx<PK>(j, j, ldr)] = s_beta[j & 1];  // (nobody reads R[j, j] after the publish)
        if (tau != 0.0) {
            double2 u[E];
#pragma unroll
            for (int e = 0; e < E; ++e) u[e] = (gl + G * e < nb) ? bj[gl + G * e] : cmk(0.0, 0.0);
            for (int c = j + 1 + gid; c < k; c += 2 * ng) {
                const int c2 = c + ng;
                const bool two = c2 < k;
                double2* bc = B + c * ldb;
                double2* bc2 = B + c2 * ldb;
                double2 x[E], x2[E];
                double2 rj = cmk(0.0, 0.0), rj2 = cmk(0.0, 0.0);
                double2 w = cmk(0.0, 0.0), w2 = cmk(0.0, 0.0);
                if (gl == 0) {
                    rj = R[ridx<PK>(j, c, ldr)];
                    cfma_cj(w, u0, rj);
                    if (two) {
                        rj2 = R[ridx<PK>(j, c2, ldr)];
                        cfma_cj(w2, u0, rj2);
                    }
                }
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const bool ok = gl + G * e < nb;
                    x[e] = ok ? bc[gl + G * e] : cmk(0.0, 0.0);
                    x2[e] = (ok && two) ? bc2[gl + G * e] : cmk(0.0, 0.0);
                    cfma_cj(w, u[e], x[e]);
                    cfma_cj(w2, u[e], x2[e]);
                }
#pragma unroll
                for (int o = G >> 1; o > 0; o >>= 1) {
                    w.x += __shfl_xor_sync(mask, w.x, o);
                    w.y += __shfl_xor_sync(mask, w.y, o);
                    w2.x += __shfl_xor_sync(mask, w2.x, o);
                    w2.y += __shfl_xor_sync(mask, w2.y, o);
                }
                w = cscale(w, tau);
                w2 = cscale(w2, tau);
                if (gl == 0) {
                    R[ridx<PK>(j, c, ldr)] = csub(rj, cmul(u0, w));
                    if (two) R[ridx<PK>(j, c2, ldr)] = csub(rj2, cmul(u0, w2));
                }
                double vn = 0.0;  // ||B(:, j+1)||^2 after this reflection (group 0, column j + 1)
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (gl + G * e < nb) {
                        x[e] = csub(x[e], cmul(u[e], w));
                        bc[gl + G * e] = x[e];
                        vn += cabs2(x[e]);
                        if (two) bc2[gl + G * e] = csub(x2[e], cmul(u[e], w2));
                    }
                if (c == j + 1) {  // only group 0 (gid == 0) meets column j + 1: next reflector now
#pragma unroll
                    for (int o = G >> 1; o > 0; o >>= 1) vn += __shfl_xor_sync(mask, vn, o);
                    if (gl == 0) publish(j + 1, vn);
                }
            }
        } else if (gid == 0 && j + 1 < k) {  // no reflection: column j + 1 unchanged
            const double v = col_norm(j + 1);
            if (gl == 0) publish(j + 1, v);
        }
        __syncthreads();
    }
}

// Flag-synchronised form of cta_qr_append: the same reflections, but no block barrier per
// reflection.  Warp w owns the columns c = w (mod #warps) for the whole chunk (its two 16-lane halves
// take two columns at a time, E rows per lane); the owner of column j+1 applies reflection j to it
// first, forms reflection j+1 and publishes it (tau, u0 in shared arrays indexed by the step, then a
// release store of the step counter); every other warp only waits (acquire load) until reflection j+1
// is published before applying it.  Warps run ahead or behind each other -- a reflection's data never
// changes after its publication (column j is final once reflected, row j of R belongs to the column
// owners), so the only synchronisation is producer -> consumers.  s_tau / s_u0 hold k entries.
template <bool PK, int E, int G = 8>  // G lanes per column (32/G columns per warp at once), E rows per lane: nb <= G E
__device__ inline void cta_qr_append_flag(double2* R, int ldr, double2* B, int ldb, int nb, int k, double* s_tau,
                                          double2* s_u0, int* s_step) {
    constexpr int NQ = 32 / G;  // column slots per warp
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const int gl = tid & (G - 1), half = lane / G;
    const unsigned mask = ((1u << G) - 1u) << (lane & ~(G - 1));
    cuda::atomic_ref<int, cuda::thread_scope_block> step(*s_step);
    auto reflector = [&](int j, double s) {  // lane 0 of the owner warp: publish reflection j
        const double2 alpha = R[ridx<PK>(j, j, ldr)];
        double tau = 0.0;
        double2 beta = alpha, u0 = cmk(0.0, 0.0);
        if (s > HH_TINY) {  // tiny columns are left as they are (1/(xn (xn + aa)) would overflow)
            const double aa = sqrt(cabs2(alpha));
            const double xn = sqrt(s + aa * aa);
            const double2 ph = aa > 0.0 ? cscale(alpha, 1.0 / aa) : cmk(1.0, 0.0);
            beta = cscale(ph, -xn);
            u0 = cscale(ph, aa + xn);
            tau = 1.0 / (xn * (xn + aa));
        }
        s_tau[j] = tau;
        s_u0[j] = u0;
        R[ridx<PK>(j, j, ldr)] = beta;  // nobody reads R[j, j] again
        step.store(j, cuda::memory_order_release);
    };
    auto col_norm16 = [&](int c) {  // ||B(:, c)||^2 over one G-lane slot
        double v = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (gl + G * e < nb) v += cabs2(B[(size_t)c * ldb + gl + G * e]);
#pragma unroll
        for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
        return v;
    };
    __syncthreads();
    if (tid == 0) *s_step = -1;
    __syncthreads();
    if (warp == 0 && k > 0) {  // column 0 is owned by warp 0
        const double v = col_norm16(0);  // (both halves compute it; lane 0 publishes)
        if (lane == 0) reflector(0, v);
    }
    // own columns of this warp: c = warp + nw * i; in a step the two halves take two of them
    for (int j = 0; j < k; ++j) {
        // wait for reflection j (the owner of column j published it after reflection j-1)
        if (lane == 0)
            while (step.load(cuda::memory_order_acquire) < j) __nanosleep(20);
        __syncwarp();
        cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_block);
        const double tau = s_tau[j];
        if (tau == 0.0) {  // no reflection: the owner of column j + 1 publishes its reflector from the column
            if (j + 1 < k && (j + 1) % nw == warp) {
                const double v = col_norm16(j + 1);
                if (lane == 0) reflector(j + 1, v);
            }
            continue;
        }
        const double2 u0 = s_u0[j];
        const double2* bj = B + (size_t)j * ldb;
        double2 u[E];
#pragma unroll
        for (int e = 0; e < E; ++e) u[e] = (gl + G * e < nb) ? bj[gl + G * e] : cmk(0.0, 0.0);
        // this warp's columns > j, the column j+1 first (it feeds the next reflection)
        int c0 = warp;
        if (c0 <= j) c0 += ((j - c0) / nw + 1) * nw;
        for (int cb = c0; cb < k; cb += NQ * nw) {
            const int c = cb + half * nw;  // slot q takes column cb + q nw
            const bool ok = c < k;
            double2 x[E];
            double2 rj = cmk(0.0, 0.0), w = cmk(0.0, 0.0);
            if (ok && gl == 0) {
                rj = R[ridx<PK>(j, c, ldr)];
                cfma_cj(w, u0, rj);
            }
#pragma unroll
            for (int e = 0; e < E; ++e) {
                x[e] = (ok && gl + G * e < nb) ? B[(size_t)c * ldb + gl + G * e] : cmk(0.0, 0.0);
                cfma_cj(w, u[e], x[e]);
            }
#pragma unroll
            for (int o = G >> 1; o > 0; o >>= 1) {
                w.x += __shfl_xor_sync(mask, w.x, o);
                w.y += __shfl_xor_sync(mask, w.y, o);
            }
            w = cscale(w, tau);
            double vn = 0.0;
            if (ok) {
                if (gl == 0) R[ridx<PK>(j, c, ldr)] = csub(rj, cmul(u0, w));
#pragma unroll
                for (int e = 0; e < E; ++e)
                    if (gl + G * e < nb) {
                        x[e] = csub(x[e], cmul(u[e], w));
                        B[(size_t)c * ldb + gl + G * e] = x[e];
                        vn += cabs2(x[e]);
                    }
            }
            if (cb == c0 && c0 == j + 1) {  // column j+1 is this warp's (half 0): form reflection j+1
#pragma unroll
                for (int o = G >> 1; o > 0; o >>= 1) vn += __shfl_xor_sync(mask, vn, o);
                __syncwarp();  // (the half-0 lanes wrote column j+1 and row j of R)
                if (lane == 0) {
                    cuda::atomic_thread_fence(cuda::memory_order_release, cuda::thread_scope_block);
                    reflector(j + 1, vn);
                }
            }
        }
    }
    __syncthreads();
}

// Blocked form of cta_qr_append (compact WY, panels of 8 columns): [R; B] = Q [R'; 0] with the same
// structured reflectors H_j = I - tau_j u_j u_j^*, u_j = [u0_j e_j; b_j] (row j of R and the nb <= 32
// rows of B).  Warp 0 factorises a panel of 8 columns in registers (lane = row of B: warp-synchronous,
// no block barrier per reflection) and builds T (8 x 8 upper triangular, H_1...H_8 = I - V T V^*);
// then every warp applies (H_1...H_8)^* = I - V T^* V^* to 8-column tiles of the trailing matrix on
// the FP64 tensor cores: W = D^* R_p + U^* B_c (DMMA, K = nb), W2 = T^* W, R_p -= D W2, B_c -= U W2
// (DMMA, K = 8) -- two block barriers per panel instead of one per column.
struct WyPanel {
    double2 u0[8];
    double tau[8];
    double2 T[64];  // T[i + 8 j]
};

template <bool PK>
__device__ inline void cta_qr_append_wy(double2* R, int ldr, double2* B, int ldb, int nb, int k, WyPanel* wp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    const unsigned FULL = 0xffffffffu;
    __syncthreads();
    for (int j0 = 0; j0 < k; j0 += 8) {
        const int P = min(8, k - j0);
        if (warp == 0) {
            double2 b[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) b[c] = (lane < nb && c < P) ? B[lane + (size_t)(j0 + c) * ldb] : cmk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j >= P) break;
                double s = 0.0;
                {
                    double v = cabs2(b[j]);
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
                    s = v;
                }
                const double2 alpha = R[ridx<PK>(j0 + j, j0 + j, ldr)];
                double tau = 0.0;
                double2 beta = alpha, u0 = cmk(0.0, 0.0);
                if (s > HH_TINY) {  // as cta_qr_append: tiny columns are left in place
                    const double aa = sqrt(cabs2(alpha));
                    const double xn = sqrt(s + aa * aa);
                    const double2 ph = aa > 0.0 ? cscale(alpha, 1.0 / aa) : cmk(1.0, 0.0);
                    beta = cscale(ph, -xn);
                    u0 = cscale(ph, aa + xn);
                    tau = 1.0 / (xn * (xn + aa));
                }
                // one batched reduction: b_j^* b_c for the panel columns c > j, and the Gram entries
                // z_i = b_i^* b_j (i < j) of the reflector vectors for T
                double2 dv[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    dv[c] = cmk(0.0, 0.0);
                    if (c > j && c < P) cfma_cj(dv[c], b[j], b[c]);
                    if (c < j) cfma_cj(dv[c], b[c], b[j]);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (c == j || c >= P) continue;
                        dv[c].x += __shfl_xor_sync(FULL, dv[c].x, o);
                        dv[c].y += __shfl_xor_sync(FULL, dv[c].y, o);
                    }
                if (tau != 0.0) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        if (c <= j || c >= P) continue;
                        const double2 rjc = R[ridx<PK>(j0 + j, j0 + c, ldr)];
                        double2 w = dv[c];
                        cfma_cj(w, u0, rjc);
                        w = cscale(w, tau);
                        if (lane == 0) R[ridx<PK>(j0 + j, j0 + c, ldr)] = csub(rjc, cmul(u0, w));
                        b[c] = csub(b[c], cmul(b[j], w));
                    }
                }
                // T(0:j, j) = -tau_j T(0:j, 0:j) z (lane i computes row i), T(j, j) = tau_j
                if (lane < j) {
                    double2 acc = cmk(0.0, 0.0);
#pragma unroll
                    for (int m = 0; m < 8; ++m)
                        if (m >= lane && m < j) cfma(acc, wp->T[lane + 8 * m], dv[m]);
                    wp->T[lane + 8 * j] = cscale(acc, -tau);
                }
                if (lane == 0) {
                    wp->T[j + 8 * j] = cmk(tau, 0.0);
                    wp->u0[j] = u0;
                    wp->tau[j] = tau;
                    R[ridx<PK>(j0 + j, j0 + j, ldr)] = beta;
                }
                __syncwarp();
            }
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (lane < nb && c < P) B[lane + (size_t)(j0 + c) * ldb] = b[c];  // reflector vectors u_B
        }
        __syncthreads();
        // trailing columns [j0 + 8, k) in tiles of 8 per warp
        const int cf = j0 + 8;
        const int ntile = cf < k ? (k - cf + 7) >> 3 : 0;
        const int ar = lane >> 2, ac = lane & 3;
        for (int tile = warp; tile < ntile; tile += nw) {
            const int c0 = cf + tile * 8;
            // W = U^* B_c  (8 x 8, K = nb)
            ZTile t{0.0, 0.0, 0.0, 0.0};
            for (int r0 = 0; r0 < nb; r0 += 4) {
                const int r = r0 + ac;
                const double2 a = (r < nb && ar < P) ? cconj(B[r + (size_t)(j0 + ar) * ldb]) : cmk(0.0, 0.0);
                const double2 bb = (r < nb && c0 + ar < k) ? B[r + (size_t)(c0 + ar) * ldb] : cmk(0.0, 0.0);
                ztile_mma(t, a, bb);
            }
            // + D^* R_p: lane holds W[ar][2ac], W[ar][2ac+1]
            const int n0 = c0 + 2 * ac, n1 = n0 + 1;
            double2 w0 = cmk(t.r0, t.i0), w1 = cmk(t.r1, t.i1);
            if (ar < P) {
                const double2 u0 = wp->u0[ar];
                if (n0 < k) cfma_cj(w0, u0, R[ridx<PK>(j0 + ar, n0, ldr)]);
                if (n1 < k) cfma_cj(w1, u0, R[ridx<PK>(j0 + ar, n1, ldr)]);
            }
            // W2 = T^* W: W2[i][n] = sum_{j <= i} conj(T[j][i]) W[j][n]; W[j][n] lives in lane 4 j + ac
            double2 v0 = cmk(0.0, 0.0), v1 = cmk(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int src = 4 * j + ac;
                const double2 x0 = cmk(__shfl_sync(FULL, w0.x, src), __shfl_sync(FULL, w0.y, src));
                const double2 x1 = cmk(__shfl_sync(FULL, w1.x, src), __shfl_sync(FULL, w1.y, src));
                if (j <= ar && ar < P && j < P) {
                    const double2 tj = wp->T[j + 8 * ar];
                    cfma_cj(v0, tj, x0);
                    cfma_cj(v1, tj, x1);
                }
            }
            // R_p -= D W2
            if (ar < P) {
                const double2 u0 = wp->u0[ar];
                if (n0 < k) R[ridx<PK>(j0 + ar, n0, ldr)] = csub(R[ridx<PK>(j0 + ar, n0, ldr)], cmul(u0, v0));
                if (n1 < k) R[ridx<PK>(j0 + ar, n1, ldr)] = csub(R[ridx<PK>(j0 + ar, n1, ldr)], cmul(u0, v1));
            }
            // B_c -= U W2  (nb x 8, K = 8): B operand W2[i][n], i = 4 kk + ac, n = ar, held by lane 4 i + (ar >> 1)
            for (int rt = 0; rt < nb; rt += 8) {
                ZTile o{0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const int i = 4 * kk + ac;
                    const int src = 4 * i + (ar >> 1);
                    const double e0 = __shfl_sync(FULL, v0.x, src), e1 = __shfl_sync(FULL, v0.y, src);
                    const double f0 = __shfl_sync(FULL, v1.x, src), f1 = __shfl_sync(FULL, v1.y, src);
                    const double2 bb = (ar & 1) ? cmk(f0, f1) : cmk(e0, e1);
                    const int r = rt + ar;
                    const double2 a = (r < nb && i < P) ? B[r + (size_t)(j0 + i) * ldb] : cmk(0.0, 0.0);
                    ztile_mma(o, a, bb);
                }
                const int r = rt + ar;
                if (r < nb) {
                    if (n0 < k) B[r + (size_t)n0 * ldb] = csub(B[r + (size_t)n0 * ldb], cmk(o.r0, o.i0));
                    if (n1 < k) B[r + (size_t)n1 * ldb] = csub(B[r + (size_t)n1 * ldb], cmk(o.r1, o.i1));
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace dh2
