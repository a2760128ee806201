// sm_100a kernels of the DH^2 set-up and hybrid recompression.
// Every kernel cites the PAPER.md passage (P:<line>) it implements.
#include <cmath>
#include <cstdio>

#include "dh2_kernels.cuh"

namespace dh2 {

__device__ double g_cheb[2 * MMAX];  // z_j and 1/prod_{i!=j}(z_j - z_i) of the current order

static inline int odd_ld(int r) { return (r | 1); }

// ============================================================== set-up (§2)

// Chebyshev points of the first kind z_j = cos(pi (2j+1)/(2m)) (Q6) and the
// barycentric denominators of the 1-D Lagrange polynomials.
__global__ void k_cheb(int m) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        for (int j = 0; j < m; ++j) g_cheb[j] = cos(M_PI * (2 * j + 1) / (2.0 * m));
        for (int j = 0; j < m; ++j) {
            double d = 1.0;
            for (int i = 0; i < m; ++i)
                if (i != j) d *= (g_cheb[j] - g_cheb[i]);
            g_cheb[MMAX + j] = 1.0 / d;
        }
    }
}

// Quadrature points of Radon's 7-point degree-5 rule on every triangle, in cluster order
// (v_{tc,i nu} integrals; DESIGN reading Q11).  qp = (x, y, z, |tau| w_q).
__global__ void k_quad(PlanD P) {
    const double s15 = sqrt(15.0);
    const double A = (6.0 - s15) / 21.0, B = (6.0 + s15) / 21.0;
    const double WA = (155.0 - s15) / 1200.0, WB = (155.0 + s15) / 1200.0;
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= P.n * 7) return;
    int p = idx / 7, q = idx % 7;
    int64_t tr = P.perm[p];
    const double* v0 = P.xyz + 3 * P.tri[3 * tr];
    const double* v1 = P.xyz + 3 * P.tri[3 * tr + 1];
    const double* v2 = P.xyz + 3 * P.tri[3 * tr + 2];
    double l0, l1, l2, w;
    switch (q) {
        case 0: l0 = l1 = l2 = 1.0 / 3.0; w = 9.0 / 40.0; break;
        case 1: l0 = A; l1 = A; l2 = 1.0 - 2.0 * A; w = WA; break;
        case 2: l0 = A; l1 = 1.0 - 2.0 * A; l2 = A; w = WA; break;
        case 3: l0 = 1.0 - 2.0 * A; l1 = A; l2 = A; w = WA; break;
        case 4: l0 = B; l1 = B; l2 = 1.0 - 2.0 * B; w = WB; break;
        case 5: l0 = B; l1 = 1.0 - 2.0 * B; l2 = B; w = WB; break;
        default: l0 = 1.0 - 2.0 * B; l1 = B; l2 = B; w = WB; break;
    }
    double e1[3], e2[3], x[3];
    for (int a = 0; a < 3; ++a) {
        e1[a] = v1[a] - v0[a];
        e2[a] = v2[a] - v0[a];
        x[a] = l0 * v0[a] + l1 * v1[a] + l2 * v2[a];
    }
    double c0 = e1[1] * e2[2] - e1[2] * e2[1], c1 = e1[2] * e2[0] - e1[0] * e2[2], c2 = e1[0] * e2[1] - e1[1] * e2[0];
    double area = 0.5 * sqrt(c0 * c0 + c1 * c1 + c2 * c2);
    P.qp[idx] = make_double4(x[0], x[1], x[2], area * w);
}

// Tensor Chebyshev grid on the tight box of every cluster: xi = mid + half z,
// a collapsed axis (hi-lo <= 1e-12 diam) keeps one node at mid (DESIGN reading Q7).
__global__ void k_grid(PlanD P) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.nclusters) return;
    GridD g;
    double ext[3];
    for (int a = 0; a < 3; ++a) ext[a] = P.c_hi[3 * t + a] - P.c_lo[3 * t + a];
    double diam = sqrt((ext[0] * ext[0] + ext[1] * ext[1]) + ext[2] * ext[2]);
    for (int a = 0; a < 3; ++a) {
        g.mid[a] = 0.5 * (P.c_lo[3 * t + a] + P.c_hi[3 * t + a]);
        g.half[a] = 0.5 * ext[a];
        g.flat[a] = ext[a] <= 1e-12 * diam;
        for (int j = 0; j < MMAX; ++j)
            g.nodes[a][j] = (j < P.m) ? (g.flat[a] ? g.mid[a] : g.mid[a] + g.half[a] * g_cheb[j]) : 0.0;
    }
    P.grid[t] = g;
}

// Output stage of k_leafV: thread per (triangle i, z-index jz) accumulates the m^2 entries
// nu = jx + m jy + m^2 jz over the 7 quadrature points from registers (tensor structure of
// L_{t,nu} = L_x L_y L_z), writes coalesced along i.
template <int MM>
__device__ inline void leafV_out(double2* V, int nt, const double2* ph, const double* L) {
    for (int task = threadIdx.x; task < nt * MM; task += blockDim.x) {
        const int i = task % nt, jz = task / nt;
        double2 acc[MM][MM];
#pragma unroll
        for (int a = 0; a < MM; ++a)
#pragma unroll
            for (int b = 0; b < MM; ++b) acc[a][b] = cmk(0.0, 0.0);
        for (int q = 0; q < 7; ++q) {
            const double* Lq = L + ((i * 7 + q) * 3) * MM;
            const double2 p = ph[i * 7 + q];
            double lx[MM], ly[MM];
#pragma unroll
            for (int j = 0; j < MM; ++j) {
                lx[j] = Lq[j];
                ly[j] = Lq[MM + j];
            }
            const double lz = Lq[2 * MM + jz];
            const double pzx = p.x * lz, pzy = p.y * lz;  // p L_z, then (p L_z) L_y: 2 FMAs per entry
#pragma unroll
            for (int b = 0; b < MM; ++b) {
                const double qx = pzx * ly[b], qy = pzy * ly[b];
#pragma unroll
                for (int a = 0; a < MM; ++a) {
                    acc[b][a].x = fma(qx, lx[a], acc[b][a].x);
                    acc[b][a].y = fma(qy, lx[a], acc[b][a].y);
                }
            }
        }
#pragma unroll
        for (int b = 0; b < MM; ++b)
#pragma unroll
            for (int a = 0; a < MM; ++a) V[(size_t)(a + MM * b + MM * MM * jz) * nt + i] = acc[b][a];
    }
}

// Leaf bases V_tc[i,nu] = sum_q |tau_i| w_q exp(i kappa <x_iq, c>) L_{t,nu}(x_iq)
// (modified Lagrange polynomials P:270-275).  One CTA per leaf basis pair.
template <int MM>  // Chebyshev order m (0: runtime m, generic output loop); one register budget per m
__global__ void k_leafV(PlanD P, const int* bps) {
    extern __shared__ double2 sm[];
    const int bp = bps[blockIdx.x];
    const int t = P.bp_t[bp];
    const int nt = P.c_size[t];
    const int64_t b0 = P.c_begin[t];
    const int m = P.m, k = P.k;
    __shared__ GridD g;
    __shared__ double cheb[2 * MMAX];
    if (threadIdx.x == 0) g = P.grid[t];
    if (threadIdx.x < 2 * MMAX) cheb[threadIdx.x] = g_cheb[threadIdx.x];
    __syncthreads();
    const double* c = P.dirs + 3 * P.bp_dir[bp];
    double2* ph = sm;                              // nt*7
    double* L = reinterpret_cast<double*>(sm + nt * 7);  // nt*7*3*m
    for (int idx = threadIdx.x; idx < nt * 7; idx += blockDim.x) {
        double4 q = P.qp[b0 * 7 + idx];
        double arg = P.kappa * ((q.x * c[0] + q.y * c[1]) + q.z * c[2]);
        double s, co;
        sincos(arg, &s, &co);
        ph[idx] = cmk(q.w * co, q.w * s);
        double xs[3] = {q.x, q.y, q.z};
        for (int a = 0; a < 3; ++a) lagrange_axis(g, a, m, cheb, cheb + MMAX, xs[a], L + (idx * 3 + a) * m);
    }
    __syncthreads();
    double2* V = P.V + P.bp_V_off[bp];
    if constexpr (MM > 0) {
        leafV_out<MM>(V, nt, ph, L);
    } else {
        for (int idx = threadIdx.x; idx < nt * k; idx += blockDim.x) {
            int i = idx % nt, nu = idx / nt;
            int jx = nu % m, jy = (nu / m) % m, jz = nu / (m * m);
            double2 acc = cmk(0.0, 0.0);
            for (int q = 0; q < 7; ++q) {
                const double* Lq = L + ((i * 7 + q) * 3) * m;
                double l = Lq[jx] * Lq[m + jy] * Lq[2 * m + jz];
                double2 p = ph[i * 7 + q];
                acc.x = fma(p.x, l, acc.x);
                acc.y = fma(p.y, l, acc.y);
            }
            V[(size_t)nu * nt + i] = acc;
        }
    }
}

// Transfer factors of E_{t'c} (Eq. 10): with c' = sd_t(c) the entry
// exp(i kappa <xi_{t'nu'}, c - c'>) L_{t,nu}(xi_{t'nu'}) factorises over the axes,
// E = Ez (x) Ey (x) Ex with E_a[j',j] = exp(i kappa xi'_{a,j'} (c-c')_a) L_{t,a,j}(xi'_{a,j'}).
__global__ void k_E(PlanD P, const int* bps, int nbps) {
    const int m = P.m, m2 = m * m;
    int idx = blockIdx.x * blockDim.x + threadIdx.x;
    int per = 2 * 3 * m2;
    if (idx >= nbps * per) return;
    int ib = idx / per, r = idx % per;
    int ci = r / (3 * m2);
    int a = (r / m2) % 3;
    int jp = (r % m2) / m, j = r % m;
    int bp = bps[ib];
    int t = P.bp_t[bp];
    int cbp = ci == 0 ? P.bp_child0[bp] : P.bp_child1[bp];
    int tc = P.bp_t[cbp];
    const GridD& gp = P.grid[t];
    const GridD& gc = P.grid[tc];
    double cheb[2 * MMAX];
    for (int i = 0; i < 2 * MMAX; ++i) cheb[i] = g_cheb[i];
    double xi = gc.nodes[a][jp];
    double L[MMAX];
    lagrange_axis(gp, a, m, cheb, cheb + MMAX, xi, L);
    double dc = P.dirs[3 * P.bp_dir[bp] + a] - P.dirs[3 * P.bp_sddir[bp] + a];
    double s, co;
    sincos(P.kappa * xi * dc, &s, &co);
    P.E[P.bp_E_off[bp] + r] = cmk(co * L[j], s * L[j]);
    (void)ci;
}

// Coupling matrices S_b[nu,mu] = g_c(xi_{t,nu}, xi_{s,mu})
//   = exp(i kappa (r - <xi_t - xi_s, c>)) / (4 pi r).  CTA per block.
__global__ void k_S(PlanD P, int b0, const int* blist) {
    const int b = blist ? blist[blockIdx.x] : b0 + blockIdx.x;
    const int m = P.m, k = P.k;
    __shared__ GridD gt, gs;
    __shared__ double c[3];
    if (threadIdx.x == 0) {
        gt = P.grid[P.blk_t[b]];
        gs = P.grid[P.blk_s[b]];
        for (int a = 0; a < 3; ++a) c[a] = P.dirs[3 * P.blk_dir[b] + a];
    }
    __syncthreads();
    double2* S = P.S + (size_t)P.blk_slot[b] * k * k;
    const double inv4pi = 1.0 / (4.0 * M_PI);
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
        int nu = idx % k, mu = idx / k;
        double d0 = gt.nodes[0][nu % m] - gs.nodes[0][mu % m];
        double d1 = gt.nodes[1][(nu / m) % m] - gs.nodes[1][(mu / m) % m];
        double d2 = gt.nodes[2][nu / (m * m)] - gs.nodes[2][mu / (m * m)];
        double r = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
        double dcv = (d0 * c[0] + d1 * c[1]) + d2 * c[2];
        double s, co;
        sincos(P.kappa * (r - dcv), &s, &co);
        double f = inv4pi / r;
        S[idx] = cmk(co * f, s * f);
    }
}

void launch_quad(const PlanD& P, cudaStream_t s) {
    k_cheb<<<1, 32, 0, s>>>(P.m);
    int tot = P.n * 7;
    k_quad<<<(tot + 255) / 256, 256, 0, s>>>(P);
}
void launch_grid(const PlanD& P, cudaStream_t s) { k_grid<<<(P.nclusters + 127) / 128, 128, 0, s>>>(P); }
void launch_leafV(const PlanD& P, const int* bps, int nbps, int maxrows, cudaStream_t s) {
    if (!nbps) return;
    size_t sm = (size_t)maxrows * 7 * sizeof(double2) + (size_t)maxrows * 7 * 3 * P.m * sizeof(double);
    switch (P.m) {
        case 2: k_leafV<2><<<nbps, 128, sm, s>>>(P, bps); break;
        case 3: k_leafV<3><<<nbps, 128, sm, s>>>(P, bps); break;
        case 4: k_leafV<4><<<nbps, 128, sm, s>>>(P, bps); break;
        case 5: k_leafV<5><<<nbps, 128, sm, s>>>(P, bps); break;
        default: k_leafV<0><<<nbps, 128, sm, s>>>(P, bps); break;
    }
}
void launch_E(const PlanD& P, const int* bps, int nbps, cudaStream_t s) {
    if (!nbps) return;
    int tot = nbps * 6 * P.m * P.m;
    k_E<<<(tot + 255) / 256, 256, 0, s>>>(P, bps, nbps);
}
void launch_S(const PlanD& P, int b0, int nb, cudaStream_t s, const int* blist) {
    if (!nb) return;
    k_S<<<nb, 256, 0, s>>>(P, b0, blist);
}

// ============================================================== recompression (§3.2)

__device__ inline void zero_lower(double2* A, int lda, int rows, int cols) {
    for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
        int i = idx % rows, j = idx / rows;
        if (i > j) A[i + (size_t)j * lda] = cmk(0.0, 0.0);
    }
}


// Chunk append into the triangle: the blocked compact-WY form (chunks of <= 32 rows, option
// "qr_wy"; measured 1.5-2x slower on C4: its panels are factorised by one warp while the others
// wait, so the k-step critical path per chunk is not shorter) or the column-by-column one (default).
template <bool PK, int E>
__device__ __forceinline__ void qr_append(const PlanD& P, double2* R, int ldr, double2* B, int ldb, int nb, int k, WyPanel* wp) {
    __shared__ double s_tau[MMAX * MMAX * MMAX];
    __shared__ double2 s_u0[MMAX * MMAX * MMAX];
    __shared__ int s_step;
    if (E == 2 && P.qr_wy)
        cta_qr_append_wy<PK>(R, ldr, B, ldb, nb, k, wp);
    else if (P.qr_flag)
        cta_qr_append_flag<PK, 2 * E, 8>(R, ldr, B, ldb, nb, k, s_tau, s_u0, &s_step);  // (nb <= 16 E = 8 (2E))
    else
        cta_qr_append<PK, E>(R, ldr, B, ldb, nb, k);  // (8-lane groups for the 48-row chunks: measured neutral)
}

// Basis weights (Eq. 18; [BO10, Alg. 16] generalised to directions), one CTA per
// basis pair of one level: leaf with #t > k: R_tc = R of QR(V_tc); non-leaf:
// R_tc = R of QR([R_{t1c1} E_{t1c}; R_{t2c2} E_{t2c}]).  Rows are streamed in chunks of <= 32,
// transformed by the Kronecker-factored E and annihilated into a k x k triangle (structured
// Householder); if the stack has <= k rows it is the weight itself (P = I) and is written out.
template <bool PK, int E>
__global__ void k_basis(PlanD P, const int* bps, int ldr, int ldb) {
    extern __shared__ double2 sm[];
    __shared__ WyPanel wp;
    const int bp = bps[blockIdx.x];
    const int k = P.k, m = P.m;
    constexpr int CH = 16 * E;
    const bool leaf = P.bp_child0[bp] < 0;
    int src_bp[2] = {bp, -1};
    int nsrc = 1, total;
    if (leaf) {
        total = P.c_size[P.bp_t[bp]];
    } else {
        src_bp[0] = P.bp_child0[bp];
        src_bp[1] = P.bp_child1[bp];
        nsrc = 2;
        total = P.bp_R_rows[src_bp[0]] + P.bp_R_rows[src_bp[1]];
    }
    const bool qr = total > k;
    double2* R = sm;                                       // k x k triangle (QR case only)
    double2* B = R + (qr ? r_elems<PK>(k, ldr) : 0);       // CH x k chunk
    double2* Ef = B + (size_t)ldb * k;                     // 6 m^2
    if (!leaf) {
        const double2* Eg = P.E + P.bp_E_off[bp];
        for (int idx = threadIdx.x; idx < 6 * m * m; idx += blockDim.x) Ef[idx] = Eg[idx];
    }
    double2* Rout = P.R + P.bp_R_off[bp];
    const int out = P.bp_R_rows[bp];
    if (qr)
        for (int idx = threadIdx.x; idx < (int)r_elems<PK>(k, ldr); idx += blockDim.x) R[idx] = cmk(0.0, 0.0);
    // rows of the stack are gathered (and transformed by E) into chunks of CH rows across the
    // sources, each full chunk annihilated into R; without QR they go straight to R_out
    int fill = 0, cur = 0;
    for (int sidx = 0; sidx < nsrc; ++sidx) {
        const int r = leaf ? total : P.bp_R_rows[src_bp[sidx]];
        const double2* X = leaf ? (P.V + P.bp_V_off[bp]) : (P.R + P.bp_R_off[src_bp[sidx]]);
        for (int i0 = 0; i0 < r;) {
            const int nb = qr ? min(CH - fill, r - i0) : min(CH, r - i0);
            double2* dst = B + fill;
            __syncthreads();
            stage_rows(dst, ldb, X, r, i0, nb, k);
            cp_async_wait_all();
            __syncthreads();
            if (!leaf) kron_apply(dst, ldb, nb, m, Ef + sidx * 3 * m * m, false);
            i0 += nb;
            if (!qr) {
                for (int idx = threadIdx.x; idx < nb * k; idx += blockDim.x)
                    Rout[cur + idx % nb + (size_t)(idx / nb) * out] = B[idx % nb + (size_t)(idx / nb) * ldb];
                cur += nb;
                continue;
            }
            fill += nb;
            if (fill == CH) {
                qr_append<PK, E>(P, R, ldr, B, ldb, fill, k, &wp);
                fill = 0;
            }
        }
    }
    if (qr && fill > 0) qr_append<PK, E>(P, R, ldr, B, ldb, fill, k, &wp);
    if (qr) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
            const int i = idx % k, nu = idx / k;
            Rout[idx] = (i > nu) ? cmk(0.0, 0.0) : R[ridx<PK>(i, nu, ldr)];
        }
    }
}

// dynamic shared memory of the chunked-Householder kernels; packed R when the square does not fit
static size_t qr_chunk_smem(const PlanD& P, bool pk, int ldr, int ldb, int nE, bool with_qr = true) {
    const size_t relems = !with_qr ? 0 : pk ? (size_t)P.k * (P.k + 1) / 2 : (size_t)ldr * P.k;
    const size_t belems = (size_t)ldb * P.k;  // chunk (staging buffer without QR)
    return (relems + belems + (size_t)nE * P.m * P.m) * sizeof(double2);
}

void launch_basis(const PlanD& P, const int* bps, int nbps, int maxrows, cudaStream_t s) {
    if (!nbps) return;
    if (P.k <= 128 && (P.k > 64 ? P.qr_cq : P.qr_cq64) && P.cq_scr) return launch_basis_cq(P, bps, nbps, s);
    const bool any_qr = maxrows > P.k;
    const int ldr = odd_ld(P.k);
    if (P.k <= 64) {  // 64-row chunks, packed triangle
        const int ldb = odd_ld(64);
        k_basis<true, 4><<<nbps, 256, qr_chunk_smem(P, true, ldr, ldb, 6, any_qr), s>>>(P, bps, ldr, ldb);
    } else if (!P.qr_wy && qr_chunk_smem(P, true, ldr, odd_ld(48), 6, any_qr) <= (size_t)P.smem_optin) {
        // k = 125: 48-row chunks beside the packed triangle (224 KB): 6 instead of 8 appends of k
        // reflector steps for a 250-row stack
        const int ldb = odd_ld(48);
        k_basis<true, 3><<<nbps, 512, qr_chunk_smem(P, true, ldr, ldb, 6, any_qr), s>>>(P, bps, ldr, ldb);
    } else {
        const int ldb = odd_ld(32);
        k_basis<true, 2><<<nbps, 512, qr_chunk_smem(P, true, ldr, ldb, 6, any_qr), s>>>(P, bps, ldr, ldb);
    }
}

// Block weights (DESIGN reading R12): ||G_b||_F^2 = ||R_tc S_b R_sc^*||_F^2 (W = P R, Eq. 18);
// w_b = 1/||G_b||_F for the block-relative modes, 1 for FROB_CLUSTERREL.  CTA per block:
// U = R_tc S_b on the FP64 tensor cores (S read coalesced through the mirror block), in chunks
// of <= 64 rows of R_tc, then ||U R_sc^*||_F^2 with a fixed-order reduction.
template <int NT>  // 256 threads, 3 CTAs per SM (k <= 64) or 512 threads, one CTA per SM (k = 125)
__global__ void __launch_bounds__(NT, NT == 512 ? 1 : 3) k_block_weights(PlanD P, int b0, int mode, int ldu, int chunk, const int* mirror,
                                                         const int* blist) {
    extern __shared__ double2 sm[];
    __shared__ double red[32];
    const int b = blist ? blist[blockIdx.x] : b0 + blockIdx.x, k = P.k;
    const int bt = P.blk_bprow[b], bs = P.sym ? P.blk_bpcs[b] : P.blk_bpcol[b];  // sym: R_sc = conj R_{s,-c}
    const int rt = P.bp_R_rows[bt], rs = P.bp_R_rows[bs];
    const double2* Rt = P.R + P.bp_R_off[bt];
    const double2* Rs = P.R + P.bp_R_off[bs];
    const int mb = mirror[b];
    const double2* Sg = P.S + (size_t)P.blk_slot[mb >= 0 ? mb : b] * k * k;
    double2* U = sm;  // chunk x k
    double part = 0.0;
    for (int i0 = 0; i0 < rt; i0 += chunk) {
        const int nb = min(chunk, rt - i0);
        if (i0) __syncthreads();
        if (P.bw_variant && k > 64) {  // (4 k-steps of loads in flight; the norm GEMM register-blocked 8 x 32: C4 -5 %, C2 +27 %)
            chunk_gemm_S_dmma<true>(Rt, rt, i0, nb, Sg, false, mb < 0, 1.0, k, U, ldu);
            __syncthreads();
            part += P.sym ? dmma_abh4_norm<true>(U, ldu, nb, Rs, rs, rs, k) : dmma_abh4_norm<false>(U, ldu, nb, Rs, rs, rs, k);
            continue;
        }
        chunk_gemm_S_dmma(Rt, rt, i0, nb, Sg, false, mb < 0, 1.0, k, U, ldu);
        __syncthreads();
        // ||U R_sc^*||_F^2 on the FP64 tensor cores (sym: R_sc^* = (conj R_{s,-c})^* = R_{s,-c}^T)
        part += P.sym ? dmma_abh<false, true>(U, ldu, nb, Rs, rs, rs, k, nullptr, 0)
                      : dmma_abh<false, false>(U, ldu, nb, Rs, rs, rs, k, nullptr, 0);
    }
    part = warp_sum(part);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += red[w];
        P.normG2[b] = sum;
        P.omega[b] = (mode == 1) ? 1.0 : 1.0 / sqrt(sum);
    }
}

void launch_block_weights(const PlanD& P, int b0, int nb, int mode, const int* mirror, cudaStream_t s, const int* blist) {
    if (!nb) return;
    // (k = 125: one 512-thread CTA per SM with 64-row chunks halves the DRAM re-reads of S_b and R_sc
    // but measured 32 % slower on C4 than 3 CTAs per SM with 32-row chunks, which stays)
    const bool big = false;
    const int chunk = P.k <= 64 ? 64 : 32;
    const int ldu = odd_ld(chunk);
    size_t sm = (size_t)ldu * P.k * sizeof(double2);
    if (big)
        k_block_weights<512><<<nb, 512, sm, s>>>(P, b0, mode, ldu, chunk, mirror, blist);
    else
        k_block_weights<256><<<nb, 256, sm, s>>>(P, b0, mode, ldu, chunk, mirror, blist);
}

// Total weights, one CTA per pair of one level (top-down):
//   Z_tc = [w_b S_b R_sc^* (s in row(t,c)) | E_{tc+} Zhat_{t+c+}^* (c+ in sd^{-1}(c))],
//   Zhat_tc = R factor of the skinny QR of Z_tc^* (gamma = 0 at the root).
// The rows of Z_tc^* are produced in chunks of <= 32 rows and annihilated into the k x k
// triangle R (structured Householder); if Z_tc^* has <= k rows it is stored as is (P = I).
// Row pass: rows w_b R_sc S_b^*.  Column pass (adjoint): rows w_b R_tc S_b.
template <bool PK, int E>
__global__ void k_total_weights(PlanD P, PassD X, bool row, int p0, const int* mirror, int ldr, int ldb) {
    extern __shared__ double2 sm[];
    __shared__ WyPanel wp;
    const int p = p0 + blockIdx.x;
    const int k = P.k, m = P.m;
    constexpr int CH = 16 * E;
    const int zr = X.Z_rows[p];
    double2* Zg = X.Z + X.Z_off[p];
    // total rows of Z^*
    int total = 0;
    for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
        const int b = X.blk[ib];
        total += P.bp_R_rows[row ? P.blk_bpcol[b] : P.blk_bprow[b]];
    }
    for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) total += X.Z_rows[X.par[ip]];
    const bool qr = total > k;
    double2* R = sm;                                  // k x k triangle (QR case)
    double2* B = R + (qr ? r_elems<PK>(k, ldr) : 0);  // CH x k chunk (ld ldb)
    double2* Ef = B + (size_t)ldb * k;                // 3 m^2
    if (qr)
        for (int idx = threadIdx.x; idx < (int)r_elems<PK>(k, ldr); idx += blockDim.x) R[idx] = cmk(0.0, 0.0);
    // the rows of Z^* are produced into chunks of CH rows across the sources, each full chunk
    // annihilated into R; without QR (<= k rows, zr == total) they are the weight itself
    // (P = I) and go straight to the global slab
    int fill = 0, cur = 0;
    auto next = [&](int nb) {
        if (!qr) {
            cur += nb;
            return;
        }
        fill += nb;
        if (fill == CH) {
            qr_append<PK, E>(P, R, ldr, B, ldb, fill, k, &wp);
            fill = 0;
        }
    };
    for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
        const int b = X.blk[ib];
        const bool cj = row && P.sym;  // R_sc = conj R_{s,-c} (adjoint symmetry)
        const int obp = row ? (cj ? P.blk_bpcs[b] : P.blk_bpcol[b]) : P.blk_bprow[b];
        const int r = P.bp_R_rows[obp];
        const double2* Ro = P.R + P.bp_R_off[obp];
        const double w = P.omega[b];
        const int mb = row ? b : mirror[b];
        const double2* Sg = P.S + (size_t)P.blk_slot[mb >= 0 ? mb : b] * k * k;
        const bool strided = !row && mb < 0;
        for (int i0 = 0; i0 < r;) {
            const int nb = qr ? min(CH - fill, r - i0) : min(CH, r - i0);
            double2* dst = qr ? B + fill : Zg + cur;
            const int ldd = qr ? ldb : zr;
            __syncthreads();
            chunk_gemm_S_dmma(Ro, r, i0, nb, Sg, row, strided, w, k, dst, ldd, cj);  // FP64 tensor cores
            i0 += nb;
            next(nb);
        }
    }
    for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) {
        const int pp = X.par[ip];
        const int ci = X.par_child[ip];
        const int r = X.Z_rows[pp];
        const double2* Zp = X.Z + X.Z_off[pp];
        const double2* Eg = P.E + P.bp_E_off[X.bp[pp]] + ci * 3 * m * m;
        __syncthreads();
        for (int idx = threadIdx.x; idx < 3 * m * m; idx += blockDim.x) Ef[idx] = Eg[idx];
        for (int i0 = 0; i0 < r;) {
            const int nb = qr ? min(CH - fill, r - i0) : min(CH, r - i0);
            double2* dst = B + (qr ? fill : 0);
            __syncthreads();
            for (int idx = threadIdx.x; idx < nb * k; idx += blockDim.x)
                dst[idx % nb + (size_t)(idx / nb) * ldb] = Zp[i0 + idx % nb + (size_t)(idx / nb) * r];
            __syncthreads();
            kron_apply(dst, ldb, nb, m, Ef, true);  // Zhat_{t+c+} E_{tc+}^*
            if (!qr)
                for (int idx = threadIdx.x; idx < nb * k; idx += blockDim.x)
                    Zg[cur + idx % nb + (size_t)(idx / nb) * zr] = B[idx % nb + (size_t)(idx / nb) * ldb];
            i0 += nb;
            next(nb);
        }
    }
    if (qr && fill > 0) qr_append<PK, E>(P, R, ldr, B, ldb, fill, k, &wp);
    if (qr) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < zr * k; idx += blockDim.x) {
            const int i = idx % zr, nu = idx / zr;
            Zg[idx] = (i > nu) ? cmk(0.0, 0.0) : R[ridx<PK>(i, nu, ldr)];
        }
    }
}

void launch_total_weights(const PlanD& P, bool row, int p0, int np, const int* mirror, cudaStream_t s, bool leaf_level) {
    if (!np) return;
    const int v = leaf_level && P.qr_cq_tw_leaf ? P.qr_cq_tw_leaf : P.qr_cq_tw;
    if (P.k <= 128 && (P.k > 64 ? v : P.qr_cq64_tw) && P.cq_scr)
        return launch_total_weights_cq(P, row, p0, np, mirror, s, P.k > 64 ? v : P.qr_cq64_tw);
    const int ldr = odd_ld(P.k);
    const PassD& X = row ? P.row : P.col;
    if (P.k <= 64) {  // 64-row chunks, packed triangle
        const int ldb = odd_ld(64);
        k_total_weights<true, 4><<<np, 256, qr_chunk_smem(P, true, ldr, ldb, 3), s>>>(P, X, row, p0, mirror, ldr, ldb);
    } else if (!P.qr_wy && qr_chunk_smem(P, true, ldr, odd_ld(48), 3) <= (size_t)P.smem_optin) {
        const int ldb = odd_ld(48);  // 48-row chunks (see launch_basis)
        k_total_weights<true, 3><<<np, 512, qr_chunk_smem(P, true, ldr, ldb, 3), s>>>(P, X, row, p0, mirror, ldr, ldb);
    } else {
        const int ldb = odd_ld(32);
        k_total_weights<true, 2><<<np, 512, qr_chunk_smem(P, true, ldr, ldb, 3), s>>>(P, X, row, p0, mirror, ldr, ldb);
    }
}

// Truncation, one CTA per pair of one level (bottom-up):
//   leaf:     M = V_tc Zhat_tc^*;  non-leaf: Vhat = [C_{t1c1} E_{t1c}; C_{t2c2} E_{t2c}], M = Vhat Zhat^*
//   left singular vectors/values of M: QR with column pivoting of M^* = Zhat Vt^* (M^* Pi = Q R,
//   so M = Pi R^* Q^*), then one-sided Jacobi on the graded columns of R^* (QR-preconditioned
//   Jacobi: high relative accuracy, few sweeps; no Gram matrix is formed, DESIGN reading Q13);
//   rank k_tc by the rule of `mode`, Q = first k_tc vectors (leaf: Q_tc, non-leaf:
//   Qhat = [F_{t1c}; F_{t2c}]), C_tc = Q^* V_tc or Qhat^* Vhat (Eq. 19).
// Truncation prologue: M^* = Zhat Vt^* (leaf Vt = V_tc; above the leaves
// Vt = Vhat = [C_{t1c1} E_{t1c}; C_{t2c2} E_{t2c}] built here) and its pivoted QR, stopped at the
// numerical rank.  On return the rows 0..ncol-1 of B hold R (zero below the pivoted diagonal), piv
// the pivot order; returns ncol, or -1 if the pair is empty (rank 0 already recorded).
template <bool LEAF>
__device__ inline int truncate_prologue(const PlanD& P, const PassD& X, int p, double2* sm, int ldv, int ldb, bool append,
                                        double2*& B, int& ldB, double*& nrm, int*& piv, int*& ord, int& rowsM,
                                        const double2*& Vt, int& ldvt, int& s_piv, double2* sh) {
    const int k = P.k, m = P.m;
    const int bp = X.bp[p];
    constexpr bool leaf = LEAF;  // one instance per kind of level (all pairs of a level are alike)
    const int zr = X.Z_rows[p];
    const double2* Z = X.Z + X.Z_off[p];
    double2* Vs = sm;                                  // non-leaf Vhat (rowsM x k, ld ldv)
    B = Vs + (leaf ? 0 : (size_t)ldv * k);             // M^* (zr x rowsM, ld ldb)
    ldB = ldb;
    double2* chunk = nullptr;
    if (leaf && append) {  // tall M^*: its R factor (rowsM x rowsM, ld ldv) from streamed 32-row chunks
        ldB = ldv;
        chunk = B + (size_t)ldv * ldv;                 // 32 x rowsM, ld 33
    }
    double2* Ef = (leaf && append) ? chunk + (size_t)33 * ldv : B + (size_t)ldb * ldv;  // 6 m^2 (non-leaf)
    nrm = reinterpret_cast<double*>(Ef + (leaf ? 0 : 6 * m * m));  // ldv
    piv = reinterpret_cast<int*>(nrm + ldv);           // ldv
    ord = piv + ldv;                                   // ldv
    if constexpr (leaf) {
        rowsM = P.c_size[P.bp_t[bp]];
        Vt = P.V + P.bp_V_off[bp];
        ldvt = rowsM;
    } else {
        const int c0 = X.child0[p], c1 = X.child1[p];
        const int k1 = X.rank[c0], k2 = X.rank[c1];
        const int l0 = X.kb[c0], l1 = X.kb[c1];
        const double2* C0 = X.C + X.C_off[c0];
        const double2* C1 = X.C + X.C_off[c1];
        for (int idx = threadIdx.x; idx < k1 * k; idx += blockDim.x) Vs[idx % k1 + (size_t)(idx / k1) * ldv] = C0[idx % k1 + (size_t)(idx / k1) * l0];
        for (int idx = threadIdx.x; idx < k2 * k; idx += blockDim.x) Vs[k1 + idx % k2 + (size_t)(idx / k2) * ldv] = C1[idx % k2 + (size_t)(idx / k2) * l1];
        const double2* Eg = P.E + P.bp_E_off[bp];
        for (int idx = threadIdx.x; idx < 6 * m * m; idx += blockDim.x) Ef[idx] = Eg[idx];
        __syncthreads();
        kron_apply(Vs, ldv, k1, m, Ef, false);
        kron_apply(Vs + k1, ldv, k2, m, Ef + 3 * m * m, false);
        rowsM = k1 + k2;
        Vt = Vs;
        ldvt = ldv;
    }
    if (rowsM == 0 || zr == 0) {
        if (threadIdx.x == 0) {
            X.rank[p] = 0;
            X.nsig[p] = 0;
            X.disc[p] = 0.0;
            X.sweeps[p] = 0;
        }
        return -1;
    }
    int Mq = zr;  // rows of the matrix the pivoted QR runs on
    if (leaf && append) {
        // M^* has more rows than columns: annihilate its row chunks (M^* chunk = Zhat chunk V^* on
        // the FP64 tensor cores) into the triangle R0 (structured Householder); the pivoted QR of R0
        // has the pivots, the R factor and the trailing norms of the pivoted QR of M^* (same
        // column norms), in rowsM instead of zr rows of shared memory
        for (int idx = threadIdx.x; idx < ldv * rowsM; idx += blockDim.x) B[idx] = cmk(0.0, 0.0);
        for (int r0 = 0; r0 < zr; r0 += 32) {
            const int nb = min(32, zr - r0);
            __syncthreads();
            dmma_abh<true>(Z + r0, zr, nb, Vt, ldvt, rowsM, k, chunk, 33);
            cta_qr_append<false, 2>(B, ldv, chunk, 33, nb, rowsM);
        }
        Mq = min(zr, rowsM);
    } else {
        // B = M^* = Zhat Vt^*  (zr x rowsM) on the FP64 tensor cores
        dmma_abh4(Z, zr, zr, Vt, ldvt, rowsM, k, B, ldb);  // (register-blocked: 8 x 32 per warp task)
    }
    // pivoted QR, stopped once the trailing block has ||R22||_F <= 1e-13 max_j ||M^*(:, j)|| <=
    // 1e-13 sigma_1: every singular value dropped with it is below the parity tolerance
    // 1e-12 sigma_1 (DESIGN §6 G3), and its share of any tail sum is < 1e-26 sigma_1^2
    const int ncol = qrcp_auto(B, ldB, Mq, rowsM, piv, nrm, sh, &s_piv, 1e-26);
    zero_lower(B, ldB, ncol, rowsM);  // drop the Householder vectors below the diagonal of R
    __syncthreads();
    return ncol;
}

// Truncation epilogue: singular values sigma_a = ||row ord[a] of R|| (rows of R
// mutually orthogonal after the Jacobi), rank by the rule of `mode`, Q / Qhat = [F1; F2] and
// C = Q^* Vt from the rows of R, the pivot order piv and Vt (rowsM x k, ld ldvt).
__device__ inline void truncate_epilogue(const PassD& X, int p, int k, const double2* B, int ldb, int ncol, int rowsM,
                                         const int* piv, const double* nrm, int* ord, const double2* Vt, int ldvt,
                                         int ldq, double eps, int mode, int& s_rank) {
    double2* Qg = X.Q + X.Q_off[p];
    double2* Cg = X.C + X.C_off[p];
    const int kb = X.kb[p];
    // singular values = norms of the rows of R; order by decreasing value (ties: lower index)
    // (keys with NaN mapped to -1 so that ord is always a permutation; such a pair is flagged below)
    for (int j = threadIdx.x; j < ncol; j += blockDim.x) {
        int pos = 0;
        const double sj = nrm[j] == nrm[j] ? nrm[j] : -1.0;
        for (int i = 0; i < ncol; ++i) {
            const double si = nrm[i] == nrm[i] ? nrm[i] : -1.0;
            pos += (si > sj) || (si == sj && i < j);
        }
        ord[pos] = j;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // rank rule (DESIGN reading Q12), tail sums from the smallest value
        double* so = X.sigma + X.sig_off[p];
        for (int a = 0; a < ncol; ++a) so[a] = sqrt(nrm[ord[a]]);
        double acc = 0.0, thr = 0.0, tot = 0.0;
        for (int a = ncol - 1; a >= 0; --a) tot += so[a] * so[a];
        thr = (mode == 0 || mode == 2) ? eps * eps : eps * eps * tot;
        int kk = ncol;
        double disc = 0.0;
        if (mode == 2) {
            kk = 0;
            while (kk < ncol && so[kk] > eps) ++kk;
            for (int a = ncol - 1; a >= kk; --a) disc += so[a] * so[a];
        } else {
            // smallest k with tail(k) <= thr: walk up from the smallest value
            kk = ncol;
            for (int a = ncol - 1; a >= 0; --a) {
                acc += so[a] * so[a];
                if (acc <= thr) { kk = a; disc = acc; } else break;
            }
        }
        if (kk > kb) kk = kb;
        bool finite = true;
        for (int a = 0; a < ncol; ++a) finite = finite && isfinite(so[a]);
        if (!finite) kk = 0;  // non-finite input: no output, rank -1 reported to the host
        s_rank = kk;
        X.rank[p] = finite ? kk : -1;
        X.nsig[p] = ncol;
        X.disc[p] = disc;
    }
    __syncthreads();
    const int kk = s_rank;
    // Q[piv[j], a] = conj(R[ord[a], j]) / s ; C[a, nu] = sum_j R[ord[a], j] / s * Vt[piv[j], nu]
    for (int idx = threadIdx.x; idx < rowsM * kk; idx += blockDim.x) {
        const int j = idx % rowsM, a = idx / rowsM;
        const int r = ord[a];
        const double s = sqrt(nrm[r]);
        const double2 v = B[r + (size_t)j * ldb];
        Qg[piv[j] + (size_t)a * ldq] = s > 0.0 ? cmk(v.x / s, -v.y / s) : cmk(0.0, 0.0);
    }
    for (int idx = threadIdx.x; idx < kk * k; idx += blockDim.x) {
        const int a = idx % kk, nu = idx / kk;
        const int r = ord[a];
        const double s = sqrt(nrm[r]);
        double2 acc = cmk(0.0, 0.0);
        for (int j = 0; j < rowsM; ++j) cfma(acc, B[r + (size_t)j * ldb], Vt[piv[j] + (size_t)nu * ldvt]);
        Cg[a + (size_t)nu * kb] = s > 0.0 ? cscale(acc, 1.0 / s) : cmk(0.0, 0.0);
    }
}

// Truncation kernels: one CTA per pair with the working set in shared memory, or, when it
// exceeds the opt-in shared memory (large k / ranks), a persistent grid whose CTAs keep their
// working set in a private global (L2-resident) workspace slab.

template <bool LEAF>
__device__ inline void truncate_pair(const PlanD& P, const PassD& X, int p, double2* sm, int ldv, int ldb, bool append,
                                     double eps, int mode, int& flag, int& s_piv, int& s_rank, double2* sh) {
    double2* B;
    double* nrm;
    int *piv, *ord;
    int rowsM, ldvt, ldB;
    const double2* Vt;
    const int ncol = truncate_prologue<LEAF>(P, X, p, sm, ldv, ldb, append, B, ldB, nrm, piv, ord, rowsM, Vt, ldvt, s_piv, sh);
    if (ncol < 0) return;
    const int nsw = jacobi_rows_auto(B, ldB, ncol, rowsM, nrm, &flag);
    if (threadIdx.x == 0) X.sweeps[p] = nsw;
    truncate_epilogue(X, p, P.k, B, ldB, ncol, rowsM, piv, nrm, ord, Vt, ldvt, LEAF ? rowsM : X.rowsb[p], eps, mode, s_rank);
}

template <bool LEAF>
__global__ void __launch_bounds__(512, 1)
    k_truncate(PlanD P, PassD X, int p0, int ldv, int ldb, bool append, double eps, int mode, const int* plist) {
    extern __shared__ double2 smd[];
    __shared__ int flag, s_piv, s_rank;
    __shared__ double2 sh[2];
    const int p = plist ? plist[blockIdx.x] : p0 + blockIdx.x;
    truncate_pair<LEAF>(P, X, p, smd, ldv, ldb, append, eps, mode, flag, s_piv, s_rank, sh);
}

template <bool LEAF>
__global__ void __launch_bounds__(128, 3)
    k_truncate_ws(PlanD P, PassD X, int p0, int np, int ldv, int ldb, bool append, double eps, int mode, double2* ws,
                  size_t ws_stride, const int* plist) {
    __shared__ int flag, s_piv, s_rank;
    __shared__ double2 sh[2];
    double2* base = ws + (size_t)blockIdx.x * ws_stride;
    for (int i = blockIdx.x; i < np; i += gridDim.x) {
        truncate_pair<LEAF>(P, X, plist ? plist[i] : p0 + i, base, ldv, ldb, append, eps, mode, flag, s_piv, s_rank, sh);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ leaf truncation, split path
// For leaf levels with #t <= 32 (C2, C3): (1) k_trunc_qr: M^* and its pivoted QR per CTA as above,
// R written to a scratch slab (32 x 32, row r = vector r, element-major) with the pivot order;
// (2) k_jacobi_w32: the one-sided Jacobi on the rows of R with one WARP per pair and the matrix in
// registers (lane = element, 32 slots = vectors): same rotation formulas, tolerance and norm
// updates as jacobi_rows_t, round-robin by the circle method (pairs = slots (2i, 2i+1), a fixed
// slot permutation after every round), no shared-memory traffic and no block barriers;
// (3) k_trunc_epi: ordering, rank rule, Q and C from the scratch (truncate_epilogue).

// circle-method tournament on 32 slots: slot <-> position, one step of the rotation
__host__ __device__ constexpr int jw_pos(int s) { return (s & 1) ? 31 - (s >> 1) : (s >> 1); }
__host__ __device__ constexpr int jw_slot(int pos) { return pos < 16 ? 2 * pos : 2 * (31 - pos) + 1; }
__host__ __device__ constexpr int jw_next(int pos) { return pos == 0 ? 0 : (pos == 31 ? 1 : pos + 1); }
__host__ __device__ constexpr int jw_prev(int pos) { return pos == 0 ? 0 : (pos == 1 ? 31 : pos - 1); }

__global__ void __launch_bounds__(128, 6) k_trunc_qr(PlanD P, PassD X, int p0, int ldv, int ldb, bool append, double2* sR,
                                                    int* sPiv, int* sMeta) {
    extern __shared__ double2 smd[];
    __shared__ int s_piv;
    __shared__ double2 sh[2];
    const int i = blockIdx.x, p = p0 + i;
    double2* B;
    double* nrm;
    int *piv, *ord;
    int rowsM, ldvt, ldB;
    const double2* Vt;
    const int ncol = truncate_prologue<true>(P, X, p, smd, ldv, ldb, append, B, ldB, nrm, piv, ord, rowsM, Vt, ldvt, s_piv, sh);
    if (threadIdx.x == 0) {
        sMeta[2 * i] = ncol;  // -1: empty pair, already recorded
        sMeta[2 * i + 1] = rowsM;
    }
    if (ncol < 0) return;
    double2* R = sR + (size_t)i * 1024;
    for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) {
        const int r = idx >> 5, j = idx & 31;
        R[idx] = (r < ncol && j < rowsM) ? B[r + (size_t)j * ldB] : cmk(0.0, 0.0);
    }
    for (int j = threadIdx.x; j < 32; j += blockDim.x) sPiv[i * 32 + j] = j < rowsM ? piv[j] : 0;
}

// (1') leaf total weights fused into (1) (k <= 64): the rows of the stack whose R factor is Zhat_tc
// (omega_b R_sc S_b^*, Zhat_{t+c+} E_{tc+}^*, as in k_total_weights) are streamed in
// chunks of 32, each chunk multiplied by V_tc^* on the FP64 tensor cores and annihilated into a
// #t x #t triangle R0.  Zhat^* Zhat = Stack^* Stack, so R0^* R0 = V Zhat^* Zhat V^* = M M^*: R0 has
// the column norms, pivots and R factor of the pivoted QR of M^* = Zhat V^* (the append mode
// above with Zhat's own QR folded in), and the leaf Zhat is never formed or stored.
__global__ void __launch_bounds__(256, 3) k_trunc_zqr(PlanD P, PassD X, bool row, int p0, const int* mirror,
                                                    int direct_max, double2* sR, int* sPiv, int* sMeta) {
    extern __shared__ double2 smd[];
    __shared__ int s_piv;
    __shared__ double2 sh[2];
    constexpr int CH = 32, LD = 33;
    const int i = blockIdx.x, p = p0 + i;
    const int k = P.k, m = P.m;
    const int bp = X.bp[p];
    const int rowsM = P.c_size[P.bp_t[bp]];
    const double2* Vt = P.V + P.bp_V_off[bp];  // rowsM x k, ld rowsM
    const int zr = X.Z_rows[p];
    if (rowsM == 0 || zr == 0) {
        if (threadIdx.x == 0) {
            X.rank[p] = 0;
            X.nsig[p] = 0;
            X.disc[p] = 0.0;
            X.sweeps[p] = 0;
            sMeta[2 * i] = -1;
            sMeta[2 * i + 1] = rowsM;
        }
        return;
    }
    // stack height; with <= direct_max (<= 64) rows M^* = Stack V^* itself is formed (Zhat = Stack, P = I) and the
    // pivoted QR runs on it directly, as k_trunc_qr does on Zhat V^*
    int total = 0;
    for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
        const int b = X.blk[ib];
        total += P.bp_R_rows[row ? P.blk_bpcol[b] : P.blk_bprow[b]];
    }
    for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) total += X.Z_rows[X.par[ip]];
    const bool direct = total <= direct_max;
    double2* B = smd;                          // CH x k stack chunk, ld LD
    double2* Pm = B + (size_t)LD * k;          // CH x rowsM product chunk, ld LD
    double2* R0 = Pm + (size_t)LD * 32;        // rowsM x rowsM triangle, ld LD
    double2* Md = Pm;                          // direct: M^* (total x rowsM, ld 65) over Pm and R0
    constexpr int LDM = 65;
    double2* Ef = R0 + (size_t)LD * 32;        // 3 m^2
    double* nrm = reinterpret_cast<double*>(Ef + 3 * m * m);  // 2 x 32
    int* piv = reinterpret_cast<int*>(nrm + 64);              // 32
    if (!direct)
        for (int idx = threadIdx.x; idx < LD * 32; idx += blockDim.x) R0[idx] = cmk(0.0, 0.0);
    int fill = 0, done = 0;
    auto flush = [&]() {
        __syncthreads();
        if (direct) {
            dmma_abh<true>(B, LD, fill, Vt, rowsM, rowsM, k, Md + done, LDM);  // rows of Stack V^*
        } else {
            dmma_abh<true>(B, LD, fill, Vt, rowsM, rowsM, k, Pm, LD);  // chunk V^*
            cta_qr_append<false, 2>(R0, LD, Pm, LD, fill, rowsM);
        }
        done += fill;
        fill = 0;
    };
    for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
        const int b = X.blk[ib];
        const bool cj = row && P.sym;  // R_sc = conj R_{s,-c} (adjoint symmetry)
        const int obp = row ? (cj ? P.blk_bpcs[b] : P.blk_bpcol[b]) : P.blk_bprow[b];
        const int r = P.bp_R_rows[obp];
        const double2* Ro = P.R + P.bp_R_off[obp];
        const double w = P.omega[b];
        const int mb = row ? b : mirror[b];
        const double2* Sg = P.S + (size_t)P.blk_slot[mb >= 0 ? mb : b] * k * k;
        const bool strided = !row && mb < 0;
        for (int i0 = 0; i0 < r;) {
            const int nb = min(CH - fill, r - i0);
            __syncthreads();
            chunk_gemm_S_dmma(Ro, r, i0, nb, Sg, row, strided, w, k, B + fill, LD, cj);
            i0 += nb;
            fill += nb;
            if (fill == CH) flush();
        }
    }
    for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) {
        const int pp = X.par[ip];
        const int ci = X.par_child[ip];
        const int r = X.Z_rows[pp];
        const double2* Zp = X.Z + X.Z_off[pp];
        const double2* Eg = P.E + P.bp_E_off[X.bp[pp]] + ci * 3 * m * m;
        __syncthreads();
        for (int idx = threadIdx.x; idx < 3 * m * m; idx += blockDim.x) Ef[idx] = Eg[idx];
        for (int i0 = 0; i0 < r;) {
            const int nb = min(CH - fill, r - i0);
            double2* dst = B + fill;
            __syncthreads();
            for (int idx = threadIdx.x; idx < nb * k; idx += blockDim.x)
                dst[idx % nb + (size_t)(idx / nb) * LD] = Zp[i0 + idx % nb + (size_t)(idx / nb) * r];
            __syncthreads();
            kron_apply(dst, LD, nb, m, Ef, true);  // Zhat_{t+c+} E_{tc+}^*
            i0 += nb;
            fill += nb;
            if (fill == CH) flush();
        }
    }
    if (fill > 0) flush();
    double2* Rf = direct ? Md : R0;
    const int ldf = direct ? LDM : LD;
    const int ncol = qrcp_auto(Rf, ldf, direct ? total : min(total, rowsM), rowsM, piv, nrm, sh, &s_piv, 1e-26);
    zero_lower(Rf, ldf, ncol, rowsM);
    __syncthreads();
    if (threadIdx.x == 0) {
        sMeta[2 * i] = ncol;
        sMeta[2 * i + 1] = rowsM;
    }
    double2* R = sR + (size_t)i * 1024;
    for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) {
        const int r = idx >> 5, j = idx & 31;
        R[idx] = (r < ncol && j < rowsM) ? Rf[r + (size_t)j * ldf] : cmk(0.0, 0.0);
    }
    for (int j = threadIdx.x; j < 32; j += blockDim.x) sPiv[i * 32 + j] = j < rowsM ? piv[j] : 0;
}

// Leaf truncation with the leaf total weights folded in, for leaves of <= 64 triangles and any k
// (C4/C5: k = 125, #t = 64 / 48): the rows of the stack whose R factor is Zhat_tc (P:1003-1036:
// w_b R_sc S_b^*, Zhat_{t+c+} E_{tc+}^*) are streamed in chunks of 32, each chunk multiplied by
// V_tc^* on the FP64 tensor cores and appended into a #t x #t triangle R0 (R0^* R0 = V Zhat^* Zhat V^*
// = M M^*); then, in the same CTA, the pivoted QR of R0, the one-sided Jacobi and the epilogue of the
// unfused truncation.  Zhat_tc (k columns) is never formed: the appends run on #t instead of k
// columns, and the leaf level needs no Zhat storage.
__global__ void __launch_bounds__(512, 1) k_truncate_fused(PlanD P, PassD X, bool row, int p0, const int* mirror, int ldv,
                                                          double eps, int mode) {
    extern __shared__ double2 smd[];
    __shared__ int flag, s_piv, s_rank;
    __shared__ double2 sh[2];
    constexpr int CH = 32, LD = 33;
    const int p = p0 + blockIdx.x;
    const int k = P.k, m = P.m;
    const int bp = X.bp[p];
    const int rowsM = P.c_size[P.bp_t[bp]];
    const double2* Vt = P.V + P.bp_V_off[bp];  // rowsM x k, ld rowsM
    const int zr = X.Z_rows[p];
    if (rowsM == 0 || zr == 0) {
        if (threadIdx.x == 0) {
            X.rank[p] = 0;
            X.nsig[p] = 0;
            X.disc[p] = 0.0;
            X.sweeps[p] = 0;
        }
        return;
    }
    double2* B = smd;                         // CH x k stack chunk, ld LD
    double2* Pm = B + (size_t)LD * k;         // CH x rowsM product chunk, ld LD
    double2* R0 = Pm + (size_t)LD * ldv;      // rowsM x rowsM triangle, ld ldv
    double2* Ef = R0 + (size_t)ldv * ldv;     // 3 m^2
    double* nrm = reinterpret_cast<double*>(Ef + 3 * m * m);  // ldv
    int* piv = reinterpret_cast<int*>(nrm + ldv);              // ldv
    int* ord = piv + ldv;                                      // ldv
    for (int idx = threadIdx.x; idx < ldv * rowsM; idx += blockDim.x) R0[idx] = cmk(0.0, 0.0);
    int fill = 0, total = 0;
    auto flush = [&]() {
        __syncthreads();
        dmma_abh<true>(B, LD, fill, Vt, rowsM, rowsM, k, Pm, LD);  // chunk V^*
        cta_qr_append<false, 2>(R0, ldv, Pm, LD, fill, rowsM);
        total += fill;
        fill = 0;
    };
    for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
        const int b = X.blk[ib];
        const bool cj = row && P.sym;  // R_sc = conj R_{s,-c} (adjoint symmetry)
        const int obp = row ? (cj ? P.blk_bpcs[b] : P.blk_bpcol[b]) : P.blk_bprow[b];
        const int r = P.bp_R_rows[obp];
        const double2* Ro = P.R + P.bp_R_off[obp];
        const double w = P.omega[b];
        const int mb = row ? b : mirror[b];
        const double2* Sg = P.S + (size_t)P.blk_slot[mb >= 0 ? mb : b] * k * k;
        const bool strided = !row && mb < 0;
        for (int i0 = 0; i0 < r;) {
            const int nb = min(CH - fill, r - i0);
            __syncthreads();
            chunk_gemm_S_dmma(Ro, r, i0, nb, Sg, row, strided, w, k, B + fill, LD, cj);
            i0 += nb;
            fill += nb;
            if (fill == CH) flush();
        }
    }
    for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) {
        const int pp = X.par[ip];
        const int ci = X.par_child[ip];
        const int r = X.Z_rows[pp];
        const double2* Zp = X.Z + X.Z_off[pp];
        const double2* Eg = P.E + P.bp_E_off[X.bp[pp]] + ci * 3 * m * m;
        __syncthreads();
        for (int idx = threadIdx.x; idx < 3 * m * m; idx += blockDim.x) Ef[idx] = Eg[idx];
        for (int i0 = 0; i0 < r;) {
            const int nb = min(CH - fill, r - i0);
            double2* dst = B + fill;
            __syncthreads();
            for (int idx = threadIdx.x; idx < nb * k; idx += blockDim.x)
                dst[idx % nb + (size_t)(idx / nb) * LD] = Zp[i0 + idx % nb + (size_t)(idx / nb) * r];
            __syncthreads();
            kron_apply(dst, LD, nb, m, Ef, true);  // Zhat_{t+c+} E_{tc+}^*
            i0 += nb;
            fill += nb;
            if (fill == CH) flush();
        }
    }
    if (fill > 0) flush();
    // pivoted QR of R0 = that of M^* = Zhat V^* (same column norms), rank stop as the unfused path
    const int ncol = qrcp_auto(R0, ldv, min(total, rowsM), rowsM, piv, nrm, sh, &s_piv, 1e-26);
    zero_lower(R0, ldv, ncol, rowsM);
    __syncthreads();
    const int nsw = jacobi_rows_auto(R0, ldv, ncol, rowsM, nrm, &flag);
    if (threadIdx.x == 0) X.sweeps[p] = nsw;
    truncate_epilogue(X, p, k, R0, ldv, ncol, rowsM, piv, nrm, ord, Vt, rowsM, rowsM, eps, mode, s_rank);
}

size_t trunc_fused_smem(const PlanD& P, int maxrows) {
    const int ldv = odd_ld(max(maxrows, 1));
    return ((size_t)33 * P.k + (size_t)33 * ldv + (size_t)ldv * ldv + 3 * P.m * P.m) * sizeof(double2) +
           (size_t)ldv * (sizeof(double) + 2 * sizeof(int));
}

void launch_truncate_fused(const PlanD& P, bool row, int p0, int np, int maxrows, double eps, int mode, const int* mirror,
                           cudaStream_t s) {
    if (!np) return;
    const PassD& X = row ? P.row : P.col;
    k_truncate_fused<<<np, 512, trunc_fused_smem(P, maxrows), s>>>(P, X, row, p0, mirror, odd_ld(max(maxrows, 1)), eps, mode);
}

size_t trunc_zqr_smem(const PlanD& P) {
    return ((size_t)33 * P.k + 2 * 33 * 32 + 3 * P.m * P.m) * sizeof(double2) + 64 * sizeof(double) + 32 * sizeof(int);
}

__global__ void __launch_bounds__(128, 3) k_jacobi_w32(PassD X, int p0, int np, double2* sR, double* sN, const int* sMeta) {
    __shared__ double4 prm[4][16];
    __shared__ double tsum[4][32 * 33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i = blockIdx.x * 4 + w;
    if (i >= np) return;  // whole warp
    const int ncol = sMeta[2 * i], len = sMeta[2 * i + 1];
    if (ncol < 0) return;
    constexpr unsigned FULL = 0xffffffffu;
    double2 x[32];  // lane = element c of the row vectors of R: x[r] = R[r, c]
    double2* R = sR + (size_t)i * 1024;
#pragma unroll
    for (int r = 0; r < 32; ++r) x[r] = R[r * 32 + lane];
    const double tol = fmax((double)len, 1.0) * 2.220446049250313e-16;
    const double tol2 = tol * tol;
    double* tbuf = tsum[w];
    auto norms = [&]() {
#pragma unroll
        for (int r = 0; r < 32; ++r) tbuf[lane * 33 + r] = cabs2(x[r]);
        __syncwarp();
        double v = 0.0;
#pragma unroll
        for (int r = 0; r < 32; ++r) v += tbuf[r * 33 + lane];
        __syncwarp();
        return v;
    };
    double nr = 0.0;
    int sweep = 0;
#pragma unroll 1
    for (; sweep < 60 && ncol > 1; ++sweep) {
        nr = norms();
        bool any = false;
        // absolute floor of the convergence test (DESIGN reading N3), as jacobi_rows_t
        double mx = nr;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        const double floor2 = 1e-56 * mx * mx;
#pragma unroll 1
        for (int round = 0; round < 31; ++round) {
            // a conj(b) of the slot pairs (2q, 2q+1), this lane's element; pairs 0-7 and 8-15 are
            // reduced separately (16 values each) so that lane 2q / 2q+1 ends with Re / Im of g_q
            double mine;
            {  // a conj(b) partials straight into the transpose buffer, then column sums
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const double2 a = x[2 * q], b = x[2 * q + 1];
                    tbuf[lane * 33 + 2 * q] = fma(a.x, b.x, a.y * b.y);
                    tbuf[lane * 33 + 2 * q + 1] = fma(a.y, b.x, -(a.x * b.y));
                }
                __syncwarp();
                mine = 0.0;
#pragma unroll
                for (int r = 0; r < 32; ++r) mine += tbuf[r * 33 + lane];
                __syncwarp();
            }
            const double other = __shfl_xor_sync(FULL, mine, 1);
            const double2 ga = (lane & 1) ? cmk(other, mine) : cmk(mine, other);
            const double nother = __shfl_xor_sync(FULL, nr, 1);
            const double al = (lane & 1) ? nother : nr, be = (lane & 1) ? nr : nother;
            const double g2 = cabs2(ga);
            double c = 1.0, sn = 0.0;
            double2 ec = cmk(1.0, 0.0);
            if (g2 > fmax(tol2 * (al * be), floor2) && al > 0.0 && be > 0.0) {  // as jacobi_rows_t
                const double ig = rsqrt(g2);
                const double gm = g2 * ig;
                const double dd = be - al;
                const double ir = rsqrt(fma(dd, dd, 4.0 * g2));
                const double c2 = fma(0.5 * fabs(dd), ir, 0.5);
                const double ic = rsqrt(c2);
                c = c2 * ic;
                const double t = (dd >= 0.0 ? gm : -gm) * ir * (ic * ic);
                sn = t * c;
                ec = cmk(ga.x * ig, ga.y * ig);
                nr = (lane & 1) ? be + t * gm : al - t * gm;
                any = true;
            }
            if (!(lane & 1)) prm[w][lane >> 1] = make_double4(c, sn, ec.x, ec.y);
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const double4 pr = prm[w][q];
                const double2 a = x[2 * q];
                const double2 bb = cmul(cmk(pr.z, pr.w), x[2 * q + 1]);
                x[2 * q] = cmk(pr.x * a.x - pr.y * bb.x, pr.x * a.y - pr.y * bb.y);
                x[2 * q + 1] = cmk(pr.y * a.x + pr.x * bb.x, pr.y * a.y + pr.x * bb.y);
                if ((q & 3) == 3) __syncwarp();  // keeps the parameter loads from being hoisted (registers)
            }
            {  // positions 1..31 advance by one (31 wraps to 1), position 0 stays: one register cycle
                const double2 tmp = x[jw_slot(31)];
#pragma unroll
                for (int pos = 31; pos >= 2; --pos) x[jw_slot(pos)] = x[jw_slot(pos - 1)];
                x[jw_slot(1)] = tmp;
            }
            nr = __shfl_sync(FULL, nr, jw_slot(jw_prev(jw_pos(lane))));
        }
        if (!__any_sync(FULL, any)) break;  // a full sweep without rotation: converged
    }
    nr = norms();
#pragma unroll
    for (int r = 0; r < 32; ++r) R[r * 32 + lane] = x[r];
    sN[i * 32 + lane] = nr;
    if (lane == 0) X.sweeps[p0 + i] = sweep;
}

__global__ void __launch_bounds__(128) k_trunc_epi(PlanD P, PassD X, int p0, const double2* sR, const double* sN,
                                                  const int* sPiv, const int* sMeta, double eps, int mode) {
    __shared__ double2 B[32 * 33];
    __shared__ double nrm[32];
    __shared__ int piv[32], ord[32];
    __shared__ int s_rank;
    const int i = blockIdx.x, p = p0 + i;
    const int ncol = sMeta[2 * i], rowsM = sMeta[2 * i + 1];
    if (ncol < 0) return;
    for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) {
        const int r = idx >> 5, j = idx & 31;
        B[r + j * 33] = sR[(size_t)i * 1024 + idx];
    }
    if (threadIdx.x < 32) {
        nrm[threadIdx.x] = sN[i * 32 + threadIdx.x];
        piv[threadIdx.x] = sPiv[i * 32 + threadIdx.x];
    }
    __syncthreads();
    const int bp = X.bp[p];
    const double2* Vt = P.V + P.bp_V_off[bp];
    truncate_epilogue(X, p, P.k, B, 33, ncol, rowsM, piv, nrm, ord, Vt, rowsM, rowsM, eps, mode, s_rank);
}

// ------------------------------------------------------------------ leaf truncation, wide split path
// Leaves of 33..64 triangles (C4/C5: 64): the one-sided Jacobi is half of the leaf truncation and
// the direct prologue (M^* = Zhat V^*, up to 125 x 64 in shared memory) allows one CTA per SM, so
// the Jacobi rounds (one block barrier each) run one pair per SM.  Split: (1) k_trunc_qr64, the
// prologue and pivoted QR exactly as k_truncate (one CTA per SM), R (ncol x rowsM) and the pivot
// order to a scratch slab; (2) k_trunc_jepi64, Jacobi on the rows of R and the epilogue with R
// alone in shared memory (66 KB: three pairs per SM).  Same device functions, same results.
constexpr int T64 = 64;
// LEAF = false (levels above the leaves with rowsM = k1 + k2 <= 64): Vhat = [C_{t1c1} E_{t1c};
// C_{t2c2} E_{t2c}] (rowsM x k, built by the prologue in shared memory) also goes to the scratch
// (sV, ld 64) for the epilogue's C = Qhat^* Vhat.
template <bool LEAF>
__global__ void __launch_bounds__(512, 1) k_trunc_qr64(PlanD P, PassD X, int p0, int ldv, int ldb, double2* sR, int* sPiv,
                                                      int* sMeta, double2* sV) {
    extern __shared__ double2 smd[];
    __shared__ int s_piv;
    __shared__ double2 sh[2];
    const int i = blockIdx.x, p = p0 + i;
    double2* B;
    double* nrm;
    int *piv, *ord;
    int rowsM, ldvt, ldB;
    const double2* Vt;
    const int ncol = truncate_prologue<LEAF>(P, X, p, smd, ldv, ldb, false, B, ldB, nrm, piv, ord, rowsM, Vt, ldvt, s_piv, sh);
    if (threadIdx.x == 0) {
        sMeta[2 * i] = ncol;  // -1: empty pair, already recorded
        sMeta[2 * i + 1] = rowsM;
    }
    if (ncol < 0) return;
    double2* R = sR + (size_t)i * T64 * T64;  // column-major, ld 64
    for (int idx = threadIdx.x; idx < ncol * rowsM; idx += blockDim.x) {
        const int r = idx % ncol, j = idx / ncol;
        R[r + (size_t)j * T64] = B[r + (size_t)j * ldB];
    }
    for (int j = threadIdx.x; j < rowsM; j += blockDim.x) sPiv[i * T64 + j] = piv[j];
    if (!LEAF) {
        double2* V = sV + (size_t)i * T64 * P.k;
        for (int idx = threadIdx.x; idx < rowsM * P.k; idx += blockDim.x) {
            const int r = idx % rowsM, nu = idx / rowsM;
            V[r + (size_t)nu * T64] = Vt[r + (size_t)nu * ldvt];
        }
    }
}

template <int NT, bool LEAF>
__global__ void __launch_bounds__(NT, NT == 64 ? 3 : NT == 128 ? 3 : 2) k_trunc_jepi64(PlanD P, PassD X, int p0, const double2* sR,
                                                                                   const int* sPiv, const int* sMeta, double eps,
                                                                                   int mode, const double2* sV) {
    constexpr int LD = T64 + 1;
    extern __shared__ double2 smd[];
    __shared__ double nrm[T64];
    __shared__ int piv[T64], ord[T64];
    __shared__ int flag, s_rank;
    const int i = blockIdx.x, p = p0 + i;
    const int ncol = sMeta[2 * i], rowsM = sMeta[2 * i + 1];
    if (ncol < 0) return;
    double2* B = smd;
    const double2* R = sR + (size_t)i * T64 * T64;
    for (int idx = threadIdx.x; idx < ncol * rowsM; idx += blockDim.x) {
        const int r = idx % ncol, j = idx / ncol;
        B[r + (size_t)j * LD] = R[r + (size_t)j * T64];
    }
    for (int j = threadIdx.x; j < rowsM; j += blockDim.x) piv[j] = sPiv[i * T64 + j];
    __syncthreads();
    const int nsw = jacobi_rows_auto(B, LD, ncol, rowsM, nrm, &flag);
    if (threadIdx.x == 0) X.sweeps[p] = nsw;
    if (LEAF) {
        const double2* Vt = P.V + P.bp_V_off[X.bp[p]];
        truncate_epilogue(X, p, P.k, B, LD, ncol, rowsM, piv, nrm, ord, Vt, rowsM, rowsM, eps, mode, s_rank);
    } else {
        const double2* Vt = sV + (size_t)i * T64 * P.k;
        truncate_epilogue(X, p, P.k, B, LD, ncol, rowsM, piv, nrm, ord, Vt, T64, X.rowsb[p], eps, mode, s_rank);
    }
}

size_t trunc_split64_scratch_bytes(int np, bool leaf, int k) {
    return (size_t)np * (T64 * T64 * sizeof(double2) + T64 * sizeof(int) + 2 * sizeof(int) +
                         (leaf ? 0 : (size_t)T64 * k * sizeof(double2))) + 16;
}

template <bool LEAF>
static void split64_launch(const PlanD& P, const PassD& X, int p0, int np, const TruncLaunch& L, double eps, int mode,
                           void* scratch, cudaStream_t s) {
    double2* sR = reinterpret_cast<double2*>(scratch);
    int* sPiv = reinterpret_cast<int*>(sR + (size_t)np * T64 * T64);
    int* sMeta = sPiv + (size_t)np * T64;
    const uintptr_t vend = reinterpret_cast<uintptr_t>(sMeta + 2 * (size_t)np);
    double2* sV = reinterpret_cast<double2*>((vend + 15) & ~(uintptr_t)15);  // (16-byte aligned)
    static size_t attr_qr = 0;
    static bool attr_j = false;
    const size_t smj = (size_t)(T64 + 1) * T64 * sizeof(double2);
    if (L.smem > attr_qr) {
        cudaFuncSetAttribute(k_trunc_qr64<LEAF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem);
        attr_qr = L.smem;
    }
    if (!attr_j) {
        cudaFuncSetAttribute(k_trunc_jepi64<64, LEAF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smj);
        cudaFuncSetAttribute(k_trunc_jepi64<128, LEAF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smj);
        cudaFuncSetAttribute(k_trunc_jepi64<256, LEAF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smj);
        attr_j = true;
    }
    k_trunc_qr64<LEAF><<<np, 512, L.smem, s>>>(P, X, p0, L.ldv, L.ldb, sR, sPiv, sMeta, sV);
    // Jacobi + epilogue threads (dh2_set_option "trunc64_threads")
    if (P.t64_threads == 64)
        k_trunc_jepi64<64, LEAF><<<np, 64, smj, s>>>(P, X, p0, sR, sPiv, sMeta, eps, mode, sV);
    else if (P.t64_threads == 256)
        k_trunc_jepi64<256, LEAF><<<np, 256, smj, s>>>(P, X, p0, sR, sPiv, sMeta, eps, mode, sV);
    else
        k_trunc_jepi64<128, LEAF><<<np, 128, smj, s>>>(P, X, p0, sR, sPiv, sMeta, eps, mode, sV);
}

void launch_truncate_split64(const PlanD& P, bool row, int p0, int np, const TruncLaunch& L, bool leaf_level, double eps,
                             int mode, void* scratch, cudaStream_t s) {
    if (!np) return;
    const PassD& X = row ? P.row : P.col;
    if (leaf_level)
        split64_launch<true>(P, X, p0, np, L, eps, mode, scratch, s);
    else
        split64_launch<false>(P, X, p0, np, L, eps, mode, scratch, s);
}

size_t trunc_split_scratch_bytes(int np) { return (size_t)np * (1024 * sizeof(double2) + 32 * sizeof(double) + 34 * sizeof(int)); }

void launch_truncate_split(const PlanD& P, bool row, int p0, int np, const TruncLaunch& L, double eps, int mode,
                           void* scratch, bool fused, int fuse_direct, const int* mirror, cudaStream_t s) {
    if (!np) return;
    const PassD& X = row ? P.row : P.col;
    double2* sR = reinterpret_cast<double2*>(scratch);
    double* sN = reinterpret_cast<double*>(sR + (size_t)np * 1024);
    int* sPiv = reinterpret_cast<int*>(sN + (size_t)np * 32);
    int* sMeta = sPiv + (size_t)np * 32;
    if (fused)
        k_trunc_zqr<<<np, 256, trunc_zqr_smem(P), s>>>(P, X, row, p0, mirror, fuse_direct, sR, sPiv, sMeta);
    else
        k_trunc_qr<<<np, 128, L.smem, s>>>(P, X, p0, L.ldv, L.ldb, L.append, sR, sPiv, sMeta);
    k_jacobi_w32<<<(np + 3) / 4, 128, 0, s>>>(X, p0, np, sR, sN, sMeta);
    k_trunc_epi<<<np, 128, 0, s>>>(P, X, p0, sR, sN, sPiv, sMeta, eps, mode);
}

TruncLaunch plan_truncate(const PlanD& P, int np, int maxrowsM, int maxZrows, bool leaf_level, bool force_ws) {
    TruncLaunch L;
    L.ldv = odd_ld(max(maxrowsM, 1));
    L.ldb = odd_ld(max(maxZrows, 1));
    // tall M^* (zr > #t) at a leaf level: reduce it to its R factor by streamed chunks when that
    // fits more CTAs per SM (C4 leaves of 64: 130 -> 102 KB, 1 -> 2 CTAs; not for C2 or C5)
    const size_t extra = (size_t)L.ldv * (sizeof(double) + 2 * sizeof(int)) + 16;
    const size_t bytes_d = ((leaf_level ? 0 : (size_t)L.ldv * P.k + 6 * P.m * P.m) + (size_t)L.ldb * L.ldv) * sizeof(double2) + extra;
    const size_t bytes_a = (size_t)(L.ldv + 33) * L.ldv * sizeof(double2) + extra;
    auto ctas = [&](size_t b) { return b > (size_t)P.smem_optin ? 0 : (int)((size_t)(228 * 1024) / (b + 1024)); };
    L.append = leaf_level && maxZrows > maxrowsM && maxrowsM > 32 && ctas(bytes_a) > ctas(bytes_d);
    if (P.trunc_mode == 1) L.append = false;  // (dh2_set_option "trunc_direct": A/B of the two leaf modes)
    const size_t bytes = L.append ? bytes_a : bytes_d;
    L.use_ws = force_ws || bytes > (size_t)P.smem_optin;
    if (L.use_ws) {
        L.smem = 0;
        L.ws_stride = (bytes + sizeof(double2) - 1) / sizeof(double2);
        L.grid = min(np, P.num_sms * 3);
    } else {
        L.smem = bytes;
        L.ws_stride = 0;
        L.grid = np;
        // 4 warps per pair, more when shared memory holds fewer than 4 pairs per SM (C4/C5: 1-2):
        // QRCP, Jacobi and the appends run their lane groups over more columns / pairs at once
        // (measured: C4 leaves, append mode, 2 pairs per SM: 128 -> 256 threads -15 %; C5 leaves,
        // direct mode, 2 pairs per SM: +18 %; one pair per SM (levels above the leaves): 512, -28 %)
        const int c = ctas(bytes);
        L.threads = (c >= 4 || (c >= 2 && !L.append)) ? 128 : c >= 2 ? 256 : 512;
    }
    return L;
}

void launch_truncate(const PlanD& P, bool row, int p0, int np, const TruncLaunch& L, bool leaf_level, double eps,
                     int mode, double2* ws, cudaStream_t s, const int* plist) {
    if (!np) return;
    const PassD& X = row ? P.row : P.col;
    if (L.use_ws) {
        if (leaf_level)
            k_truncate_ws<true><<<L.grid, 128, 0, s>>>(P, X, p0, np, L.ldv, L.ldb, L.append, eps, mode, ws, L.ws_stride, plist);
        else
            k_truncate_ws<false><<<L.grid, 128, 0, s>>>(P, X, p0, np, L.ldv, L.ldb, L.append, eps, mode, ws, L.ws_stride, plist);
    } else if (leaf_level) {
        k_truncate<true><<<np, L.threads, L.smem, s>>>(P, X, p0, L.ldv, L.ldb, L.append, eps, mode, plist);
    } else {
        k_truncate<false><<<np, L.threads, L.smem, s>>>(P, X, p0, L.ldv, L.ldb, L.append, eps, mode, plist);
    }
}

// Column pass from the row pass by adjoint symmetry (check_symmetry in
// dh2_api.cu): for the column pair p = (s,c) and the row pair q = (s,-c), the column-pass
// matrices are the complex conjugates of the row-pass ones, so k' = k, sigma' = sigma,
// Q' = conj(Q) (F' = conj(F)) and C' = conj(C).  CTA per column pair.
__global__ void k_mirror_pass(PlanD P, const int* col2row, int p0) {
    const int p = p0 + blockIdx.x;
    const int q = col2row[p];
    const PassD& R = P.row;
    const PassD& X = P.col;
    if (threadIdx.x == 0) {  // the factors themselves are read conjugated from the row storage (P.col_conj)
        X.rank[p] = R.rank[q];
        X.nsig[p] = R.nsig[q];
        X.disc[p] = R.disc[q];
        X.sweeps[p] = R.sweeps[q];
    }
}

void launch_mirror_pass(const PlanD& P, const int* col2row, int p0, int np, cudaStream_t s) {
    if (np) k_mirror_pass<<<np, 32, 0, s>>>(P, col2row, p0);
}

// Projection (Lemma Projections): T_b = C_tc S_b, S~_b = T_b C'_sc^*.  CTA per block,
// rows of C_tc in chunks of <= `chunk` (T chunk x k in shared memory); both products on the FP64
// tensor cores, S_b read coalesced through its antipodal mirror block where that is local.
__global__ void __launch_bounds__(128, 4) k_project(PlanD P, int b0, int ldt, int chunk, const int* mirror, const int* blist) {
    extern __shared__ double2 sm[];
    const int b = blist ? blist[blockIdx.x] : b0 + blockIdx.x, k = P.k;
    const int pr = P.blk_prow[b], pc = P.blk_pcol[b];
    const int kt = P.row.rank[pr], ks = P.col.rank[pc];
    const int lt = P.row.kb[pr], ls = P.col.kb[pc];
    const double2* Ct = P.row.C + P.row.C_off[pr];
    const double2* Cs = P.col.C + P.col.C_off[pc];
    const int mb = mirror[b];
    const double2* Sg = P.S + (size_t)P.blk_slot[mb >= 0 ? mb : b] * k * k;
    double2* St = P.St + P.blk_St_off[b];
    double2* T = sm;
    for (int a0 = 0; a0 < kt; a0 += chunk) {
        const int nb = min(chunk, kt - a0);
        if (a0) __syncthreads();
        chunk_gemm_S_dmma<true>(Ct, lt, a0, nb, Sg, false, mb < 0, 1.0, k, T, ldt);
        __syncthreads();
        if (P.col_conj)  // C'_sc stored as the row C at (s,-c): C' = conj(stored)
            dmma_abh<true, true>(T, ldt, nb, Cs, ls, ks, k, St + a0, lt);
        else
            dmma_abh<true, false>(T, ldt, nb, Cs, ls, ks, k, St + a0, lt);
    }
}

void launch_project(const PlanD& P, int b0, int nb, int maxkrow, const int* mirror, cudaStream_t s, const int* blist) {
    if (!nb) return;
    const int chunk = max(1, min(maxkrow, 64));
    int ldt = odd_ld(chunk);
    size_t sm = (size_t)ldt * P.k * sizeof(double2);
    k_project<<<nb, 128, sm, s>>>(P, b0, ldt, chunk, mirror, blist);
}

// ============================================================== matvec (far field)
// Forward transformation on the column basis: xh_sc = B_sc^* x|_s, nested through the
// transfers (V, E for ORIG; Q', F' for RECOMP).  Coefficients stored with stride k.
__global__ void k_mv_forward(PlanD P, bool recomp, int p0, int pend, int wpp, const double2* xp, double2* xh) {
    const PassD& X = P.col;
    // wpp: one warp per pair and blockDim / 32 pairs per CTA (RECOMP, small ranks), else one CTA per pair
    const int lane = threadIdx.x & 31;
    const int p = p0 + (wpp ? blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) : blockIdx.x), k = P.k, m = P.m;
    if (p >= pend) return;
    const int tid = wpp ? lane : threadIdx.x, nth = wpp ? 32 : blockDim.x;
    // sym: V_sc and E of the column pair are the conjugates of those of the row pair (s,-c)
    const bool vcj = !recomp && P.sym;
    const int bp = vcj ? P.row.bp[P.col2row[p]] : X.bp[p];
    const bool leaf = X.child0[p] < 0;
    const int kout = recomp ? X.rank[p] : k;
    if (leaf && P.mv_fwd_warp) {
        // a warp per output coefficient (two at a time): lanes over the rows of the leaf (coalesced reads
        // of the column B(:, a); a thread per coefficient, as below, reads with stride nt and leaves
        // most lanes idle at small ranks), shuffle reduction in a fixed order
        const int w = wpp ? 0 : threadIdx.x >> 5, nw = wpp ? 1 : blockDim.x >> 5;
        const int t = P.bp_t[bp];
        const int nt = P.c_size[t];
        const double2* x = xp + P.c_begin[t];
        const double2* B = recomp ? (X.Q + X.Q_off[p]) : (P.V + P.bp_V_off[bp]);
        const bool plain = (recomp && P.col_conj) || vcj;
        for (int a = w; a < kout; a += 2 * nw) {
            const int a2 = a + nw;
            const bool two = a2 < kout;
            double2 acc = cmk(0.0, 0.0), acc2 = cmk(0.0, 0.0);
            for (int i = lane; i < nt; i += 32) {
                const double2 xv = x[i], b1 = B[i + (size_t)a * nt], b2 = two ? B[i + (size_t)a2 * nt] : cmk(0.0, 0.0);
                if (plain) {
                    cfma(acc, b1, xv);
                    cfma(acc2, b2, xv);
                } else {
                    cfma_cj(acc, b1, xv);
                    cfma_cj(acc2, b2, xv);
                }
            }
            acc = warp_sum2(acc);
            acc2 = warp_sum2(acc2);
            if (lane == 0) {
                xh[(size_t)p * k + a] = acc;
                if (two) xh[(size_t)p * k + a2] = acc2;
            }
        }
        return;
    }
    for (int a = tid; a < kout; a += nth) {
        double2 acc = cmk(0.0, 0.0);
        if (leaf) {
            const int t = P.bp_t[bp];
            const int nt = P.c_size[t];
            const double2* x = xp + P.c_begin[t];
            const double2* B = recomp ? (X.Q + X.Q_off[p]) : (P.V + P.bp_V_off[bp]);
            if ((recomp && P.col_conj) || vcj)  // Q' (V) stored as the row Q (V) at (s,-c): conj(Q') = stored
                for (int i = 0; i < nt; ++i) cfma(acc, B[i + (size_t)a * nt], x[i]);
            else
                for (int i = 0; i < nt; ++i) cfma_cj(acc, B[i + (size_t)a * nt], x[i]);
        } else {
            const int ch[2] = {X.child0[p], X.child1[p]};
            if (recomp) {
                const double2* F = X.Q + X.Q_off[p];
                const int ldf = X.rowsb[p];
                int off = 0;
                for (int c = 0; c < 2; ++c) {
                    const int kc = X.rank[ch[c]];
                    if (P.col_conj)
                        for (int r = 0; r < kc; ++r) cfma(acc, F[off + r + (size_t)a * ldf], xh[(size_t)ch[c] * k + r]);
                    else
                        for (int r = 0; r < kc; ++r) cfma_cj(acc, F[off + r + (size_t)a * ldf], xh[(size_t)ch[c] * k + r]);
                    off += kc;
                }
            } else {
                const double2* Eg = P.E + P.bp_E_off[bp];
                int jx = a % m, jy = (a / m) % m, jz = a / (m * m);
                for (int c = 0; c < 2; ++c) {
                    const double2* F = Eg + c * 3 * m * m;
                    for (int nup = 0; nup < k; ++nup) {
                        int px = nup % m, py = (nup / m) % m, pz = nup / (m * m);
                        double2 e = cmul(cmul(F[px * m + jx], F[m * m + py * m + jy]), F[2 * m * m + pz * m + jz]);
                        if (vcj)  // E_{s'c} = conj E_{s',-c}
                            cfma(acc, e, xh[(size_t)ch[c] * k + nup]);
                        else
                            cfma_cj(acc, e, xh[(size_t)ch[c] * k + nup]);
                    }
                }
            }
        }
        xh[(size_t)p * k + a] = acc;
    }
}

// Coupling: yh_tc = sum_{b=(t,s,c)} S_b xh_sc (ORIG) or S~_b xh'_sc (RECOMP).
// gsz threads per pair, blockDim / gsz pairs per CTA (RECOMP ranks are ~10-20: 16 lanes per pair keep
// the lanes busy and cut the CTA count by 8; each coefficient is summed by one thread in the same order).
__global__ void k_mv_couple(PlanD P, bool recomp, int p0, int pend, int gsz, const double2* xh, double2* yh) {
    const PassD& X = P.row;
    const int p = p0 + blockIdx.x * (blockDim.x / gsz) + threadIdx.x / gsz, k = P.k;
    if (p >= pend) return;
    const int kout = recomp ? X.rank[p] : k;
    for (int a = threadIdx.x % gsz; a < kout; a += gsz) {
        double2 acc = cmk(0.0, 0.0);
        for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
            const int b = X.blk[ib];
            const int pc = P.blk_pcol[b];
            const double2* x = xh + (size_t)pc * k;
            if (recomp) {
                const double2* St = P.St + P.blk_St_off[b];
                const int ks = P.col.rank[pc];
                const int lt = X.kb[p];
                for (int c = 0; c < ks; ++c) cfma(acc, St[a + (size_t)c * lt], x[c]);
            } else {
                const double2* S = P.S + (size_t)P.blk_slot[b] * k * k;
                for (int c = 0; c < k; ++c) cfma(acc, S[a + (size_t)c * k], x[c]);
            }
        }
        yh[(size_t)p * k + a] = acc;
    }
}

// Backward transformation (top-down): yh_{t'c'} += T yh_{tc} for every parent (t,c) with
// sd(c) = c'; T = E_{t'c} (ORIG) or F_{t'c} (RECOMP).
__global__ void k_mv_backward(PlanD P, bool recomp, int p0, int pend, int gsz, double2* yh) {
    const PassD& X = P.row;
    const int p = p0 + blockIdx.x * (blockDim.x / gsz) + threadIdx.x / gsz, k = P.k, m = P.m;
    if (p >= pend) return;
    const int kout = recomp ? X.rank[p] : k;
    for (int a = threadIdx.x % gsz; a < kout; a += gsz) {
        double2 acc = yh[(size_t)p * k + a];
        for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) {
            const int pp = X.par[ip];
            const int ci = X.par_child[ip];
            const double2* v = yh + (size_t)pp * k;
            if (recomp) {
                const double2* F = X.Q + X.Q_off[pp];
                const int ldf = X.rowsb[pp];
                const int off = ci == 0 ? 0 : X.rank[X.child0[pp]];
                const int kp = X.rank[pp];
                for (int c = 0; c < kp; ++c) cfma(acc, F[off + a + (size_t)c * ldf], v[c]);
            } else {
                const double2* F = P.E + P.bp_E_off[X.bp[pp]] + ci * 3 * m * m;
                int px = a % m, py = (a / m) % m, pz = a / (m * m);
                for (int nu = 0; nu < k; ++nu) {
                    int jx = nu % m, jy = (nu / m) % m, jz = nu / (m * m);
                    double2 e = cmul(cmul(F[px * m + jx], F[m * m + py * m + jy]), F[2 * m * m + pz * m + jz]);
                    cfma(acc, e, v[nu]);
                }
            }
        }
        yh[(size_t)p * k + a] = acc;
    }
}

// Leaf output: y|_t = sum_{c} B_tc yh_tc over the row pairs of each leaf cluster.
// Leaf output: y|_t = sum_c B_tc yh_tc over the row pairs of each leaf cluster.  CTA per leaf
// cluster, 256 threads = (row i, pair slice): the pairs are split into blockDim/nt slices summed
// separately, then added in slice order (fixed order: deterministic).
__global__ void __launch_bounds__(256) k_mv_leaf_out(PlanD P, bool recomp, const int* lc, const int* lc_ptr, int g0,
                                                     const double2* yh, double2* yp) {
    __shared__ double2 part[256];
    const PassD& X = P.row;
    const int g = g0 + blockIdx.x, k = P.k;
    const int q0 = lc_ptr[g], q1 = lc_ptr[g + 1];
    const int t = P.bp_t[X.bp[lc[q0]]];
    const int nt = P.c_size[t];
    const int ns = max(1, (int)blockDim.x / max(nt, 1));  // pair slices
    for (int i0 = 0; i0 < nt; i0 += blockDim.x / ns) {
        const int i = i0 + threadIdx.x % (blockDim.x / ns), sl = threadIdx.x / (blockDim.x / ns);
        double2 acc = cmk(0.0, 0.0);
        if (i < nt && sl < ns)
            for (int q = q0 + sl; q < q1; q += ns) {
                const int p = lc[q];
                const double2* v = yh + (size_t)p * k;
                if (recomp) {
                    const double2* Q = X.Q + X.Q_off[p];
                    const int kp = X.rank[p];
                    for (int a = 0; a < kp; ++a) cfma(acc, Q[i + (size_t)a * nt], v[a]);
                } else {
                    const double2* V = P.V + P.bp_V_off[X.bp[p]];
                    for (int a = 0; a < k; ++a) cfma(acc, V[i + (size_t)a * nt], v[a]);
                }
            }
        part[threadIdx.x] = acc;
        __syncthreads();
        if (threadIdx.x < blockDim.x / ns && i < nt) {
            double2 sum = cmk(0.0, 0.0);
            for (int r = 0; r < ns; ++r) sum = cadd(sum, part[r * (blockDim.x / ns) + threadIdx.x]);
            yp[P.c_begin[t] + i] = sum;
        }
        __syncthreads();
    }
}

__global__ void k_permute(const int64_t* perm, const double2* in, double2* out, int n, bool gather) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (gather)
        out[p] = in[perm[p]];
    else
        out[perm[p]] = in[p];
}

void launch_mv_forward(const PlanD& P, bool recomp, int p0, int np, const double2* xp, double2* xh, cudaStream_t s) {
    if (!np) return;
    if (recomp && P.mv_fwd_warp == 2)
        k_mv_forward<<<(np + 3) / 4, 128, 0, s>>>(P, recomp, p0, p0 + np, 1, xp, xh);
    else
        k_mv_forward<<<np, 64, 0, s>>>(P, recomp, p0, p0 + np, 0, xp, xh);
}
void launch_mv_couple(const PlanD& P, bool recomp, int p0, int np, const double2* xh, double2* yh, cudaStream_t s) {
    if (!np) return;
    if (recomp && P.mv_fwd_warp)
        k_mv_couple<<<(np + 7) / 8, 128, 0, s>>>(P, recomp, p0, p0 + np, 16, xh, yh);
    else
        k_mv_couple<<<np, 64, 0, s>>>(P, recomp, p0, p0 + np, 64, xh, yh);
}
void launch_mv_backward(const PlanD& P, bool recomp, int p0, int np, double2* yh, cudaStream_t s) {
    if (!np) return;
    if (recomp && P.mv_fwd_warp)
        k_mv_backward<<<(np + 7) / 8, 128, 0, s>>>(P, recomp, p0, p0 + np, 16, yh);
    else
        k_mv_backward<<<np, 64, 0, s>>>(P, recomp, p0, p0 + np, 64, yh);
}
void launch_mv_leaf_out(const PlanD& P, bool recomp, const int* lc, const int* lc_ptr, int g0, int nlc, const double2* yh,
                        double2* yp, cudaStream_t s) {
    if (nlc) k_mv_leaf_out<<<nlc, 256, 0, s>>>(P, recomp, lc, lc_ptr, g0, yh, yp);
}
// Exchange packing: dst[doff[i] + j] = src[soff[i] + j] for j < len[i], CTA per segment.
template <typename T>
__global__ void k_copy_segments(const T* src, T* dst, const int64_t* soff, const int64_t* doff, const int64_t* len) {
    const int i = blockIdx.x;
    const T* a = src + soff[i];
    T* b = dst + doff[i];
    for (int64_t j = threadIdx.x; j < len[i]; j += blockDim.x) b[j] = a[j];
}
void launch_copy_segments(const double2* src, double2* dst, const int64_t* soff, const int64_t* doff, const int64_t* len,
                          int nseg, cudaStream_t s) {
    if (nseg) k_copy_segments<double2><<<nseg, 128, 0, s>>>(src, dst, soff, doff, len);
}
void launch_copy_segments_i(const int* src, int* dst, const int64_t* soff, const int64_t* doff, const int64_t* len,
                            int nseg, cudaStream_t s) {
    if (nseg) k_copy_segments<int><<<nseg, 32, 0, s>>>(src, dst, soff, doff, len);
}

// Compaction of truncation outputs (memory-lean path): item i copies the rows x cols matrix at
// src + soff[i] (leading dimension lds[i]) to dst + doff[i] with leading dimension rows[i].  CTA per item.
__global__ void k_copy_mat(const double2* src, double2* dst, const int64_t* soff, const int64_t* doff, const int* rows,
                           const int* cols, const int* lds) {
    const int i = blockIdx.x;
    const int r = rows[i], c = cols[i], ld = lds[i];
    const double2* a = src + soff[i];
    double2* b = dst + doff[i];
    for (int idx = threadIdx.x; idx < r * c; idx += blockDim.x) {
        const int x = idx % r, y = idx / r;
        b[idx] = a[x + (size_t)y * ld];
    }
}
void launch_copy_mat(const double2* src, double2* dst, const int64_t* soff, const int64_t* doff, const int* rows,
                     const int* cols, const int* lds, int n, cudaStream_t s) {
    if (n) k_copy_mat<<<n, 128, 0, s>>>(src, dst, soff, doff, rows, cols, lds);
}

void launch_permute(const int64_t* perm, const double2* in, double2* out, int n, bool gather, cudaStream_t s) {
    k_permute<<<(n + 255) / 256, 256, 0, s>>>(perm, in, out, n, gather);
}

}  // namespace dh2

namespace dh2 {
// Opt the shared-memory-heavy kernels into the full dynamic shared memory of sm_100a
// (227 KB per CTA minus the kernel's static shared memory).  Returns the first error.
cudaError_t configure_kernels() {
    static cudaError_t done = cudaErrorNotReady;
    if (done != cudaErrorNotReady) return done;
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const void* ks[] = {(const void*)k_leafV<0>, (const void*)k_leafV<2>, (const void*)k_leafV<3>, (const void*)k_leafV<4>,
                        (const void*)k_leafV<5>, (const void*)k_basis<true, 4>, (const void*)k_basis<true, 2>,
                        (const void*)k_basis<true, 3>, (const void*)k_total_weights<true, 3>, (const void*)k_truncate_fused,
                        (const void*)k_block_weights<256>, (const void*)k_block_weights<512>, (const void*)k_total_weights<true, 4>, (const void*)k_total_weights<true, 2>, (const void*)k_truncate<true>, (const void*)k_truncate<false>, (const void*)k_trunc_qr, (const void*)k_trunc_zqr,
                        (const void*)k_project};
    for (const void* f : ks) {
        if (e != cudaSuccess) break;
        cudaFuncAttributes a;
        e = cudaFuncGetAttributes(&a, f);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)a.sharedSizeBytes);
    }
    done = e;
    return e;
}
}  // namespace dh2
