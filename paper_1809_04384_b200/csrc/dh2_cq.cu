// Column-per-thread chunk appends for k > 64 (C4/C5: k = 125): the basis weights (Eq. 18,
// P:934-956) and the total weights as structured Householder QRs whose reflections
// run with thread c owning column c of the chunk in REGISTERS and of the triangle R in a global
// (L2-resident) scratch slab of the CTA, instead of the whole CTA cooperating on one column at a
// time in shared memory (cta_qr_append: lane-group reductions per column, 512 threads, one pair
// per SM, barrier- and shuffle-bound).
//
// One reflection j of an NB-row chunk B appended to the k x k upper-triangular R
// ([R; B] = Q [R'; 0], the same structured reflectors H_j = I - tau_j u_j u_j^* as cta_qr_append,
// u_j = [u0_j e_j; B(:, j)]):
//   every thread c > j:  w = tau_j (conj(u0_j) R[j, c] + B(:, j)^* B(:, c)),
//                        R[j, c] -= u0_j w,  B(:, c) -= B(:, j) w
// -- a dot product and an axpy over the thread's own NB registers, no reductions across threads.
// Thread j + 1 forms reflector j + 1 right after its update of step j (look-ahead) and publishes
// B(:, j + 1), u0 and tau in shared memory (double-buffered by step parity): one 128-thread
// barrier per reflection.  Thread c reads and writes only column c of R (row j at step j,
// prefetched three steps ahead), so R needs no shared memory: 128 threads, ~40 KB of shared
// memory (the staging buffer of the chunk formation) and <= 128 registers give 4 pairs per SM
// whose reflection chains hide each other's latency.
#include "dh2_kernels.cuh"

namespace dh2 {

constexpr int CQ_KP = 128;    // row pitch of the scratch triangle (k <= 128)

template <int NB>
struct CqRefl {
    double2 u[2][NB];  // reflector j: B(:, j) after the reflections < j (double-buffered by step parity)
    double2 u0[2];
    double tau[2];
};

// Reflector j formed by the owner of column j from its column b (after the reflections < j) and
// alpha = R[j, j]: H = I - tau v v^*, v = [u0; b], H^* [alpha; b] = [beta; 0]; R[j, j] <- beta.
// Tiny columns are left in place (tau = 0, see HH_TINY).  The owner is on the critical path of
// every reflection: the norm is summed in 8 independent chains and the reflector formed from two
// independent rsqrt and one division, xn = t rsqrt(t), t = s + |alpha|^2,
// ph = alpha rsqrt(|alpha|^2), tau = rsqrt(t) / (xn + |alpha|).
template <int NB>
__device__ __forceinline__ void cq_publish(CqRefl<NB>& sh, int j, const double2 (&b)[NB], double2 alpha, double2* Rs) {
    double sp[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) sp[c] = 0.0;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        sp[(2 * i) & 7] = fma(b[i].x, b[i].x, sp[(2 * i) & 7]);
        sp[(2 * i + 1) & 7] = fma(b[i].y, b[i].y, sp[(2 * i + 1) & 7]);
    }
    const double s = ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
    double tau = 0.0;
    double2 beta = alpha, u0 = cmk(0.0, 0.0);
    if (s > HH_TINY) {
        const double a2 = cabs2(alpha);
        const double t = s + a2;
        const double rx = rsqrt(t);
        const double ra = a2 > 0.0 ? rsqrt(a2) : 0.0;
        const double xn = t * rx, aa = a2 * ra;
        const double2 ph = a2 > 0.0 ? cscale(alpha, ra) : cmk(1.0, 0.0);
        beta = cscale(ph, -xn);
        u0 = cscale(ph, aa + xn);
        tau = rx / (xn + aa);
    }
    const int buf = j & 1;
#pragma unroll
    for (int i = 0; i < NB; ++i) sh.u[buf][i] = b[i];
    sh.u0[buf] = u0;
    sh.tau[buf] = tau;
    Rs[(size_t)j * CQ_KP + j] = beta;
}

// Columns of thread t: NC = 1 (128 threads): {t}; NC = 2 (64 threads): {t, 127 - t} -- every warp
// then holds low and high columns, so the warps (and the SM sub-partitions they run on) stay
// equally busy while the active columns c > j shrink towards the right of the triangle.
template <int NC>
__device__ __forceinline__ int cq_col(int q) {
    return q == 0 ? (int)threadIdx.x : CQ_KP - 1 - (int)threadIdx.x;
}
// the thread and column slot holding column c
template <int NC>
__device__ __forceinline__ void cq_owner(int c, int& t, int& q) {
    if (NC == 1 || c < CQ_KP / 2) {
        t = c;
        q = 0;
    } else {
        t = CQ_KP - 1 - c;
        q = 1;
    }
}

// One reflection on the column slots in MASK (warp-uniform: slots no lane of the warp has active
// are skipped; inactive lanes compute on their registers, which are dead, and store nothing):
// w = tau (conj(u0) R[j, c] + u^* b), R[j, c] -= u0 w, b -= u w (FMA form).
template <int NB, int NC, int MASK, int CH>
__device__ __forceinline__ void cq_step(double2 (&b)[NC][NB], const double2 (&r0)[NC], const bool (&act)[NC],
                                        const CqRefl<NB>& sh, int buf, double2* Rs, int j) {
    const double tau = sh.tau[buf];
    const double2 u0 = sh.u0[buf];
    // w in CH independent chains (the dot product is on the critical path)
    double2 wc[NC][CH];
#pragma unroll
    for (int q = 0; q < NC; ++q) {
#pragma unroll
        for (int c = 0; c < CH; ++c) wc[q][c] = cmk(0.0, 0.0);
        if (MASK >> q & 1) cfma_cj(wc[q][NB % CH], u0, r0[q]);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const double2 u = sh.u[buf][i];
#pragma unroll
        for (int q = 0; q < NC; ++q)
            if (MASK >> q & 1) cfma_cj(wc[q][i % CH], u, b[q][i]);
    }
    double2 w[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q)
        if (MASK >> q & 1) {
#pragma unroll
            for (int h = 1; h < CH; h *= 2)
#pragma unroll
                for (int c = 0; c + h < CH; c += 2 * h) wc[q][c] = cadd(wc[q][c], wc[q][c + h]);
            w[q] = cscale(wc[q][0], tau);
            if (act[q]) {
                double2 r = r0[q];
                r.x = fma(-u0.x, w[q].x, r.x);
                r.x = fma(u0.y, w[q].y, r.x);
                r.y = fma(-u0.x, w[q].y, r.y);
                r.y = fma(-u0.y, w[q].x, r.y);
                Rs[(size_t)j * CQ_KP + cq_col<NC>(q)] = r;
            }
        }
    // (u re-read from shared memory rather than kept live across the dot product)
    const volatile double2* uv = sh.u[buf];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const double ux = uv[i].x, uy = uv[i].y;
#pragma unroll
        for (int q = 0; q < NC; ++q)
            if (MASK >> q & 1) {
                double2& x = b[q][i];
                x.x = fma(-ux, w[q].x, x.x);
                x.x = fma(uy, w[q].y, x.x);
                x.y = fma(-ux, w[q].y, x.y);
                x.y = fma(-uy, w[q].x, x.y);
            }
    }
}

// Append the chunk held in registers (thread t: b[q] = B(:, column q of t); rows >= the chunk's
// fill are zero, which leaves every norm and dot product unchanged) into R (scratch, row-major,
// pitch CQ_KP).  first: R is zero (not read).  All threads of the CTA call it.  One barrier per
// reflection; the owner of column j + 1 forms and publishes reflector j + 1 right after its update
// of step j (look-ahead).
template <int NB, int NC, int CH = 4>
__device__ inline void cq_append(double2 (&b)[NC][NB], double2* Rs, int k, bool first, CqRefl<NB>& sh) {
    bool has[NC];
    // R[j, c] prefetched four steps ahead into a ring of four registers per column slot; the steps
    // are unrolled by four so the ring rotates by name (a register move of a pending load would
    // wait for it: the L2 latency would be exposed on every step)
    double2 rq[4][NC];
    auto ldR = [&](int j, int q) -> double2 {
        const int c = cq_col<NC>(q);
        return (!first && has[q] && j <= c) ? Rs[(size_t)j * CQ_KP + c] : cmk(0.0, 0.0);
    };
#pragma unroll
    for (int q = 0; q < NC; ++q) has[q] = cq_col<NC>(q) < k;
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < NC; ++q) rq[u][q] = ldR(u, q);
    if (threadIdx.x == 0) cq_publish<NB>(sh, 0, b[0], rq[0][0], Rs);
    __syncthreads();
    for (int j0 = 0; j0 < k; j0 += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = j0 + u;
            if (j >= k) break;
            const int buf = j & 1;
            bool act[NC];
            int mask = 0;
#pragma unroll
            for (int q = 0; q < NC; ++q) {
                act[q] = has[q] && cq_col<NC>(q) > j;
                if (__any_sync(0xffffffffu, act[q])) mask |= 1 << q;
            }
            if (mask == 3)
                cq_step<NB, NC, (NC == 2 ? 3 : 1), CH>(b, rq[u], act, sh, buf, Rs, j);
            else if (mask == 2)
                cq_step<NB, NC, (NC == 2 ? 2 : 1), CH>(b, rq[u], act, sh, buf, Rs, j);
            else if (mask == 1)
                cq_step<NB, NC, 1, CH>(b, rq[u], act, sh, buf, Rs, j);
            if (j + 1 < k) {
                int ot, oq;
                cq_owner<NC>(j + 1, ot, oq);
                if ((int)threadIdx.x == ot) {
                    if (NC == 1 || oq == 0)
                        cq_publish<NB>(sh, j + 1, b[0], rq[(u + 1) & 3][0], Rs);
                    else
                        cq_publish<NB>(sh, j + 1, b[NC - 1], rq[(u + 1) & 3][NC - 1], Rs);
                }
            }
#pragma unroll
            for (int q = 0; q < NC; ++q) rq[u][q] = ldR(j + 4, q);
            __syncthreads();
        }
    }
}

// chunk rows [0, fill) of the staging buffer (ld LDB) into the registers of thread t
template <int NB, int NC>
__device__ __forceinline__ void cq_load(double2 (&b)[NC][NB], const double2* Bs, int ldb, int fill, int k) {
#pragma unroll
    for (int q = 0; q < NC; ++q) {
        const int c = cq_col<NC>(q);
#pragma unroll
        for (int i = 0; i < NB; ++i) b[q][i] = (c < k && i < fill) ? Bs[i + (size_t)c * ldb] : cmk(0.0, 0.0);
    }
}

// R (scratch, rows [0, rows)) -> out (rows x k, column-major, ld rows), zero below the diagonal
__device__ inline void cq_store(const double2* Rs, double2* out, int rows, int k) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < rows * k; idx += blockDim.x) {
        const int i = idx % rows, nu = idx / rows;
        out[idx] = (i > nu) ? cmk(0.0, 0.0) : Rs[(size_t)i * CQ_KP + nu];
    }
}

// Basis weights, persistent grid, one pair per CTA at a time (see k_basis for the algorithm:
// leaf with #t > k: R of QR(V_tc); non-leaf: R of QR([R_{t1c1} E_{t1c}; R_{t2c2} E_{t2c}]); a
// stack of <= k rows is the weight itself).
template <int NB, int NC, int CTAS, int NT = 128 / NC>
__global__ void __launch_bounds__(NT, CTAS) k_basis_cq(PlanD P, const int* bps, int nbps, double2* scr) {
    extern __shared__ double2 sm[];
    __shared__ CqRefl<NB> sh;
    constexpr int LDB = NB + 1;
    const int k = P.k, m = P.m;
    double2* Bs = sm;                          // NB x k staging (ld LDB)
    double2* Ef = Bs + (size_t)LDB * k;        // 6 m^2
    double2* Rs = scr + (size_t)blockIdx.x * k * CQ_KP;
    double2 b[NC][NB];
    for (int pi = blockIdx.x; pi < nbps; pi += gridDim.x) {
        const int bp = bps[pi];
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
        __syncthreads();  // previous pair done with Ef / Bs
        if (!leaf) {
            const double2* Eg = P.E + P.bp_E_off[bp];
            for (int idx = threadIdx.x; idx < 6 * m * m; idx += blockDim.x) Ef[idx] = Eg[idx];
        }
        double2* Rout = P.R + P.bp_R_off[bp];
        const int out = P.bp_R_rows[bp];
        int fill = 0, cur = 0;
        bool first = true;
        for (int sidx = 0; sidx < nsrc; ++sidx) {
            const int r = leaf ? total : P.bp_R_rows[src_bp[sidx]];
            const double2* X = leaf ? (P.V + P.bp_V_off[bp]) : (P.R + P.bp_R_off[src_bp[sidx]]);
            for (int i0 = 0; i0 < r;) {
                const int nb = qr ? min(NB - fill, r - i0) : min(NB, r - i0);
                double2* dst = Bs + fill;
                __syncthreads();
                stage_rows(dst, LDB, X, r, i0, nb, k);
                cp_async_wait_all();
                __syncthreads();
                if (!leaf) kron_apply(dst, LDB, nb, m, Ef + sidx * 3 * m * m, false);
                i0 += nb;
                if (!qr) {
                    for (int idx = threadIdx.x; idx < nb * k; idx += blockDim.x)
                        Rout[cur + idx % nb + (size_t)(idx / nb) * out] = Bs[idx % nb + (size_t)(idx / nb) * LDB];
                    cur += nb;
                    continue;
                }
                fill += nb;
                if (fill == NB) {
                    cq_load<NB, NC>(b, Bs, LDB, fill, k);
                    cq_append<NB, NC>(b, Rs, k, first, sh);
                    first = false;
                    fill = 0;
                }
            }
        }
        if (qr && fill > 0) {
            cq_load<NB, NC>(b, Bs, LDB, fill, k);
            cq_append<NB, NC>(b, Rs, k, first, sh);
        }
        if (qr) cq_store(Rs, Rout, k, k);
    }
}

// Chunk rows of the total weights by thread-column FP64 FMAs (qr_cq_tw = 3): thread c forms column c
// of the NB-row chunk w X~ S~ directly in its registers, X~ = the staged rows of R_sc (shared,
// broadcast reads; conjugated when stored conjugated), S~(mu, c) = S_b[c, mu] (or S_b[mu, c] when
// strided), conjugated for the row pass -- one coalesced 16-byte load per mu per thread, NB
// independent accumulators.  X~ S~ with an odd number of conjugations is accumulated as
// x conj(s); conj_x is applied to the sum: sum conj(x) s = conj(sum x conj(s)).
template <int NB, bool XCS>
__device__ __forceinline__ void cq_gemm_cols(double2 (&b)[NB], const double2* Xs, int ldx, const double2* Sg, bool strided,
                                             int k) {
    const int c = threadIdx.x;
#pragma unroll
    for (int i = 0; i < NB; ++i) b[i] = cmk(0.0, 0.0);
    if (c >= k) return;
    const double2* sp = strided ? Sg + (size_t)c * k : Sg + c;
    const size_t ss = strided ? 1 : (size_t)k;
#pragma unroll 2
    for (int mu = 0; mu < k; ++mu) {
        const double2 sv = sp[(size_t)mu * ss];
        const double2* xr = Xs + (size_t)mu * ldx;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            if (XCS)
                cfma_bj(b[i], xr[i], sv);
            else
                cfma(b[i], xr[i], sv);
        }
    }
}

// Total weights, persistent grid (see k_total_weights: the rows of Z_tc^* are w_b R_sc S_b^*
// (row pass; column pass w_b R_tc S_b) for the blocks of the pair, then Zhat_{t+c+} E_{tc+}^* for
// its parents; Zhat_tc = R of their QR, or the rows themselves when there are <= k of them).
template <int NB, int NC, int CTAS, bool TCOL, int NT = 128 / NC>
__global__ void __launch_bounds__(NT, CTAS) k_total_weights_cq(PlanD P, PassD X, bool row, int p0, int np,
                                                                         const int* mirror, double2* scr) {
    extern __shared__ double2 sm[];
    __shared__ CqRefl<NB> sh;
    constexpr int LDB = NB + 1;
    const int k = P.k, m = P.m;
    double2* Bs = sm;                    // NB x k staging (ld LDB)
    double2* Ef = Bs + (size_t)LDB * k;  // 3 m^2
    double2* Rs = scr + (size_t)blockIdx.x * k * CQ_KP;
    double2 b[NC][NB];
    for (int pi = blockIdx.x; pi < np; pi += gridDim.x) {
        const int p = p0 + pi;
        const int zr = X.Z_rows[p];
        double2* Zg = X.Z + X.Z_off[p];
        int total = 0;
        for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
            const int bb = X.blk[ib];
            total += P.bp_R_rows[row ? P.blk_bpcol[bb] : P.blk_bprow[bb]];
        }
        for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) total += X.Z_rows[X.par[ip]];
        const bool qr = total > k;
        int fill = 0, cur = 0;
        bool first = true;
        auto next = [&](int nb) {
            if (!qr) {
                cur += nb;
                return;
            }
            fill += nb;
            if (fill == NB) {
                __syncthreads();
                cq_load<NB, NC>(b, Bs, LDB, fill, k);
                cq_append<NB, NC>(b, Rs, k, first, sh);
                first = false;
                fill = 0;
            }
        };
        for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
            const int bb = X.blk[ib];
            const bool cj = row && P.sym;  // R_sc = conj R_{s,-c} (adjoint symmetry)
            const int obp = row ? (cj ? P.blk_bpcs[bb] : P.blk_bpcol[bb]) : P.blk_bprow[bb];
            const int r = P.bp_R_rows[obp];
            const double2* Ro = P.R + P.bp_R_off[obp];
            const double w = P.omega[bb];
            const int mb = row ? bb : mirror[bb];
            const double2* Sg = P.S + (size_t)P.blk_slot[mb >= 0 ? mb : bb] * k * k;
            const bool strided = !row && mb < 0;
            if (qr && TCOL) {
                // chunks of one block only (the last one zero-padded: zero rows change no norm or dot
                // product), formed in the registers by cq_gemm_cols and appended at once
                if (fill > 0) {  // (rows of an earlier source pending)
                    __syncthreads();
                    cq_load<NB, NC>(b, Bs, LDB, fill, k);
                    cq_append<NB, NC>(b, Rs, k, first, sh);
                    first = false;
                    fill = 0;
                }
                const bool xcs = row != cj;  // S conjugated XOR X stored conjugated
                for (int i0 = 0; i0 < r; i0 += NB) {
                    const int nb = min(NB, r - i0);
                    __syncthreads();
                    stage_rows(Bs, LDB, Ro, r, i0, nb, k);
                    for (int idx = threadIdx.x; idx < (NB - nb) * k; idx += blockDim.x)
                        Bs[nb + idx % (NB - nb) + (size_t)(idx / (NB - nb)) * LDB] = cmk(0.0, 0.0);
                    cp_async_wait_all();
                    __syncthreads();
                    if (xcs)
                        cq_gemm_cols<NB, true>(b[0], Bs, LDB, Sg, strided, k);
                    else
                        cq_gemm_cols<NB, false>(b[0], Bs, LDB, Sg, strided, k);
#pragma unroll
                    for (int i = 0; i < NB; ++i) b[0][i] = cj ? cmk(w * b[0][i].x, -w * b[0][i].y) : cscale(b[0][i], w);
                    cq_append<NB, NC>(b, Rs, k, first, sh);
                    first = false;
                }
                continue;
            }
            for (int i0 = 0; i0 < r;) {
                const int nb = qr ? min(NB - fill, r - i0) : min(NB, r - i0);
                double2* dst = qr ? Bs + fill : Zg + cur;
                const int ldd = qr ? LDB : zr;
                __syncthreads();
                chunk_gemm_S_dmma<true>(Ro, r, i0, nb, Sg, row, strided, w, k, dst, ldd, cj);  // FP64 tensor cores
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
                const int nb = qr ? min(NB - fill, r - i0) : min(NB, r - i0);
                double2* dst = Bs + (qr ? fill : 0);
                __syncthreads();
                stage_rows(dst, LDB, Zp, r, i0, nb, k);
                cp_async_wait_all();
                __syncthreads();
                kron_apply(dst, LDB, nb, m, Ef, true);  // Zhat_{t+c+} E_{tc+}^*
                if (!qr)
                    for (int idx = threadIdx.x; idx < nb * k; idx += blockDim.x)
                        Zg[cur + idx % nb + (size_t)(idx / nb) * zr] = Bs[idx % nb + (size_t)(idx / nb) * LDB];
                i0 += nb;
                next(nb);
            }
        }
        if (qr && fill > 0) {
            __syncthreads();
            cq_load<NB, NC>(b, Bs, LDB, fill, k);
            cq_append<NB, NC>(b, Rs, k, first, sh);
        }
        if (qr) cq_store(Rs, Zg, zr, k);
    }
}

// Variants (dh2_set_option "qr_cq" for the basis weights, "qr_cq_tw" for the total weights):
// 1 = NB 16 rows at 4 CTAs per SM (128 registers; default), 2 = NB 24 at 3 (168 registers).
// 3 = total weights with thread-column chunk rows (cq_gemm_cols).  Measured on C4 (k = 125):
// basis weights 3.1 s (cta_qr_append) -> 1.8 s (1) / 2.14 s (2: the 128-row stacks of the level
// above the leaves fill 6 chunks of 24 = 144 rows); total weights: the CTA-cooperative kernel
// stays above the leaves (its 48-row DMMA chunks read S_b three times per 125-row block; the
// thread-column rows of 16-row chunks eight times: +9 %), variant 3 runs the leaf levels (blocks
// of 64-row leaf weights: C4 1.36 -> 1.24 s, C5 1.91 -> 1.81 s).
// Microbenchmark (tools/cq_bench.cu, k = 125, appends only): 2: 9.96 TF/s, 1: 9.07, NB 32 at 2 CTAs
// 8.58, NB 8 at 4 CTAs 6.57; two columns per thread (t, 127 - t) at NB 8 / 8 CTAs: 6.3.
constexpr int CQ_MAX_CTAS = 8;
size_t cq_scratch_elems(const PlanD& P) { return (size_t)P.num_sms * CQ_MAX_CTAS * P.k * CQ_KP; }

static size_t cq_smem(const PlanD& P, int NB, int nE) {
    return ((size_t)(NB + 1) * P.k + (size_t)nE * P.m * P.m) * sizeof(double2);
}

template <int NB, int NC, int CTAS, int NT = 128 / NC>
static void cq_basis(const PlanD& P, const int* bps, int nbps, cudaStream_t s) {
    static_assert(CTAS <= CQ_MAX_CTAS, "scratch");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_basis_cq<NB, NC, CTAS, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
    }
    const int grid = std::min(nbps, P.num_sms * CTAS);
    k_basis_cq<NB, NC, CTAS, NT><<<grid, NT, cq_smem(P, NB, 6), s>>>(P, bps, nbps, P.cq_scr);
}

template <int NB, int NC, int CTAS, bool TCOL, int NT = 128 / NC>
static void cq_total(const PlanD& P, const PassD& X, bool row, int p0, int np, const int* mirror, cudaStream_t s) {
    static_assert(CTAS <= CQ_MAX_CTAS, "scratch");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_total_weights_cq<NB, NC, CTAS, TCOL, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
    }
    const int grid = std::min(np, P.num_sms * CTAS);
    k_total_weights_cq<NB, NC, CTAS, TCOL, NT><<<grid, NT, cq_smem(P, NB, 3), s>>>(P, X, row, p0, np, mirror, P.cq_scr);
}

void launch_basis_cq(const PlanD& P, const int* bps, int nbps, cudaStream_t s) {
    if (!nbps) return;
    if (P.k <= 64) {  // (k = 64: 64 threads, one column each, 8 pairs per SM)
        cq_basis<16, 1, 8, 64>(P, bps, nbps, s);
        return;
    }
    switch (P.qr_cq) {
        case 2: cq_basis<24, 1, 3>(P, bps, nbps, s); break;
        default: cq_basis<16, 1, 4>(P, bps, nbps, s); break;
    }
}

void launch_total_weights_cq(const PlanD& P, bool row, int p0, int np, const int* mirror, cudaStream_t s, int variant) {
    if (!np) return;
    const PassD& X = row ? P.row : P.col;
    if (P.k <= 64) {
        if (variant == 3)
            cq_total<16, 1, 8, true, 64>(P, X, row, p0, np, mirror, s);
        else
            cq_total<16, 1, 8, false, 64>(P, X, row, p0, np, mirror, s);
        return;
    }
    switch (variant) {
        case 2: cq_total<24, 1, 3, false>(P, X, row, p0, np, mirror, s); break;
        case 3: cq_total<16, 1, 4, true>(P, X, row, p0, np, mirror, s); break;
        default: cq_total<16, 1, 4, false>(P, X, row, p0, np, mirror, s); break;
    }
}

}  // namespace dh2
