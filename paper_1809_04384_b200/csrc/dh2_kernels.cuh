// Kernel declarations and the device-side plan shared by dh2_kernels.cu and dh2_api.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dh2_device.cuh"

namespace dh2 {

// Per-pass (row basis or column basis) device tables; "pair" = active (t,c) of that pass.
struct PassD {
    int npairs;
    const int* bp;        // pair -> basis pair id
    const int* child0;    // pair -> pass-local child pair (t1, sd c), -1 at leaves
    const int* child1;
    const int64_t* Z_off; // Zhat slab offset (double2 units), Zhat is Zrows x k, ld = Zrows
    const int* Z_rows;    // r_Z = min(#rows of Z^*, k)
    const int* blk_ptr;   // CSR: contributing admissible blocks of the pair
    const int* blk;
    const int* par_ptr;   // CSR: parent pairs (t+, c+) with sd(c+) = c
    const int* par;       // parent pass-local pair id
    const int* par_child; // which child of t+ the pair's cluster is (selects E factor)
    const int* rowsb;     // bound on #rows of the truncated matrix (leaf #t, else kb1 + kb2)
    const int* kb;        // bound on the new rank, min(rowsb, r_Z)
    const int64_t* C_off; // C slab, kb x k, ld kb
    const int64_t* Q_off; // leaf: Q (#t x kb, ld #t); non-leaf: Qhat = [F1; F2] (rowsb x kb, ld rowsb)
    const int64_t* sig_off;  // singular values, min(rowsb, r_Z) doubles
    double2* Z;
    double2* C;
    double2* Q;
    double* sigma;
    int* rank;
    int* nsig;            // number of singular values computed
    double* disc;         // discarded sum of squares per pair
    int* sweeps;          // Jacobi sweeps used per pair (diagnostics / executed-flop model)
};

struct PlanD {
    int n, m, k, nclusters;
    int smem_optin;       // opt-in dynamic shared memory per CTA (bytes), minus a static-smem margin
    int num_sms;
    int col_conj;         // 1: column factors C', Q' are stored as the row factors at -c (read conjugated)
    int qr_wy;            // 1: chunk appends of <= 32 rows in the blocked compact-WY form (dh2_set_option "qr_wy", default 0)
    int qr_flag;          // 1: chunk appends synchronised by per-reflection flags instead of block barriers ("qr_flag")
    int trunc_mode;       // 1: leaf truncation on M^* directly, never by streamed appends ("trunc_direct")
    int qr_cq;            // != 0: k > 64 basis weights by column-per-thread appends (dh2_cq.cu; "qr_cq" = variant)
    int qr_cq_tw;         // != 0: the same for the total weights ("qr_cq_tw")
    int qr_cq_tw_leaf;    // variant at leaf levels ("qr_cq_tw_leaf", default 3: thread-column chunk rows)
    int qr_cq64, qr_cq64_tw;  // k <= 64: the column-per-thread basis / total weights ("qr_cq64", "qr_cq64_tw": 0, 1, 3)
    double2* cq_scr;      // their scratch triangles (cq_scratch_elems), null when unused
    int mv_fwd_warp;      // leaf forward transform of the matvec: 1 = one warp per coefficient, coalesced ("mv_forward_warp")
    int bw_variant;       // block weights at k > 64: 1 = unrolled S loads + register-blocked norm GEMM ("bw_variant")
    int t64_threads;      // threads of the Jacobi + epilogue kernel of the wide split leaf truncation ("trunc64_threads")
    int sym;              // 1: only row basis pairs have V/R/E; the column side of a block (t,s,c) reads
                          //    the row basis pair (s,-c) conjugated (blk_bpcs; matvec: col2row)
    const int* col2row;   // column pair (s,c) -> row pair (s,-c) (adjoint-symmetric structures)
    double kappa;
    // geometry
    const double* xyz;
    const int64_t* tri;
    const int64_t* perm;
    double4* qp;  // n*7 quadrature points (x, y, z, |tau| w) in cluster order
    const double* c_lo;
    const double* c_hi;
    const int64_t* c_begin;
    const int* c_size;
    GridD* grid;
    const double* dirs;  // all directions, 3 doubles each (global index)
    // basis pairs
    int nbp;
    const int* bp_t;
    const int* bp_dir;      // global direction index of c
    const int* bp_sddir;    // global direction index of sd(c) (children's direction), -1 at leaves
    const int* bp_child0;
    const int* bp_child1;
    const int64_t* bp_V_off;  // leaf V slab (#t x k, ld #t), -1 for non-leaf
    const int64_t* bp_R_off;  // basis weight slab (Rrows x k, ld Rrows)
    const int* bp_R_rows;
    const int64_t* bp_E_off;  // 2 * 3 m^2 complex transfer factors, -1 at leaves
    double2* V;
    double2* R;
    double2* E;
    // blocks
    int nblk;
    const int* blk_t;
    const int* blk_s;
    const int* blk_dir;
    const int* blk_bprow;
    const int* blk_bpcol;
    const int* blk_bpcs;  // basis pair id of (s,-c)
    const int* blk_prow;  // row-pass pair id of (t,c)
    const int* blk_pcol;  // col-pass pair id of (s,c)
    const int64_t* blk_St_off;  // kb_row x kb_col slab, ld kb_row
    const int* blk_slot;  // slot of block b in S (full plan: b - b_lo; lean plan: position in its chunk)
    double2* S;           // slots * k * k
    double2* St;
    double* omega;
    double* normG2;
    PassD row, col;
};

// setup (Eq. 10)
void launch_quad(const PlanD& P, cudaStream_t s);
void launch_grid(const PlanD& P, cudaStream_t s);
void launch_leafV(const PlanD& P, const int* bps, int nbps, int maxrows, cudaStream_t s);
void launch_E(const PlanD& P, const int* bps, int nbps, cudaStream_t s);
void launch_S(const PlanD& P, int b0, int nb, cudaStream_t s, const int* blist = nullptr);
// recompression (§3.2)
void launch_basis(const PlanD& P, const int* bps, int nbps, int maxrows, cudaStream_t s);
void launch_block_weights(const PlanD& P, int b0, int nb, int mode, const int* mirror, cudaStream_t s,
                          const int* blist = nullptr);
// leaf_level: every pair of the launch is a leaf (k > 64: the thread-column form, qr_cq_tw_leaf)
void launch_total_weights(const PlanD& P, bool row, int p0, int np, const int* mirror, cudaStream_t s, bool leaf_level = false);
// column-per-thread chunk appends (k in (64, 128]; dh2_cq.cu), persistent grid on P.cq_scr
size_t cq_scratch_elems(const PlanD& P);
inline size_t cq_scratch_bytes_bound(int k) { return k <= 128 ? (size_t)160 * 8 * k * 128 * 16 : 0; }
void launch_basis_cq(const PlanD& P, const int* bps, int nbps, cudaStream_t s);
void launch_total_weights_cq(const PlanD& P, bool row, int p0, int np, const int* mirror, cudaStream_t s, int variant);
struct TruncLaunch {
    int ldv = 1, ldb = 1, grid = 0;
    bool use_ws = false;      // working set in a global workspace (persistent grid) instead of smem
    bool append = false;      // leaf level with zr > #t: M^* reduced to its R factor by streamed chunks
    size_t smem = 0;          // dynamic shared memory per CTA
    size_t ws_stride = 0;     // workspace per CTA (double2 units); total grid * ws_stride
    int threads = 128;        // CTA size: more threads per pair when shared memory limits the CTAs per SM
};
TruncLaunch plan_truncate(const PlanD& P, int np, int maxrowsM, int maxZrows, bool leaf_level, bool force_ws);
// plist (optional): the pairs to truncate (np of them) instead of [p0, p0 + np) -- levels mixing
// leaf and inner clusters are truncated in one launch per kind
void launch_truncate(const PlanD& P, bool row, int p0, int np, const TruncLaunch& L, bool leaf_level, double eps,
                     int mode, double2* ws, cudaStream_t s, const int* plist = nullptr);
// leaf levels with #t <= 32: pivoted QR per CTA, register-resident warp Jacobi, epilogue
size_t trunc_split_scratch_bytes(int np);
// leaf levels with 32 < #t <= 64 (C4/C5): prologue + pivoted QR (one CTA per SM), then Jacobi +
// epilogue with R alone in shared memory (three pairs per SM)
// (levels above the leaves with k1 + k2 <= 64 rows: the same split, Vhat kept in the scratch)
size_t trunc_split64_scratch_bytes(int np, bool leaf, int k);
void launch_truncate_split64(const PlanD& P, bool row, int p0, int np, const TruncLaunch& L, bool leaf_level, double eps,
                             int mode, void* scratch, cudaStream_t s);
// fused: leaf total weights folded into the QR kernel (k_trunc_zqr, k <= 64; the level's Zhat is
// not formed; stacks of <= fuse_direct rows form M^* directly, taller ones are QR-appended;
// mirror as for launch_total_weights)
void launch_truncate_split(const PlanD& P, bool row, int p0, int np, const TruncLaunch& L, double eps, int mode,
                           void* scratch, bool fused, int fuse_direct, const int* mirror, cudaStream_t s);
// fused leaf total weights + truncation for leaves of <= 64 triangles, any k (one CTA per pair does
// everything: stack x V^* appended into a #t x #t triangle, pivoted QR, Jacobi, epilogue)
size_t trunc_fused_smem(const PlanD& P, int maxrows);
void launch_truncate_fused(const PlanD& P, bool row, int p0, int np, int maxrows, double eps, int mode, const int* mirror,
                           cudaStream_t s);
void launch_mirror_pass(const PlanD& P, const int* col2row, int p0, int np, cudaStream_t s);
void launch_project(const PlanD& P, int b0, int nb, int maxkrow, const int* mirror, cudaStream_t s,
                    const int* blist = nullptr);
// matvec (forward / coupling / backward)
void launch_mv_forward(const PlanD& P, bool recomp, int p0, int np, const double2* xp, double2* xh,
                       cudaStream_t s);
void launch_mv_couple(const PlanD& P, bool recomp, int p0, int np, const double2* xh, double2* yh, cudaStream_t s);
void launch_mv_backward(const PlanD& P, bool recomp, int p0, int np, double2* yh, cudaStream_t s);
void launch_mv_leaf_out(const PlanD& P, bool recomp, const int* lc, const int* lc_ptr, int g0, int nlc, const double2* yh,
                        double2* yp, cudaStream_t s);
// exchange packing / unpacking (multi-GPU sharding)
void launch_copy_segments(const double2* src, double2* dst, const int64_t* soff, const int64_t* doff, const int64_t* len,
                          int nseg, cudaStream_t s);
void launch_copy_segments_i(const int* src, int* dst, const int64_t* soff, const int64_t* doff, const int64_t* len,
                            int nseg, cudaStream_t s);
void launch_permute(const int64_t* perm, const double2* in, double2* out, int n, bool gather, cudaStream_t s);
void launch_copy_mat(const double2* src, double2* dst, const int64_t* soff, const int64_t* doff, const int* rows,
                     const int* cols, const int* lds, int n, cudaStream_t s);

}  // namespace dh2
