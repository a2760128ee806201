/*
 * dh2.h — C ABI of libdh2.so: B200-native hybrid recompression of directional
 * H^2-matrices (DH^2), arXiv 1809.04384 (the paper's text is PAPER.md).
 *
 * Citations are PAPER.md line numbers (P:<line>) plus the section/equation.
 *
 * Problem (Eq. helmholtz/matrix): Galerkin matrix of the Helmholtz single
 * layer potential g(x,y) = exp(i kappa |x-y|)/(4 pi |x-y|) with piecewise-constant
 * basis functions on a flat triangle mesh.  dh2_build_interp builds
 * the DH^2 approximation of its far field by directional Chebyshev interpolation
 * (Eq. 4, Eq. 10/11, Def. 2.7); dh2_recompress
 * replaces the interpolation bases by orthogonal, nested, adaptively truncated
 * ones (§3.2) and projects the couplings.  The
 * nearfield (inadmissible leaves) is untouched by the recompression; it is assembled on
 * request by dh2_nearfield_assemble (NEXT-4) and added by dh2_matvec(DH2_ADD_NEAR).
 *
 * Conventions (all functions):
 *   - return int: 0 = DH2_OK, < 0 = error code below; no C++ exception crosses the ABI;
 *     dh2_last_error(ctx) returns a message for the last failing call on ctx
 *     (dh2_last_error(NULL) for failures before a context exists).
 *   - complex values are interleaved (re, im) float64; matrices are column-major.
 *   - vectors x, y are in the ORIGINAL triangle order; the cluster permutation is internal.
 *   - input buffers are copied during the call; the caller keeps ownership and may
 *     free them after return.  Output buffers are caller-owned.
 *   - a context owns all its device memory and is not thread-safe; distinct
 *     contexts are independent.  All work is issued on the context's stream
 *     (dh2_set_stream) and every API call synchronises that stream before return
 *     unless stated otherwise.
 *   - there is no CPU fallback: without a CUDA device every compute call fails
 *     with DH2_ECUDA.
 */
#ifndef DH2_H
#define DH2_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    DH2_OK = 0,
    DH2_EINVAL = -1,    /* bad parameter, bad mesh index, triangle area <= 0, size mismatch */
    DH2_ENOMEM = -2,    /* the device memory plan does not fit (checked before any launch) */
    DH2_ECUDA = -3,     /* CUDA runtime error or no device */
    DH2_ENCCL = -4,     /* multi-GPU transport (NCCL) error or NCCL unavailable */
    DH2_ESTATE = -5,    /* call order: recompress before build, RECOMP matvec before recompress */
    DH2_EMISMATCH = -6, /* ranks of a multi-GPU context passed different arguments (parameter hash, all-reduced) */
    DH2_ENOTIMPL = -7,  /* configuration outside what this build supports (e.g. m > 5, k > 125) */
    DH2_ENUMERIC = -8   /* numerical failure: non-finite singular values, or a one-sided Jacobi SVD that did
                           not converge in 60 sweeps (the factors of that recompression are not used) */
};

/* recompression error-control modes (reading Q12 of DESIGN.md) */
enum {
    DH2_FROB_BLOCKREL = 0,   /* w_b = 1/||G_b||_F, k_tc = min{k : sum_{i>k} s_i^2 <= eps^2} (default) */
    DH2_FROB_CLUSTERREL = 1, /* w_b = 1, k_tc = min{k : sum_{i>k} s_i^2 <= eps^2 sum_i s_i^2} */
    DH2_SPEC_BLOCKREL = 2    /* w_b = 1/||G_b||_F, k_tc = min{k : s_{k+1} <= eps} */
};

/* which matrix: the interpolation DH^2 (V, E, S) or the recompressed one (Q, F, S~) */
enum { DH2_ORIG = 0, DH2_RECOMP = 1 };

/* matvec flags */
enum { DH2_HOST_PTRS = 0, DH2_DEVICE_PTRS = 1, DH2_ADD_NEAR = 2 /* y += N x (assembled nearfield) */ };

typedef struct dh2_ctx dh2_ctx; /* opaque; owns all device memory */

/* Triangle mesh.  xyz: nv*3 float64 row-major vertex coordinates;
 * tri: nt*3 int64 0-based vertex indices.  DoF i = triangle i. */
typedef struct {
    int64_t nv, nt;
    const double* xyz;
    const int64_t* tri;
} dh2_mesh;

/* Parameters (BASELINE.json configs).
 *   kappa     wave number >= 0 (Eq. helmholtz)
 *   m         Chebyshev order per axis, k = m^3; this build supports 1 <= m <= 5
 *   leaf_size clusters are split while #t > leaf_size
 *   eta1      direction parameter of Eq. 3a / Remark 2.4
 *   eta2      admissibility parameter of Eq. 3b/3c
 *   quad      triangle quadrature points for V (must be 7: Radon's degree-5 rule) */
typedef struct {
    double kappa;
    int32_t m;
    int32_t leaf_size;
    double eta1, eta2;
    int32_t quad;
} dh2_params;

/* Device selection and multi-GPU description (NULL = device 0, one shard).
 *   device   CUDA ordinal, or DH2_DEVICE_NONE: build the host structures only (cluster
 *            tree, directions, blocks, pairs, shard ownership and exchange lists — no
 *            device memory, no kernels); such a context supports dh2_export of host arrays
 *            and dh2_storage(DH2_ORIG) and fails every compute call with DH2_ESTATE.  It
 *            exists so structure parity can be checked without a GPU; it is not a compute
 *            fallback.
 *   world    number of shards P (a power of two).  The partition: cut level
 *            log2 P of the cluster tree; shard r owns the subtree of the r-th cluster on that
 *            level, i.e. its row/column pairs and every block (t,s,c) whose row cluster t it
 *            owns.  Every active level must lie on or below the cut (DH2_ENOTIMPL otherwise),
 *            and the structure must admit the adjoint symmetry (W = V, antipodal directions).
 *            Exchanges: after the basis weights the R_sc computed by QR of column pairs that
 *            other shards' blocks reference, after the truncation C'_sc and k'_sc, in the
 *            matvec the coefficients xh'_sc, then the output slices.  Results are bitwise
 *            identical for every P.
 *   rank     this process's shard, 0 <= rank < world.
 *   nccl_uid 128-byte ncclUniqueId from dh2_nccl_unique_id on rank 0, broadcast by the
 *            caller: one process per GPU, exchanges with NCCL over NVLink, every call is
 *            collective.  NULL with world > 1: "virtual" mode — this process runs all
 *            `world` shards on `device`, phase by phase, with device-to-device exchanges
 *            (same shard code and exchange items; used to test the partition on one GPU). */
enum { DH2_DEVICE_NONE = -1 };
typedef struct {
    int32_t rank, world;
    const void* nccl_uid;
    int32_t device;
} dh2_dist;

/* Build the interpolation DH^2 matrix (§2).  Host: cluster tree (Def. 2.1, median
 * split on the longest axis of the tight box), directions D_l (Remark 2.4) and sd_l
 * (P:323-330), block tree (Def. 2.5, Eq. 3), row/column pair closure.  Device
 * (sm_100a kernels): quadrature points, Chebyshev grids, leaf bases V_tc,
 * transfer factors E_{t'c} (Eq. 10, Kronecker-factored), couplings S_b.
 * On success *out receives a new context; on failure *out is NULL. */
int dh2_build_interp(const dh2_mesh* mesh, const dh2_params* params, const dh2_dist* dist, dh2_ctx** out);

/* Re-run only the device set-up kernels of dh2_build_interp on the resident
 * structure (used to time the device part of the whole path). */
int dh2_setup_device(dh2_ctx* ctx);

/* Hybrid recompression (§3.2; Lemma Projections) with
 * accuracy eps >= 0 and error-control mode.  Phases: basis weights (Eq. 18),
 * block weights, total weights row/col (Eq. 17), truncation row/col (Eq. 19),
 * projection S~_b = C_tc S_b C'_sc^*.  May be called repeatedly (it recomputes
 * from the interpolation matrix). */
int dh2_recompress(dh2_ctx* ctx, double eps, int32_t mode);

/* Matrix-vector product y = G_far x of the ORIG or RECOMP matrix (the admissible blocks), plus
 * the nearfield N x with DH2_ADD_NEAR.  ORIG needs V and S resident: DH2_ENOTIMPL on the
 * memory-lean plan (dh2_get_stats "lean").
 * x, y: n complex (2n float64) in original triangle order; host pointers
 * (flags = DH2_HOST_PTRS, copied through the context's stream) or device
 * pointers (DH2_DEVICE_PTRS, no copies).  Without DH2_ADD_NEAR the result is the far field
 * only; with DH2_ADD_NEAR (after dh2_nearfield_assemble) it is the whole Galerkin product
 * G x = G_far x + N x.  DH2_ESTATE if DH2_ADD_NEAR is set before the nearfield is assembled. */
int dh2_matvec(dh2_ctx* ctx, int32_t which, const double* x, double* y, int32_t flags);

/* Nearfield assembly (NEXT-4; Section 5): every inadmissible leaf (t, s) of
 * the block tree (export "near", sorted by (t, s)) is stored as a dense #t x #s block, column-major,
 * rows and columns in cluster order, entries the Galerkin integrals
 *     g_ij = int_{tau_i} int_{tau_j} exp(i kappa |x-y|) / (4 pi |x-y|) dy dx
 * of the piecewise-constant basis: Sauter-Erichsen-Schwab quadrature of order nq_singular (paper:
 * 5) on [0,1]^4 for identical, edge- and vertex-adjacent triangles, Gauss quadrature with the Duffy
 * transformation of order nq_regular (paper: 3) per axis otherwise.  Orders in 1..8 (DH2_EINVAL
 * otherwise).  Device memory: 16 B per coefficient (dh2_storage's nearfield_bytes), owned by ctx;
 * a second call re-assembles.  Shards assemble the blocks of the row leaves they own.  Exports:
 * "near_values" (complex, the blocks concatenated in "near" order), "near_off" (int64 entry offset
 * per block).  Collective with world > 1. */
int dh2_nearfield_assemble(dh2_ctx* ctx, int32_t nq_singular, int32_t nq_regular);

/* Storage report, 16 B per complex coefficient, 1 KB = 1024 B.
 * basis = leaf matrices + transfers of the row and the column basis;
 * matrix = basis + couplings + nearfield (nearfield counted from block sizes). */
typedef struct {
    int64_t n;
    double row_basis_bytes, col_basis_bytes, coupling_bytes, nearfield_bytes;
    double kb_per_dof_basis, kb_per_dof_matrix;
    int32_t max_rank;
    double mean_rank;
} dh2_storage_report;
int dh2_storage(const dh2_ctx* ctx, int32_t which, dh2_storage_report* out);

/* Set the CUDA stream (cudaStream_t) all work of ctx is issued on; NULL = the
 * context's own stream.  The caller keeps ownership of the stream. */
int dh2_set_stream(dh2_ctx* ctx, void* cuda_stream);

/* Options (take effect at the next dh2_recompress):
 *   "adjoint_symmetry" (0 | 1, default 1): derive the column pass from the row pass.  For the
 *     single-layer operator W = V and, with antipodal direction sets (DESIGN
 *     readings R2/R4), V_{s,-c} = conj(V_{s,c}) and S_{(s,t,-c)} = S_{(t,s,c)}^T, so the
 *     column-pass matrices of (s,c) are the complex conjugates of the row-pass
 *     matrices of (s,-c): Zhat', sigma', k', Q', F', C' follow by conjugation.  Used only if
 *     dh2_build_interp verified that correspondence on the whole structure (stats key
 *     "adjoint_symmetry"); otherwise, or with value 0, both passes run.
 *   "truncate_workspace" (0 | 1, default 0): force the global-workspace truncation kernel.
 *   "truncate_split" (0 | 1, default 1): leaf levels with #t <= 32 truncate in three kernels
 *     (pivoted QR, warp-level one-sided Jacobi, epilogue) instead of one CTA per pair.
 *   "fuse_leaf_weights" (0 | 1, default 0): on those leaf levels (k <= 64) fold the total
 *     weights into the truncation's QR kernel: the rows of the stack whose R factor is Zhat_tc
 *     are multiplied by V_tc^* and reduced directly, Zhat_tc is never formed (stats
 *     "fused_leaf_levels_row/col"; export "Z" is not defined on those levels).
 *   "fuse_direct_rows" (0..64, default 64): fused stacks up to this height form M^* directly,
 *     taller ones are reduced by Householder appends (stats "fused_append_pairs").
 *   "truncate_split64" (0 | 1, default 1): leaf levels with 32 < #t <= 64 truncate in two kernels
 *     (prologue + pivoted QR; one-sided Jacobi + epilogue at three pairs per SM); bitwise equal.
 *   "truncate_split64_inner" (0 | 1, default 1): the same for inner levels (k > 64, <= 64 rows).
 *   "trunc64_threads" (64 | 128 | 256, default 128): threads of that Jacobi + epilogue kernel.
 *   "qr_cq" (0..2, default 1): k > 64 basis weights by column-per-thread Householder appends
 *     (thread c holds column c of a 16-row (1) or 24-row (2) chunk in registers); 0: CTA-cooperative.
 *   "qr_cq_tw" (0..3, default 0), "qr_cq_tw_leaf" (0..3, default 3): the same for the total
 *     weights above / at the leaf levels (3: chunk rows formed by thread-column FMAs).
 *   "near_tma" (0 | 1, default 1): nearfield matvec streams the blocks N_b through a ring of
 *     shared-memory stages filled by cp.async.bulk (TMA) on mbarriers; 0: direct global loads.
 *   "mv_forward_warp" (0 | 1 | 2, default 2): launch shapes of the far-field matvec.  1: leaf forward
 *     transform with one warp per coefficient (coalesced column reads, shuffle reduction), coupling
 *     and backward steps with 16 lanes per pair (RECOMP); 2: also one warp per pair, four pairs per
 *     CTA, in the forward transform (RECOMP); 0: a thread per coefficient and a CTA per pair.
 *   Further A/B switches (qr_wy, qr_flag, trunc_direct, lean_chunks) are listed in DESIGN.md §8.
 *   All variants give the same ranks, singular values and matrices up to rounding (tests).
 * Errors: DH2_EINVAL for an unknown name or value. */
int dh2_set_option(dh2_ctx* ctx, const char* name, int64_t value);

/* Profiling: when enabled, every kernel class is bracketed by CUDA events on the
 * context's stream; dh2_get_stats then reports per-class device time. */
int dh2_set_profiling(dh2_ctx* ctx, int32_t enable);

/* Statistics as a JSON document (two-call pattern: buf = NULL returns the size in
 * *len).  Keys: n, structure counts, per kernel class {launches, ms, flops, bytes},
 * certified E_row, E_col, ||G_far||_F^2 (after recompress), kernel launch count. */
int dh2_get_stats(const dh2_ctx* ctx, char* buf, int64_t* len);

/* Introspection for parity tests (two-call pattern): copy the named array into
 * buf (nbytes = size of buf; buf = NULL returns the size in *nbytes).  Names and
 * layouts are listed in DESIGN.md §"Export names" (structure arrays, offsets,
 * and the device pools V, E, S, R, omega, Zhat_row/col, rank_row/col,
 * sigma_row/col, Q_row/col, F_row/col, C_row/col, St).  "<name>@<offset>:<count>"
 * exports the element slice [offset, offset + count) of the array. */
int dh2_export(const dh2_ctx* ctx, const char* name, void* buf, int64_t* nbytes);

/* As dh2_export, for shard `shard` (0 <= shard < number of shards in this process; > 1 only
 * in the virtual mode).  Extra names of the partition: "owner" (int32 per cluster, -1 above
 * the cut), "own_range" (int32 b_lo, b_hi, pos_lo, pos_hi: own blocks and cluster-ordered positions),
 * "xR_send", "xR_recv", "xC_send", "xC_recv" (int32: for every peer, a count then the item
 * ids: basis pair ids for R, column pair ids for C', k', xh'). */
int dh2_export_shard(const dh2_ctx* ctx, int32_t shard, const char* name, void* buf, int64_t* nbytes);

/* Write a fresh 128-byte ncclUniqueId to uid (call on rank 0, broadcast to all ranks before
 * dh2_build_interp).  NCCL (libnccl.so.2) is loaded at run time; DH2_ENCCL if unavailable. */
int dh2_nccl_unique_id(void* uid);

/* Release all memory of ctx (NULL is a no-op). */
int dh2_destroy(dh2_ctx* ctx);

/* Message of the last failing call on ctx (or of the last failure without a context). */
const char* dh2_last_error(const dh2_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DH2_H */
