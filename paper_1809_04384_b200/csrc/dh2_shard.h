// Host-side context of one shard of a DH^2 matrix (shared by dh2_api.cu and dh2_lean.cu):
// error types, device buffers, per-pass host tables and the Shard itself.
#pragma once
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "dh2_host.h"
#include "dh2_kernels.cuh"

namespace dh2 {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NotImpl : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NoMem : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct MismatchError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                          \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));       \
    } while (0)

// Device memory comes from the device's stream-ordered pool, which keeps freed memory reserved
// (release threshold = max): a new context in the same process reuses it instead of paying
// cudaMalloc/cudaFree of many GB again.  Allocation and release are ordered on the legacy stream
// and completed before use; every context synchronises its streams before it frees.
inline void pool_setup(int dev) {
    static int done_dev = -1;
    if (done_dev == dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_dev = dev;
}
// bytes the pool holds in reserve (freed by earlier contexts), usable by a new plan
inline size_t pool_reusable(int dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return 0;
    uint64_t res = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &res);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    return res > used ? (size_t)(res - used) : 0;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void alloc(size_t cnt) {
        free();
        n = cnt;
        if (cnt) {
            CK(cudaMallocAsync(reinterpret_cast<void**>(&p), cnt * sizeof(T), 0));
            CK(cudaStreamSynchronize(0));
        }
    }
    void upload(const std::vector<T>& v, cudaStream_t s) {
        alloc(v.size());
        if (n) CK(cudaMemcpyAsync(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void free() {
        if (p) cudaFreeAsync(p, 0);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { free(); }
};

struct PassH {
    std::vector<int> bp, child0, child1, Z_rows, blk_ptr, blk, par_ptr, par, par_child, rowsb, kb;
    std::vector<int64_t> Z_off, C_off, Q_off, sig_off;  // active offsets (column pass: aliases, see below)
    // column pass of an adjoint-symmetric structure: C', Q', sigma' of an own pair are read as the
    // conjugate of the row results at (s,-c) in the row pools (no copies); imported C' of the
    // partition sit after the row C pool.  *_own: compact offsets of a separate column storage
    // (used when two passes are requested).
    bool alias = false;
    std::vector<int64_t> C_off_own, Q_off_own, sig_off_own, C_off_alias, Q_off_alias, sig_off_alias;
    int64_t C_imp_total = 0, C_extra = 0;
    std::vector<int> lev_ptr;  // pairs of level l: [lev_ptr[l], lev_ptr[l+1])
    std::vector<int> lc, lc_ptr;  // leaf-cluster groups (matvec output)
    std::vector<int> bp2p;        // basis pair id -> pair id of this pass (-1 if absent)
    std::vector<int> own_lo, own_hi;  // per level: pairs of this shard [own_lo[l], own_hi[l])
    int lc_lo = 0, lc_hi = 0;         // leaf-cluster groups of this shard
    int64_t Z_total = 0, C_total = 0, Q_total = 0, sig_total = 0;
    int max_total_rows_level(int l) const { return lev_max_total[l]; }
    std::vector<int> lev_max_total, lev_max_zrows, lev_max_leafrows;
    std::vector<int> total_rows;
    // device
    DevBuf<int> d_bp, d_child0, d_child1, d_Z_rows, d_blk_ptr, d_blk, d_par_ptr, d_par, d_par_child, d_rowsb, d_kb,
        d_rank, d_nsig, d_lc, d_lc_ptr, d_sweeps;
    DevBuf<int64_t> d_Z_off, d_C_off, d_Q_off, d_sig_off;
    DevBuf<double2> d_Z, d_C, d_Q;
    DevBuf<double> d_sigma, d_disc;
    std::vector<int> rank;  // host copy after recompression
    std::vector<double> disc;
};

struct KStat {
    int64_t launches = 0;
    double ms = 0.0;
    double flops = 0.0;
    double bytes = 0.0;
};

// Growable device arrays on reserved virtual address space (CUDA VMM: cuMemAddressReserve +
// cuMemCreate/cuMemMap on demand): one base pointer whose regions grow without copies, so that
// data sized by the ranks found during the recompression (compact C, Q/F) can be laid out as it
// is produced.  Region r starts at byte offset r * region_bytes.
struct VaPool {
    unsigned long long base = 0;  // CUdeviceptr
    size_t region_bytes = 0, gran = 0;
    int dev = 0;
    std::vector<size_t> mapped_end;  // per region: bytes mapped from its start
    struct Map {
        size_t off, len;
        unsigned long long handle;
    };
    std::vector<Map> maps;
    void reserve(int device, int nregions, size_t region_bytes);
    void ensure(int region, size_t bytes);  // map at least `bytes` from the region's start
    void release();
    size_t mapped_bytes() const;
    double2* ptr() const { return reinterpret_cast<double2*>(base); }
    int64_t region_off(int region) const { return (int64_t)(region * region_bytes / sizeof(double2)); }
    VaPool() = default;
    VaPool(const VaPool&) = delete;
    VaPool& operator=(const VaPool&) = delete;
    ~VaPool() { release(); }
};

// Memory-lean plan (SURVEY §7.4 rules 2-7): the shard's row pairs are processed in chunks of whole
// subtrees below the top active level l0 (the chunk is the shard abstraction applied inside one
// GPU).  Persistent: the basis weights R (leaf: V) of the DIRECT row basis pairs (referenced by a
// block, as (t,c) or, through the adjoint symmetry, as (s,-c)), the transfer factors, and the
// outputs (compact Q/F, the C of direct pairs, S~).  Per chunk, regenerated or scratch: leaf V,
// non-direct R, Zhat, S_b, bound-layout C/Q of one level.  Needs the adjoint symmetry.
struct LeanState {
    bool on = false;
    int G = 0, l0 = 0;
    std::vector<int> p_lo, p_hi;        // row pairs of chunk g on level l: [p_lo[g*(L+1)+l], p_hi[...])
    std::vector<int> blk_ptr, blk;      // own blocks per chunk (CSR); slot of a block = its position in the chunk
    std::vector<int> qr_ptr, qr;        // per (g,l): row basis pairs weighted by QR (phase b)
    std::vector<int> lvb_ptr, lvb;      // per (g,l): row leaf pairs whose V phase b needs
    std::vector<int> lvd_ptr, lvd;      // per (g,l): row leaf pairs whose V is regenerated for the truncation
    std::vector<int> lvi;               // (s,-c) of other shards with R = V: regenerated from the mesh
    std::vector<char> keep;             // per basis pair: R (or V = R) persists after phase b
    std::vector<char> keepC;            // per row pair: C persists (projection)
    int64_t VR_persist = 0, VR_scratch = 0, E_total = 0, Z_scratch = 0, S_slots = 0;  // double2 units / slots
    std::vector<int64_t> E_off;         // lean transfer-factor layout (row basis pairs only)
    std::vector<int> kb_cur, rowsb_cur;  // row pass: current leading dimensions (rank after compaction)
    std::vector<int64_t> C_off_cur, Q_off_cur;
    int64_t C_used = 0, Q_used = 0;     // persistent compact bytes in use (double2 units)
    VaPool Cpool, Qpool;                // C: regions 0 persistent, 1 bound scratch, 2/3 compact scratch; Q: 0, 1
    DevBuf<int> d_blk, d_qr, d_lvb, d_lvd, d_lvi, d_mirror;
    DevBuf<double2> d_Zs, d_Ss;
    DevBuf<int64_t> d_soff, d_doff;
    DevBuf<int> d_rows, d_cols, d_lds;
    int64_t compact_items = 0;
    double peak_bytes = 0;              // device memory in use at the end of the last recompression
    // host plan only (device buffers and pools are kept; they are re-sized by lean_alloc)
    void clear_plan() {
        on = false;
        G = l0 = 0;
        for (auto* v : {&p_lo, &p_hi, &blk_ptr, &blk, &qr_ptr, &qr, &lvb_ptr, &lvb, &lvd_ptr, &lvd, &lvi, &kb_cur, &rowsb_cur})
            v->clear();
        keep.clear();
        keepC.clear();
        E_off.clear();
        C_off_cur.clear();
        Q_off_cur.clear();
        VR_persist = VR_scratch = E_total = Z_scratch = S_slots = 0;
        C_used = Q_used = compact_items = 0;
    }
};

struct Shard {
    Structure st;
    // sharding: shard `rank` of `world` owns the subtree of the rank-th cluster on
    // the cut level log2(world) -- its row/column pairs, and the blocks (t,s,c) with t in it.
    // world == 1 owns everything.
    int rank = 0, world = 1, cut = 0;
    std::vector<int> owner;          // per cluster, -1 above the cut
    std::vector<char> bp_own;        // basis pair computed by this shard
    int b_lo = 0, b_hi = 0;          // own blocks [b_lo, b_hi) (blocks sorted by owner of t)
    int64_t pos_lo = 0, pos_hi = 0;  // own range of cluster-ordered positions
    // exchange items per peer, in the same order on both sides (host-computed, replicated)
    std::vector<std::vector<int>> R_send, R_recv;  // basis pair ids: R_sc computed by QR (non-leaf)
    std::vector<std::vector<int>> C_send, C_recv;  // column pair ids: C'_sc, k'_sc, xh'_sc
    int n = 0, k = 0, m = 0, nclusters = 0;
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    bool profiling = false;
    bool recompressed = false;
    std::string err;
    double eps = 0.0;
    int mode = 0;
    // directions
    std::vector<int64_t> dir_off;
    std::vector<double> dirs_flat;
    // basis pairs
    // basis pair lookup: the ids of cluster t are [bp_cl[t], bp_cl[t+1]), sorted by direction
    std::vector<int> bp_cl;
    int bp_find(int64_t t, int64_t c) const {
        auto b = bp_c.begin() + bp_cl[t], e = bp_c.begin() + bp_cl[t + 1];
        auto it = std::lower_bound(b, e, (int)c);
        return (it != e && *it == c) ? (int)(it - bp_c.begin()) : -1;
    }
    int bp_at(int64_t t, int64_t c) const {
        const int id = bp_find(t, c);
        if (id < 0) throw std::logic_error("basis pair missing (closure broken)");
        return id;
    }
    std::vector<int> bp_t, bp_dir, bp_sddir, bp_child0, bp_child1, bp_R_rows, bp_level, bp_c;
    std::vector<int64_t> bp_V_off, bp_R_off, bp_E_off;
    std::vector<int> bp_lev_ptr;
    int64_t VR_total = 0, E_total = 0;
    std::vector<std::vector<int>> leafV_lists, basis_lists, E_lists;  // per level
    // adjoint symmetry (NEXT-1) applied to the basis weights: only ROW basis pairs are set up and
    // weighted; the column side of a block (t,s,c) reads R/V/E of the row basis pair (s,-c)
    // conjugated (V_{s,-c} = conj V_{s,c}, hence R and E likewise)
    std::vector<std::vector<int>> leafV_lists_sym, basis_lists_sym, E_lists_sym;
    std::vector<int> bp_neg;   // basis pair id of (t,-c), -1 if absent
    std::vector<int> blk_bpcs; // per block: basis pair id of (s,-c) (column side under the symmetry)
    bool col_data = false;     // column-only basis pairs' V/E have been generated (two-pass mode)
    bool sym_setup = false;    // the last set-up generated the row basis pairs only
    std::vector<int> basis_maxrows;
    int max_leaf = 0;
    // blocks
    std::vector<int> blk_t, blk_s, blk_dir, blk_bprow, blk_bpcol, blk_prow, blk_pcol, blk_mirror;
    int64_t mirror_missing = 0;
    // adjoint symmetry: column pair p = (s,c) <-> row pair col2row[p] = (s,-c)
    std::vector<int> col2row;
    bool sym_ok = false;     // structure admits it (checked in build_tables)
    int sym_opt = 1;         // dh2_set_option("adjoint_symmetry")
    int force_ws = 0;        // dh2_set_option("truncate_workspace")
    int qr_flag_init = 0;    // initial value of PlanD::qr_flag
    int qr_cq_init = 1;      // initial value of PlanD::qr_cq (column-per-thread basis-weight appends for k > 64:
                             // variant 1 = 16-row chunks, measured C4 basis -43 %)
    int qr_cq64_init = 1, qr_cq64_tw_init = 0;  // k <= 64 column-per-thread appends (basis: C3 -3 %, C2 -15 %; total weights +10 %)
    int qr_cq_tw_leaf_init = 3;  // PlanD::qr_cq_tw_leaf (thread-column total weights at leaf levels: C4 -9 %)
    int qr_cq_tw_init = 0;   // initial value of PlanD::qr_cq_tw (total weights: measured slower above the leaves, 0)
    DevBuf<double2> d_cq;    // their scratch triangles
    int trunc_mode_init = 1; // initial value of PlanD::trunc_mode (direct: measured -3 % C4, -16 % C5 leaves)
    int qr_wy_init = 0;      // initial value of PlanD::qr_wy (blocked WY appends measured slower on C4: 0) (dh2_set_option("qr_wy") sets the plan directly)
    int near_tma = 1;         // dh2_set_option("near_tma"): nearfield matvec streams N_b by cp.async.bulk (TMA) stages
    int mv_fwd_warp_init = 2; // PlanD::mv_fwd_warp (measured C4 matvec 12.0 / 7.7 / 6.6 ms for 0 / 1 / 2)
    int bw_variant_init = 1;  // PlanD::bw_variant (k > 64 only: C4 block weights -5 %)
    int t64_threads_init = 128;  // PlanD::t64_threads
    int split_trunc64 = 1;
    int split_trunc64_inner = 1;  // dh2_set_option("truncate_split64_inner")   // dh2_set_option("truncate_split64"): leaves of 33..64 as QR kernel + Jacobi/epilogue kernel
    int split_trunc = 1;     // dh2_set_option("truncate_split"): warp-register Jacobi for leaves <= 32
    int fuse_leaf = 0;       // dh2_set_option("fuse_leaf_weights"): leaf Zhat folded into the split QR
    std::vector<int> fused_levels[2];  // levels of the last recompress whose Zhat was fused (row, col)
    int64_t fused_append = 0;          // fused pairs whose stack (> fuse_direct rows) took the QR-append mode
    int fuse_direct = 64;              // dh2_set_option("fuse_direct_rows")
    DevBuf<char> d_tscr;     // scratch of the split truncation
    DevBuf<double2> d_ws;    // truncation workspace (persistent grid), grown on demand
    int64_t ws_launches = 0; // truncation launches that used the workspace
    bool sym_used = false;   // the last dh2_recompress derived the column pass from the row pass
    std::string sym_why;     // why sym_ok is false
    DevBuf<int> d_col2row;
    std::vector<int64_t> blk_St_off;
    int64_t St_total = 0;
    PassH row, col;
    std::vector<int> sweeps_h;  // Jacobi sweeps of the last truncated level (convergence check)
    LeanState lean;
    bool lean_required = false;  // set by the context: the partition's shards all take the lean plan
    std::vector<int> lean_slot, lean_mirror;  // lean plan: S slot of each block in its chunk; chunk-local mirrors
    // device
    DevBuf<double> d_xyz, d_c_lo, d_c_hi, d_dirs, d_omega, d_normG2;
    DevBuf<int64_t> d_tri, d_perm, d_c_begin, d_bp_V_off, d_bp_R_off, d_bp_E_off, d_blk_St_off;
    DevBuf<int> d_blk_mirror;
    DevBuf<int> d_c_size, d_bp_t, d_bp_dir, d_bp_sddir, d_bp_child0, d_bp_child1, d_bp_R_rows, d_blk_t, d_blk_s,
        d_blk_dir, d_blk_bprow, d_blk_bpcol, d_blk_prow, d_blk_pcol;
    std::vector<std::unique_ptr<DevBuf<int>>> d_lists;
    std::vector<const int*> d_leafV_list, d_basis_list, d_E_list, d_leafV_list_sym, d_basis_list_sym, d_E_list_sym;
    DevBuf<int> d_blk_bpcs, d_blk_slot, d_plist;
    DevBuf<double4> d_qp;
    DevBuf<GridD> d_grid;
    DevBuf<double2> d_VR, d_E, d_S, d_St, d_x, d_y, d_xp, d_yp, d_xh, d_yh;
    PlanD P{};
    // nearfield (NEXT-4, dh2_near.cu): this shard's inadmissible leaves (t owned), dense #t x #s
    // column-major in cluster order, assembled by dh2_nearfield_assemble
    struct NearH {
        bool on = false;
        int nq_sing = 0, nq_reg = 0;
        int nblk = 0, ngroups = 0;     // own blocks, distinct row leaves
        int max_rows = 0;               // largest row leaf
        int64_t nsing = 0, values = 0;  // touching entries, stored coefficients
        double evals = 0;               // kernel evaluations of the last assembly
        std::vector<int> t, s;          // per own block
        std::vector<int64_t> off;       // entry offset per own block
        DevBuf<int> d_t, d_s, d_gptr;   // d_gptr: blocks of row group g = [gptr[g], gptr[g+1])
        DevBuf<int> d_gord;             // row groups ordered by the tree level of their row cluster
        std::vector<int> glev_ptr;      // d_gord[glev_ptr[i] .. glev_ptr[i+1]): one level (disjoint rows: one launch)
        DevBuf<int64_t> d_off;
        DevBuf<double4> d_pts;          // n x nq_reg^2 Duffy-Gauss points (x, y, z, w 2|tau|), cluster order
        DevBuf<double2> d_val;
    } near;
    // stats
    std::map<std::string, KStat> kstat;
    std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> pending;
    std::vector<cudaEvent_t> ev_pool;
    int64_t launches_total = 0;
    double host_build_ms = 0.0, host_tables_ms = 0.0;
    std::vector<double> lean_wall_ms;  // host wall clock per lean recompression phase (last call)
    double tab_ms[6] = {0, 0, 0, 0, 0, 0};  // build_tables: basis pairs, blocks, passes, mirror, symmetry, exchange
    double E_row = 0, E_col = 0, far2 = 0;

    ~Shard() {
        for (auto& e : ev_pool) cudaEventDestroy(e);
        for (auto& p : pending) {
            cudaEventDestroy(std::get<1>(p));
            cudaEventDestroy(std::get<2>(p));
        }
        if (own_stream) cudaStreamDestroy(own_stream);
    }

    cudaEvent_t ev() {
        cudaEvent_t e;
        if (!ev_pool.empty()) {
            e = ev_pool.back();
            ev_pool.pop_back();
        } else {
            CK(cudaEventCreate(&e));
        }
        return e;
    }
    // run `f` (which launches `nl` kernels) under the timing class `cls`
    bool debug_sync = std::getenv("DH2_DEBUG_SYNC") != nullptr;
    template <typename F>
    void timed(const std::string& cls, int nl, F&& f) {
        struct Nvtx {  // one NVTX range per kernel class and level (visible to nsys / ncu --nvtx)
            explicit Nvtx(const std::string& n) { nvtxRangePushA(n.c_str()); }
            ~Nvtx() { nvtxRangePop(); }
        } range(cls);
        if (profiling) {
            cudaEvent_t a = ev(), b = ev();
            CK(cudaEventRecord(a, stream));
            f();
            CK(cudaEventRecord(b, stream));
            pending.emplace_back(cls, a, b);
        } else {
            f();
        }
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess && debug_sync) e = cudaStreamSynchronize(stream);  // DH2_DEBUG_SYNC=1
        if (e != cudaSuccess) throw CudaError("kernel class '" + cls + "': " + cudaGetErrorString(e));
        kstat[cls].launches += nl;
        launches_total += nl;
    }
    void finish() {
        CK(cudaStreamSynchronize(stream));
        for (auto& p : pending) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, std::get<1>(p), std::get<2>(p)));
            kstat[std::get<0>(p)].ms += ms;
            ev_pool.push_back(std::get<1>(p));
            ev_pool.push_back(std::get<2>(p));
        }
        pending.clear();
    }
};


// truncation of one level's pairs (dh2_api.cu)
void truncate_level(Shard* C, PassH& X, bool row, int l, int p0, int np, int maxrows, int maxz, bool all_leaf, bool fused,
                    double eps, int mode, const int* mirror);
bool fuse_leaf_level(const Shard* C, int leafrows, int maxz, int np);
// nearfield, NEXT-4 (dh2_near.cu)
void near_assemble(Shard* C, int nq_sing, int nq_reg);
void near_matvec(Shard* C);
// memory-lean plan (dh2_lean.cu)
void lean_plan(Shard* C, int G);
double lean_bytes(const Shard* C);
void lean_alloc(Shard* C);
void lean_begin(Shard* C);
void lean_basis(Shard* C);
void lean_weights_truncate(Shard* C, double eps, int mode);
void lean_columns(Shard* C);
void lean_project(Shard* C);
void lean_finish(Shard* C);

}  // namespace dh2
