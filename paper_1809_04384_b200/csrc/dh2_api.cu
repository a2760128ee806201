// C-ABI implementation of libdh2.so (include/dh2.h): host structure -> device tables ->
// level-batched sm_100a kernels.  No CPU fallback: every compute step runs on the GPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <sstream>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dh2.h"
#include "dh2_host.h"
#include "dh2_kernels.cuh"

namespace dh2 {
cudaError_t configure_kernels();
}

using namespace dh2;

namespace {

std::string g_last_error;

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

#define CK(x)                                                                                          \
    do {                                                                                               \
        cudaError_t e_ = (x);                                                                          \
        if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));       \
    } while (0)

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t cnt) {
        free();
        n = cnt;
        if (cnt) CK(cudaMalloc(&p, cnt * sizeof(T)));
    }
    void upload(const std::vector<T>& v, cudaStream_t s) {
        alloc(v.size());
        if (n) CK(cudaMemcpyAsync(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { free(); }
};

struct PassH {
    std::vector<int> bp, child0, child1, Z_rows, blk_ptr, blk, par_ptr, par, par_child, rowsb, kb;
    std::vector<int64_t> Z_off, C_off, Q_off, sig_off;
    std::vector<int> lev_ptr;  // pairs of level l: [lev_ptr[l], lev_ptr[l+1])
    std::vector<int> lc, lc_ptr;  // leaf-cluster groups (matvec output)
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

}  // namespace

struct dh2_ctx {
    Structure st;
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
    std::unordered_map<uint64_t, int> bp_id;  // (level-independent) key (t<<32)|c
    std::vector<int> bp_t, bp_dir, bp_sddir, bp_child0, bp_child1, bp_R_rows, bp_level, bp_c;
    std::vector<int64_t> bp_V_off, bp_R_off, bp_E_off;
    std::vector<int> bp_lev_ptr;
    int64_t VR_total = 0, E_total = 0;
    std::vector<std::vector<int>> leafV_lists, basis_lists, E_lists;  // per level
    std::vector<int> basis_maxrows;
    int max_leaf = 0;
    // blocks
    std::vector<int> blk_t, blk_s, blk_dir, blk_bprow, blk_bpcol, blk_prow, blk_pcol, blk_mirror;
    int64_t mirror_missing = 0;
    // adjoint symmetry: column pair p = (s,c) <-> row pair col2row[p] = (s,-c)
    std::vector<int> col2row;
    bool sym_ok = false;     // structure admits it (checked in build_tables)
    int sym_opt = 1;         // dh2_set_option("adjoint_symmetry")
    bool sym_used = false;   // the last dh2_recompress derived the column pass from the row pass
    std::string sym_why;     // why sym_ok is false
    DevBuf<int> d_col2row;
    std::vector<int64_t> blk_St_off;
    int64_t St_total = 0;
    PassH row, col;
    // device
    DevBuf<double> d_xyz, d_c_lo, d_c_hi, d_dirs, d_omega, d_normG2;
    DevBuf<int64_t> d_tri, d_perm, d_c_begin, d_bp_V_off, d_bp_R_off, d_bp_E_off, d_blk_St_off;
    DevBuf<int> d_blk_mirror;
    DevBuf<int> d_c_size, d_bp_t, d_bp_dir, d_bp_sddir, d_bp_child0, d_bp_child1, d_bp_R_rows, d_blk_t, d_blk_s,
        d_blk_dir, d_blk_bprow, d_blk_bpcol, d_blk_prow, d_blk_pcol;
    std::vector<std::unique_ptr<DevBuf<int>>> d_lists;
    std::vector<const int*> d_leafV_list, d_basis_list, d_E_list;
    DevBuf<double4> d_qp;
    DevBuf<GridD> d_grid;
    DevBuf<double2> d_VR, d_E, d_S, d_St, d_x, d_y, d_xp, d_yp, d_xh, d_yh;
    PlanD P{};
    // stats
    std::map<std::string, KStat> kstat;
    std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t>> pending;
    std::vector<cudaEvent_t> ev_pool;
    int64_t launches_total = 0;
    double host_build_ms = 0.0, host_tables_ms = 0.0;
    double E_row = 0, E_col = 0, far2 = 0;

    ~dh2_ctx() {
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
    template <typename F>
    void timed(const std::string& cls, int nl, F&& f) {
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
        if (e != cudaSuccess) throw CudaError("launch of kernel class '" + cls + "': " + cudaGetErrorString(e));
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

namespace {

inline uint64_t key(int64_t t, int64_t c) { return ((uint64_t)t << 32) | (uint64_t)c; }

// Adjoint symmetry of the single-layer DH^2 (W = V; column pass =
// row pass on G^*).  With antipodal direction sets (DESIGN R2/R4), V_{s,-c} =
// conj(V_{s,c}), E likewise, and the mirror block (s,t,-c) has S = S_b^T.  The column-pass
// matrix of (s,c), rows w_b R_tc S_b over t in col(s,c) plus inherited E Zhat'^*, is then the
// complex conjugate of the row-pass matrix of (s,-c), so Zhat', sigma', k', Q', F', C' are
// the conjugates of the row results at (s,-c).  This checks that the structure has exactly
// that correspondence (pairs, blocks, parents, children, bounds); otherwise two passes run.
void check_symmetry(dh2_ctx* C) {
    Structure& S = C->st;
    const int L = S.ct.depth;
    const PassH &R = C->row, &X = C->col;
    C->sym_ok = false;
    C->col2row.clear();
    if (C->mirror_missing) { C->sym_why = "blocks without an antipodal mirror"; return; }
    if (R.bp.size() != X.bp.size()) { C->sym_why = "row and column pair counts differ"; return; }
    std::unordered_map<uint64_t, int> rowpid;
    for (size_t q = 0; q < R.bp.size(); ++q) rowpid[key(C->bp_t[R.bp[q]], C->bp_c[R.bp[q]])] = (int)q;
    std::vector<std::vector<int64_t>> neg(L + 1);
    for (int l = 0; l <= L; ++l) {
        if (S.basis_pairs[l].empty()) continue;
        const auto& D = S.D(l);
        const int nd = (int)D.size() / 3;
        std::map<std::tuple<double, double, double>, int64_t> idx;
        for (int c = 0; c < nd; ++c) idx[{D[3 * c] + 0.0, D[3 * c + 1] + 0.0, D[3 * c + 2] + 0.0}] = c;
        neg[l].assign(nd, -1);
        for (int c = 0; c < nd; ++c) {
            auto it = idx.find({-D[3 * c] + 0.0, -D[3 * c + 1] + 0.0, -D[3 * c + 2] + 0.0});
            if (it != idx.end()) neg[l][c] = it->second;
        }
    }
    std::vector<int> c2r(X.bp.size(), -1);
    for (size_t p = 0; p < X.bp.size(); ++p) {
        const int id = X.bp[p];
        const int64_t nc = neg[C->bp_level[id]][C->bp_c[id]];
        auto it = nc < 0 ? rowpid.end() : rowpid.find(key(C->bp_t[id], nc));
        if (it == rowpid.end()) { C->sym_why = "column pair without a row pair at -c"; return; }
        c2r[p] = it->second;
    }
    for (size_t p = 0; p < X.bp.size(); ++p) {
        const int q = c2r[p];
        if (X.Z_rows[p] != R.Z_rows[q] || X.total_rows[p] != R.total_rows[q] || X.kb[p] != R.kb[q] ||
            X.rowsb[p] != R.rowsb[q]) { C->sym_why = "bounds differ"; return; }
        if ((X.child0[p] < 0) != (R.child0[q] < 0)) { C->sym_why = "leaf mismatch"; return; }
        if (X.child0[p] >= 0 && (c2r[X.child0[p]] != R.child0[q] || c2r[X.child1[p]] != R.child1[q])) {
            C->sym_why = "children differ"; return;
        }
        std::vector<int> a, b;
        for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) a.push_back(C->blk_mirror[X.blk[ib]]);
        for (int ib = R.blk_ptr[q]; ib < R.blk_ptr[q + 1]; ++ib) b.push_back(R.blk[ib]);
        std::sort(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        if (a != b) { C->sym_why = "block sets differ"; return; }
        std::vector<int> pa, pb;
        for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) pa.push_back(c2r[X.par[ip]] * 2 + X.par_child[ip]);
        for (int ip = R.par_ptr[q]; ip < R.par_ptr[q + 1]; ++ip) pb.push_back(R.par[ip] * 2 + R.par_child[ip]);
        std::sort(pa.begin(), pa.end());
        std::sort(pb.begin(), pb.end());
        if (pa != pb) { C->sym_why = "parents differ"; return; }
    }
    C->col2row.swap(c2r);
    C->sym_ok = true;
    C->sym_why.clear();
}

void build_tables(dh2_ctx* C) {
    Structure& S = C->st;
    const ClusterTree& T = S.ct;
    const int k = S.k, L = T.depth;
    C->n = (int)T.n;
    C->k = k;
    C->m = S.p.m;
    C->nclusters = (int)T.begin.size();
    // directions of the materialised levels
    C->dir_off.assign(L + 2, -1);
    for (int l = 0; l <= L; ++l) {
        if (S.basis_pairs[l].empty()) continue;
        C->dir_off[l] = (int64_t)C->dirs_flat.size() / 3;
        const auto& D = S.D(l);
        C->dirs_flat.insert(C->dirs_flat.end(), D.begin(), D.end());
    }
    // basis pairs, bottom-up order not required; ids level by level
    C->bp_lev_ptr.assign(L + 2, 0);
    for (int l = 0; l <= L; ++l) {
        C->bp_lev_ptr[l] = (int)C->bp_t.size();
        for (const Pair& pr : S.basis_pairs[l]) {
            int id = (int)C->bp_t.size();
            C->bp_id[key(pr.t, pr.c)] = id;
            C->bp_t.push_back((int)pr.t);
            C->bp_c.push_back((int)pr.c);
            C->bp_level.push_back(l);
            C->bp_dir.push_back((int)(C->dir_off[l] + pr.c));
        }
    }
    C->bp_lev_ptr[L + 1] = (int)C->bp_t.size();
    const int nbp = (int)C->bp_t.size();
    C->bp_child0.assign(nbp, -1);
    C->bp_child1.assign(nbp, -1);
    C->bp_sddir.assign(nbp, -1);
    C->bp_V_off.assign(nbp, -1);
    C->bp_R_off.assign(nbp, -1);
    C->bp_E_off.assign(nbp, -1);
    C->bp_R_rows.assign(nbp, 0);
    C->leafV_lists.assign(L + 1, {});
    C->basis_lists.assign(L + 1, {});
    C->E_lists.assign(L + 1, {});
    C->basis_maxrows.assign(L + 1, 0);
    int64_t off = 0;
    for (int id = 0; id < nbp; ++id) {
        int t = C->bp_t[id], l = C->bp_level[id];
        if (T.is_leaf(t)) {
            int sz = (int)T.size(t);
            C->max_leaf = std::max(C->max_leaf, sz);
            C->bp_V_off[id] = off;
            off += (int64_t)sz * k;
            C->leafV_lists[l].push_back(id);
        } else {
            int64_t c2 = S.sd(l, C->bp_c[id]);
            C->bp_sddir[id] = (int)(C->dir_off[l + 1] + c2);
            auto it0 = C->bp_id.find(key(T.child0[t], c2));
            auto it1 = C->bp_id.find(key(T.child1[t], c2));
            if (it0 == C->bp_id.end() || it1 == C->bp_id.end()) throw std::logic_error("closure broken");
            C->bp_child0[id] = it0->second;
            C->bp_child1[id] = it1->second;
            C->E_lists[l].push_back(id);
        }
    }
    // basis weights: rows bottom-up
    for (int l = L; l >= 0; --l) {
        for (int id = C->bp_lev_ptr[l]; id < C->bp_lev_ptr[l + 1]; ++id) {
            int t = C->bp_t[id];
            if (T.is_leaf(t)) {
                int sz = (int)T.size(t);
                if (sz <= k) {
                    C->bp_R_rows[id] = sz;
                    C->bp_R_off[id] = C->bp_V_off[id];  // R = V, P = I (Eq. 18)
                } else {
                    C->bp_R_rows[id] = k;
                    C->bp_R_off[id] = off;
                    off += (int64_t)k * k;
                    C->basis_lists[l].push_back(id);
                    C->basis_maxrows[l] = std::max(C->basis_maxrows[l], sz);
                }
            } else {
                int rows = C->bp_R_rows[C->bp_child0[id]] + C->bp_R_rows[C->bp_child1[id]];
                C->bp_R_rows[id] = std::min(rows, k);
                C->bp_R_off[id] = off;
                off += (int64_t)C->bp_R_rows[id] * k;
                C->basis_lists[l].push_back(id);
                C->basis_maxrows[l] = std::max(C->basis_maxrows[l], rows);
            }
        }
    }
    C->VR_total = off;
    int64_t eoff = 0;
    for (int id = 0; id < nbp; ++id)
        if (C->bp_child0[id] >= 0) {
            C->bp_E_off[id] = eoff;
            eoff += 6LL * C->m * C->m;
        }
    C->E_total = eoff;
    // blocks
    const int nb = (int)S.blocks.size();
    for (const Block& b : S.blocks) {
        int l = (int)T.level[b.t];
        C->blk_t.push_back((int)b.t);
        C->blk_s.push_back((int)b.s);
        C->blk_dir.push_back((int)(C->dir_off[l] + b.c));
        C->blk_bprow.push_back(C->bp_id.at(key(b.t, b.c)));
        C->blk_bpcol.push_back(C->bp_id.at(key(b.s, b.c)));
    }
    // passes
    for (int side = 0; side < 2; ++side) {
        PassH& X = side == 0 ? C->row : C->col;
        const auto& pairs = side == 0 ? S.row_pairs : S.col_pairs;
        std::unordered_map<uint64_t, int> pid;
        X.lev_ptr.assign(L + 2, 0);
        for (int l = 0; l <= L; ++l) {
            X.lev_ptr[l] = (int)X.bp.size();
            for (const Pair& pr : pairs[l]) {
                pid[key(pr.t, pr.c)] = (int)X.bp.size();
                X.bp.push_back(C->bp_id.at(key(pr.t, pr.c)));
            }
        }
        X.lev_ptr[L + 1] = (int)X.bp.size();
        const int np = (int)X.bp.size();
        X.child0.assign(np, -1);
        X.child1.assign(np, -1);
        for (int p = 0; p < np; ++p) {
            int id = X.bp[p];
            int t = C->bp_t[id];
            if (!T.is_leaf(t)) {
                int l = C->bp_level[id];
                int64_t c2 = S.sd(l, C->bp_c[id]);
                X.child0[p] = pid.at(key(T.child0[t], c2));
                X.child1[p] = pid.at(key(T.child1[t], c2));
            }
        }
        // blocks CSR (blocks sorted by (t,s): per pair sorted by the other cluster)
        std::vector<std::vector<int>> bl(np);
        for (int b = 0; b < nb; ++b) {
            const Block& B = S.blocks[b];
            int p = pid.at(key(side == 0 ? B.t : B.s, B.c));
            bl[p].push_back(b);
            if (side == 0)
                C->blk_prow.push_back(p);
            else
                C->blk_pcol.push_back(p);
        }
        X.blk_ptr.assign(np + 1, 0);
        for (int p = 0; p < np; ++p) {
            X.blk_ptr[p + 1] = X.blk_ptr[p] + (int)bl[p].size();
            X.blk.insert(X.blk.end(), bl[p].begin(), bl[p].end());
        }
        // parents CSR: (t+, c+) -> children (t_i, sd(c+))
        std::vector<std::vector<std::pair<int, int>>> pl(np);
        for (int p = 0; p < np; ++p) {
            if (X.child0[p] < 0) continue;
            pl[X.child0[p]].push_back({p, 0});
            pl[X.child1[p]].push_back({p, 1});
        }
        X.par_ptr.assign(np + 1, 0);
        for (int p = 0; p < np; ++p) {
            X.par_ptr[p + 1] = X.par_ptr[p] + (int)pl[p].size();
            for (auto& q : pl[p]) {
                X.par.push_back(q.first);
                X.par_child.push_back(q.second);
            }
        }
        // Zhat rows, top-down
        X.Z_rows.assign(np, 0);
        X.total_rows.assign(np, 0);
        X.lev_max_total.assign(L + 1, 0);
        X.lev_max_zrows.assign(L + 1, 0);
        X.lev_max_leafrows.assign(L + 1, 0);
        for (int l = 0; l <= L; ++l)
            for (int p = X.lev_ptr[l]; p < X.lev_ptr[l + 1]; ++p) {
                int tot = 0;
                for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
                    int b = X.blk[ib];
                    tot += C->bp_R_rows[side == 0 ? C->blk_bpcol[b] : C->blk_bprow[b]];
                }
                for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) tot += X.Z_rows[X.par[ip]];
                X.total_rows[p] = tot;
                X.Z_rows[p] = std::min(tot, k);
                X.lev_max_total[l] = std::max(X.lev_max_total[l], tot);
                X.lev_max_zrows[l] = std::max(X.lev_max_zrows[l], X.Z_rows[p]);
            }
        // rank bounds, bottom-up
        X.rowsb.assign(np, 0);
        X.kb.assign(np, 0);
        for (int l = L; l >= 0; --l)
            for (int p = X.lev_ptr[l]; p < X.lev_ptr[l + 1]; ++p) {
                int t = C->bp_t[X.bp[p]];
                X.rowsb[p] = X.child0[p] < 0 ? (int)T.size(t) : X.kb[X.child0[p]] + X.kb[X.child1[p]];
                X.kb[p] = std::min(X.rowsb[p], X.Z_rows[p]);
                if (X.child0[p] < 0) X.lev_max_leafrows[l] = std::max(X.lev_max_leafrows[l], (int)T.size(t));
            }
        X.Z_off.assign(np, 0);
        X.C_off.assign(np, 0);
        X.Q_off.assign(np, 0);
        X.sig_off.assign(np, 0);
        for (int p = 0; p < np; ++p) {
            X.Z_off[p] = X.Z_total;
            X.Z_total += (int64_t)X.Z_rows[p] * k;
            X.C_off[p] = X.C_total;
            X.C_total += (int64_t)X.kb[p] * k;
            X.Q_off[p] = X.Q_total;
            X.Q_total += (int64_t)X.rowsb[p] * X.kb[p];
            X.sig_off[p] = X.sig_total;
            X.sig_total += X.kb[p];
        }
        // leaf-cluster groups (contiguous pairs of one leaf cluster)
        X.lc_ptr.push_back(0);
        int lastt = -1;
        for (int p = 0; p < np; ++p) {
            int t = C->bp_t[X.bp[p]];
            if (!T.is_leaf(t)) continue;
            if (t != lastt && !X.lc.empty()) X.lc_ptr.push_back((int)X.lc.size());
            X.lc.push_back(p);
            lastt = t;
        }
        if (!X.lc.empty()) X.lc_ptr.push_back((int)X.lc.size());
    }
    // antipodal mirror b' = (s, t, -c) of every block: S_{b'} = S_b^T exactly (DESIGN §total weights)
    {
        std::unordered_map<uint64_t, int> ts;
        for (int b = 0; b < nb; ++b) ts[key(S.blocks[b].t, S.blocks[b].s)] = b;
        C->blk_mirror.assign(nb, -1);
        for (int b = 0; b < nb; ++b) {
            const Block& B = S.blocks[b];
            auto it = ts.find(key(B.s, B.t));
            if (it == ts.end()) { ++C->mirror_missing; continue; }
            int l = (int)T.level[B.t];
            const auto& D = S.D(l);
            int64_t c2 = S.blocks[it->second].c;
            bool neg = D[3 * c2] == -D[3 * B.c] && D[3 * c2 + 1] == -D[3 * B.c + 1] && D[3 * c2 + 2] == -D[3 * B.c + 2];
            if (neg) C->blk_mirror[b] = it->second; else ++C->mirror_missing;
        }
    }
    check_symmetry(C);
    C->blk_St_off.assign(nb, 0);
    for (int b = 0; b < nb; ++b) {
        C->blk_St_off[b] = C->St_total;
        C->St_total += (int64_t)C->row.kb[C->blk_prow[b]] * C->col.kb[C->blk_pcol[b]];
    }
}

void upload_pass(dh2_ctx* C, PassH& X, PassD& D, bool alloc_Z) {
    cudaStream_t s = C->stream;
    X.d_bp.upload(X.bp, s);
    X.d_child0.upload(X.child0, s);
    X.d_child1.upload(X.child1, s);
    X.d_Z_rows.upload(X.Z_rows, s);
    X.d_blk_ptr.upload(X.blk_ptr, s);
    X.d_blk.upload(X.blk, s);
    X.d_par_ptr.upload(X.par_ptr, s);
    X.d_par.upload(X.par, s);
    X.d_par_child.upload(X.par_child, s);
    X.d_rowsb.upload(X.rowsb, s);
    X.d_kb.upload(X.kb, s);
    X.d_Z_off.upload(X.Z_off, s);
    X.d_C_off.upload(X.C_off, s);
    X.d_Q_off.upload(X.Q_off, s);
    X.d_sig_off.upload(X.sig_off, s);
    X.d_lc.upload(X.lc, s);
    X.d_lc_ptr.upload(X.lc_ptr, s);
    const size_t np = X.bp.size();
    X.d_rank.alloc(np);
    X.d_nsig.alloc(np);
    X.d_disc.alloc(np);
    X.d_sweeps.alloc(np);
    if (alloc_Z) X.d_Z.alloc(X.Z_total);
    X.d_C.alloc(X.C_total);
    X.d_Q.alloc(X.Q_total);
    X.d_sigma.alloc(X.sig_total);
    D.npairs = (int)np;
    D.bp = X.d_bp.p;
    D.child0 = X.d_child0.p;
    D.child1 = X.d_child1.p;
    D.Z_off = X.d_Z_off.p;
    D.Z_rows = X.d_Z_rows.p;
    D.blk_ptr = X.d_blk_ptr.p;
    D.blk = X.d_blk.p;
    D.par_ptr = X.d_par_ptr.p;
    D.par = X.d_par.p;
    D.par_child = X.d_par_child.p;
    D.rowsb = X.d_rowsb.p;
    D.kb = X.d_kb.p;
    D.C_off = X.d_C_off.p;
    D.Q_off = X.d_Q_off.p;
    D.sig_off = X.d_sig_off.p;
    D.Z = X.d_Z.p;
    D.C = X.d_C.p;
    D.Q = X.d_Q.p;
    D.sigma = X.d_sigma.p;
    D.rank = X.d_rank.p;
    D.nsig = X.d_nsig.p;
    D.disc = X.d_disc.p;
    D.sweeps = X.d_sweeps.p;
}

size_t plan_bytes(const dh2_ctx* C) {
    size_t b = 0;
    b += (size_t)C->VR_total * 16 + (size_t)C->E_total * 16 + C->st.blocks.size() * (size_t)C->k * C->k * 16;
    b += (size_t)C->St_total * 16;
    for (const PassH* X : {&C->row, &C->col})
        b += (size_t)((X == &C->col && C->sym_ok ? 0 : X->Z_total) + X->C_total + X->Q_total) * 16 + (size_t)X->sig_total * 8;
    b += (size_t)C->n * 7 * 32 + (size_t)C->nclusters * sizeof(GridD);
    return b;
}

void upload_all(dh2_ctx* C, const double* xyz, int64_t nv, const int64_t* tri) {
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    size_t freeb = 0, totb = 0;
    CK(cudaMemGetInfo(&freeb, &totb));
    size_t need = plan_bytes(C);
    if (need + (size_t)256 * 1024 * 1024 > freeb)
        throw NoMem("device memory plan needs " + std::to_string(need >> 20) + " MiB, free " + std::to_string(freeb >> 20) + " MiB");
    C->d_xyz.upload(std::vector<double>(xyz, xyz + 3 * nv), s);
    C->d_tri.upload(std::vector<int64_t>(tri, tri + 3 * C->n), s);
    C->d_perm.upload(T.perm, s);
    C->d_c_lo.upload(T.lo, s);
    C->d_c_hi.upload(T.hi, s);
    C->d_c_begin.upload(T.begin, s);
    std::vector<int> csz(C->nclusters);
    for (int t = 0; t < C->nclusters; ++t) csz[t] = (int)T.size(t);
    C->d_c_size.upload(csz, s);
    C->d_dirs.upload(C->dirs_flat, s);
    C->d_bp_t.upload(C->bp_t, s);
    C->d_bp_dir.upload(C->bp_dir, s);
    C->d_bp_sddir.upload(C->bp_sddir, s);
    C->d_bp_child0.upload(C->bp_child0, s);
    C->d_bp_child1.upload(C->bp_child1, s);
    C->d_bp_R_rows.upload(C->bp_R_rows, s);
    C->d_bp_V_off.upload(C->bp_V_off, s);
    C->d_bp_R_off.upload(C->bp_R_off, s);
    C->d_bp_E_off.upload(C->bp_E_off, s);
    C->d_blk_t.upload(C->blk_t, s);
    C->d_blk_s.upload(C->blk_s, s);
    C->d_blk_dir.upload(C->blk_dir, s);
    C->d_blk_bprow.upload(C->blk_bprow, s);
    C->d_blk_bpcol.upload(C->blk_bpcol, s);
    C->d_blk_prow.upload(C->blk_prow, s);
    C->d_blk_pcol.upload(C->blk_pcol, s);
    C->d_blk_St_off.upload(C->blk_St_off, s);
    C->d_blk_mirror.upload(C->blk_mirror, s);
    auto up_list = [&](const std::vector<int>& v) -> const int* {
        C->d_lists.emplace_back(new DevBuf<int>());
        C->d_lists.back()->upload(v, s);
        return C->d_lists.back()->p;
    };
    const int L = T.depth;
    for (int l = 0; l <= L; ++l) {
        C->d_leafV_list.push_back(up_list(C->leafV_lists[l]));
        C->d_basis_list.push_back(up_list(C->basis_lists[l]));
        C->d_E_list.push_back(up_list(C->E_lists[l]));
    }
    C->d_qp.alloc((size_t)C->n * 7);
    C->d_grid.alloc(C->nclusters);
    C->d_VR.alloc(C->VR_total);
    C->d_E.alloc(C->E_total);
    const size_t nb = C->st.blocks.size();
    C->d_S.alloc(nb * C->k * C->k);
    C->d_St.alloc(C->St_total);
    C->d_omega.alloc(nb);
    C->d_normG2.alloc(nb);
    C->d_xp.alloc(C->n);
    C->d_yp.alloc(C->n);
    C->d_x.alloc(C->n);
    C->d_y.alloc(C->n);
    C->d_xh.alloc((size_t)C->col.bp.size() * C->k);
    C->d_yh.alloc((size_t)C->row.bp.size() * C->k);

    PlanD& P = C->P;
    P.n = C->n;
    P.m = C->m;
    P.k = C->k;
    P.nclusters = C->nclusters;
    P.kappa = C->st.p.kappa;
    P.xyz = C->d_xyz.p;
    P.tri = C->d_tri.p;
    P.perm = C->d_perm.p;
    P.qp = C->d_qp.p;
    P.c_lo = C->d_c_lo.p;
    P.c_hi = C->d_c_hi.p;
    P.c_begin = C->d_c_begin.p;
    P.c_size = C->d_c_size.p;
    P.grid = C->d_grid.p;
    P.dirs = C->d_dirs.p;
    P.nbp = (int)C->bp_t.size();
    P.bp_t = C->d_bp_t.p;
    P.bp_dir = C->d_bp_dir.p;
    P.bp_sddir = C->d_bp_sddir.p;
    P.bp_child0 = C->d_bp_child0.p;
    P.bp_child1 = C->d_bp_child1.p;
    P.bp_V_off = C->d_bp_V_off.p;
    P.bp_R_off = C->d_bp_R_off.p;
    P.bp_R_rows = C->d_bp_R_rows.p;
    P.bp_E_off = C->d_bp_E_off.p;
    P.V = C->d_VR.p;
    P.R = C->d_VR.p;
    P.E = C->d_E.p;
    P.nblk = (int)nb;
    P.blk_t = C->d_blk_t.p;
    P.blk_s = C->d_blk_s.p;
    P.blk_dir = C->d_blk_dir.p;
    P.blk_bprow = C->d_blk_bprow.p;
    P.blk_bpcol = C->d_blk_bpcol.p;
    P.blk_prow = C->d_blk_prow.p;
    P.blk_pcol = C->d_blk_pcol.p;
    P.blk_St_off = C->d_blk_St_off.p;
    P.S = C->d_S.p;
    P.St = C->d_St.p;
    P.omega = C->d_omega.p;
    P.normG2 = C->d_normG2.p;
    upload_pass(C, C->row, P.row, true);
    upload_pass(C, C->col, P.col, !C->sym_ok);  // column Zhat only when two passes can run
    if (C->sym_ok) C->d_col2row.upload(C->col2row, s);
}

// Device set-up (§2): quadrature points, grids, leaf V, E factors, S.
void run_setup(dh2_ctx* C) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const int L = C->st.ct.depth;
    const int k = C->k;
    C->timed("setup_quad", 2, [&] { launch_quad(P, s); });
    C->timed("setup_grid", 1, [&] { launch_grid(P, s); });
    for (int l = 0; l <= L; ++l) {
        int nl = (int)C->leafV_lists[l].size();
        if (nl) {
            C->timed("setup_leafV", 1, [&] { launch_leafV(P, C->d_leafV_list[l], nl, C->max_leaf, s); });
            double ent = 0;
            for (int id : C->leafV_lists[l]) ent += (double)C->st.ct.size(C->bp_t[id]) * k;
            auto& st = C->kstat["setup_leafV"];
            st.flops += ent * 7 * 6;
            st.bytes += ent * 16 + ent / k * 7 * 32;
        }
        int ne = (int)C->E_lists[l].size();
        if (ne) {
            C->timed("setup_E", 1, [&] { launch_E(P, C->d_E_list[l], ne, s); });
            C->kstat["setup_E"].bytes += (double)ne * 6 * C->m * C->m * 16;
        }
    }
    C->timed("setup_S", 1, [&] { launch_S(P, s); });
    auto& st = C->kstat["setup_S"];
    double ent = (double)C->st.blocks.size() * k * k;
    st.flops += ent * 20;
    st.bytes += ent * 16;
}

inline double qr_flops(double M, double N) {
    double K = std::min(M, N);
    return 8.0 * (M * N * K - (M + N) * K * K / 2.0 + K * K * K / 3.0);
}

void run_recompress(dh2_ctx* C, double eps, int mode) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    const int L = T.depth, k = C->k, m = C->m;
    // basis weights, bottom-up (Eq. 18)
    for (int l = L; l >= 0; --l) {
        int nb = (int)C->basis_lists[l].size();
        if (!nb) continue;
        C->timed("basis@" + std::to_string(l), 1, [&] { launch_basis(P, C->d_basis_list[l], nb, C->basis_maxrows[l], s); });
        double fl = 0;
        for (int id : C->basis_lists[l]) {
            int rows;
            if (C->bp_child0[id] < 0)
                rows = (int)T.size(C->bp_t[id]);
            else {
                int r0 = C->bp_R_rows[C->bp_child0[id]], r1 = C->bp_R_rows[C->bp_child1[id]];
                rows = r0 + r1;
                fl += 8.0 * 3 * rows * k * m;
            }
            if (rows > k) fl += qr_flops(rows, k);
        }
        C->kstat["basis@" + std::to_string(l)].flops += fl;
    }
    // block weights
    C->timed("block_weights", 1, [&] { launch_block_weights(P, mode, C->d_blk_mirror.p, s); });
    {
        double fl = 0;
        for (size_t b = 0; b < C->st.blocks.size(); ++b) {
            double rt = C->bp_R_rows[C->blk_bprow[b]], rs = C->bp_R_rows[C->blk_bpcol[b]];
            fl += 8.0 * (rt * k * k + rt * rs * k);
        }
        C->kstat["block_weights"].flops += fl;
    }
    const bool sym = C->sym_ok && C->sym_opt;
    if (!sym && !C->col.d_Z.p && C->col.Z_total) {  // two passes requested on a symmetric structure
        C->col.d_Z.alloc(C->col.Z_total);
        C->P.col.Z = C->col.d_Z.p;
    }
    C->sym_used = sym;
    for (int side = 0; side < 2; ++side) {
        PassH& X = side == 0 ? C->row : C->col;
        const bool row = side == 0;
        if (!row && sym) {
            // column pass = conjugate of the row pass at -c (check_symmetry)
            const int np = (int)X.bp.size();
            C->timed("mirror_col", 1, [&] { launch_mirror_pass(P, C->d_col2row.p, np, s); });
            X.rank.resize(np);
            for (int p = 0; p < np; ++p) X.rank[p] = C->row.rank[C->col2row[p]];
            double by = 0;
            for (int p = 0; p < np; ++p) {
                const int kk = X.rank[p];
                by += 2.0 * 16.0 * ((double)kk * k + (double)X.rowsb[p] * kk);
            }
            C->kstat["mirror_col"].bytes += by;
            continue;
        }
        // total weights, top-down
        for (int l = 0; l <= L; ++l) {
            int p0 = X.lev_ptr[l], np = X.lev_ptr[l + 1] - p0;
            if (!np) continue;
            C->timed(std::string(row ? "total_weights_row@" : "total_weights_col@") + std::to_string(l), 1, [&] { launch_total_weights(P, row, p0, np, C->d_blk_mirror.p, s); });
            double fl = 0;
            for (int p = p0; p < p0 + np; ++p) {
                for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
                    int b = X.blk[ib];
                    fl += 8.0 * C->bp_R_rows[row ? C->blk_bpcol[b] : C->blk_bprow[b]] * (double)k * k;
                }
                for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) fl += 8.0 * 3 * X.Z_rows[X.par[ip]] * (double)k * m;
                if (X.total_rows[p] > k) fl += 8.0 * X.total_rows[p] * (double)k * k;  // structured QR appends
            }
            C->kstat[std::string(row ? "total_weights_row@" : "total_weights_col@") + std::to_string(l)].flops += fl;
        }
        // truncation, bottom-up
        X.rank.assign(X.bp.size(), 0);
        for (int l = L; l >= 0; --l) {
            int p0 = X.lev_ptr[l], np = X.lev_ptr[l + 1] - p0;
            if (!np) continue;
            int maxrows = X.lev_max_leafrows[l];
            for (int p = p0; p < p0 + np; ++p)
                if (X.child0[p] >= 0) maxrows = std::max(maxrows, X.rank[X.child0[p]] + X.rank[X.child1[p]]);
            int maxz = X.lev_max_zrows[l];
            bool all_leaf = true, any_leaf = false;
            for (int p = p0; p < p0 + np; ++p) {
                all_leaf = all_leaf && X.child0[p] < 0;
                any_leaf = any_leaf || X.child0[p] < 0;
            }
            if (any_leaf && !all_leaf)  // median-split trees never mix leaves and inner clusters on a level
                throw NotImpl("a tree level mixing leaf and non-leaf clusters is not supported by k_truncate");
            C->timed(std::string(row ? "truncate_row@" : "truncate_col@") + std::to_string(l), 1, [&] { launch_truncate(P, row, p0, np, maxrows, maxz, all_leaf, eps, mode, s); });
            CK(cudaMemcpyAsync(X.rank.data() + p0, X.d_rank.p + p0, np * sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            double fl = 0;
            for (int p = p0; p < p0 + np; ++p) {
                double rows = X.child0[p] < 0 ? (double)T.size(C->bp_t[X.bp[p]]) : X.rank[X.child0[p]] + X.rank[X.child1[p]];
                double zr = X.Z_rows[p];
                if (X.child0[p] >= 0) fl += 8.0 * 3 * rows * k * m;
                fl += 8.0 * rows * zr * k;  // M
                double n = std::min(rows, zr);
                if (rows < zr) fl += qr_flops(zr, rows);
                fl += 8.0 * 10.0 * rows * n * n;  // SVD, C_svd = 10 model (DESIGN §flop model)
                fl += 8.0 * X.rank[p] * rows * k;  // C
            }
            C->kstat[std::string(row ? "truncate_row@" : "truncate_col@") + std::to_string(l)].flops += fl;
        }
    }
    // projection
    int maxkrow = 0;
    for (int r : C->row.rank) maxkrow = std::max(maxkrow, r);
    C->timed("project", 1, [&] { launch_project(P, maxkrow, s); });
    {
        double fl = 0;
        for (size_t b = 0; b < C->st.blocks.size(); ++b) {
            double kt = C->row.rank[C->blk_prow[b]], ks = C->col.rank[C->blk_pcol[b]];
            fl += 8.0 * (kt * k * k + kt * ks * k);
        }
        C->kstat["project"].flops += fl;
    }
}

void run_matvec(dh2_ctx* C, bool recomp, const double2* x, double2* y) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const int L = C->st.ct.depth, n = C->n;
    C->timed("matvec", 1, [&] { launch_permute(P.perm, x, C->d_xp.p, n, true, s); });
    for (int l = L; l >= 0; --l) {
        int p0 = C->col.lev_ptr[l], np = C->col.lev_ptr[l + 1] - p0;
        if (np) C->timed("matvec", 1, [&] { launch_mv_forward(P, recomp, p0, np, C->d_xp.p, C->d_xh.p, s); });
    }
    C->timed("matvec", 1, [&] { launch_mv_couple(P, recomp, C->d_xh.p, C->d_yh.p, s); });
    for (int l = 0; l <= L; ++l) {
        int p0 = C->row.lev_ptr[l], np = C->row.lev_ptr[l + 1] - p0;
        if (np) C->timed("matvec", 1, [&] { launch_mv_backward(P, recomp, p0, np, C->d_yh.p, s); });
    }
    CK(cudaMemsetAsync(C->d_yp.p, 0, sizeof(double2) * n, s));
    int nlc = (int)C->row.lc_ptr.size() - 1;
    C->timed("matvec", 1, [&] {
        launch_mv_leaf_out(P, recomp, C->row.d_lc.p, C->row.d_lc_ptr.p, std::max(nlc, 0), C->d_yh.p, C->d_yp.p, s);
    });
    C->timed("matvec", 1, [&] { launch_permute(P.perm, C->d_yp.p, y, n, false, s); });
}

void require_device(const dh2_ctx* C) {
    if (C->device == DH2_DEVICE_NONE) throw StateError("structure-only context (device = DH2_DEVICE_NONE) has no device data");
}

int fail(dh2_ctx* C, int code, const std::string& msg) {
    if (C) C->err = msg;
    g_last_error = msg;
    return code;
}

template <typename F>
int guarded(dh2_ctx* C, F&& f) {
    try {
        f();
        return DH2_OK;
    } catch (const std::invalid_argument& e) {
        return fail(C, DH2_EINVAL, e.what());
    } catch (const CudaError& e) {
        return fail(C, DH2_ECUDA, e.what());
    } catch (const StateError& e) {
        return fail(C, DH2_ESTATE, e.what());
    } catch (const NotImpl& e) {
        return fail(C, DH2_ENOTIMPL, e.what());
    } catch (const NoMem& e) {
        return fail(C, DH2_ENOMEM, e.what());
    } catch (const std::bad_alloc& e) {
        return fail(C, DH2_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(C, DH2_ECUDA, std::string("internal error: ") + e.what());
    }
}

void storage_report(const dh2_ctx* C, int which, dh2_storage_report* out) {
    const Structure& S = C->st;
    const ClusterTree& T = S.ct;
    const int k = C->k;
    double near = 0;
    for (auto& pr : S.near) near += (double)T.size(pr.first) * T.size(pr.second) * 16.0;
    auto basis = [&](const PassH& X, bool recomp) {
        double tot = 0;
        for (size_t p = 0; p < X.bp.size(); ++p) {
            int t = C->bp_t[X.bp[p]];
            if (X.child0[p] < 0)
                tot += (double)T.size(t) * (recomp ? X.rank[p] : k);
            else if (recomp)
                tot += (double)(X.rank[X.child0[p]] + X.rank[X.child1[p]]) * X.rank[p];
            else
                tot += 2.0 * k * k;
        }
        return tot * 16.0;
    };
    const bool rc = which == DH2_RECOMP;
    out->n = C->n;
    out->row_basis_bytes = basis(C->row, rc);
    out->col_basis_bytes = basis(C->col, rc);
    double coup = 0;
    int maxr = 0;
    double sumr = 0;
    int64_t cnt = 0;
    if (rc) {
        for (size_t b = 0; b < S.blocks.size(); ++b)
            coup += (double)C->row.rank[C->blk_prow[b]] * C->col.rank[C->blk_pcol[b]] * 16.0;
        for (const PassH* X : {&C->row, &C->col})
            for (int r : X->rank) {
                maxr = std::max(maxr, r);
                sumr += r;
                ++cnt;
            }
    } else {
        coup = (double)S.blocks.size() * k * k * 16.0;
        maxr = k;
        sumr = k;
        cnt = 1;
    }
    out->coupling_bytes = coup;
    out->nearfield_bytes = near;
    out->kb_per_dof_basis = (out->row_basis_bytes + out->col_basis_bytes) / C->n / 1024.0;
    out->kb_per_dof_matrix = (out->row_basis_bytes + out->col_basis_bytes + coup + near) / C->n / 1024.0;
    out->max_rank = maxr;
    out->mean_rank = cnt ? sumr / cnt : 0.0;
}

struct ExportItem {
    const void* p;
    size_t bytes;
    bool device;
    size_t elem;
};

template <typename T>
ExportItem hv(const std::vector<T>& v) {
    return {v.data(), v.size() * sizeof(T), false, sizeof(T)};
}
template <typename T>
ExportItem dv(const DevBuf<T>& b) {
    return {b.p, b.n * sizeof(T), true, sizeof(T)};
}

}  // namespace

// ============================================================== C ABI
extern "C" {

int dh2_build_interp(const dh2_mesh* mesh, const dh2_params* params, const dh2_dist* dist, dh2_ctx** out) {
    if (out) *out = nullptr;
    if (!mesh || !params || !out) return fail(nullptr, DH2_EINVAL, "null argument");
    std::unique_ptr<dh2_ctx> C(new dh2_ctx());
    int rc = guarded(C.get(), [&] {
        const dh2_params& p = *params;
        if (!(p.kappa >= 0.0) || p.m < 1 || p.leaf_size < 1 || !(p.eta1 > 0.0) || !(p.eta2 > 0.0))
            throw std::invalid_argument("invalid parameters");
        if (p.quad != 7) throw std::invalid_argument("quad must be 7 (Radon's degree-5 rule)");
        if (p.m > 4) throw NotImpl("m > 4 (k > 64) needs the cluster/DSMEM kernels (not in this build)");
        if (mesh->nt > (int64_t)1 << 30) throw std::invalid_argument("mesh too large");
        validate_mesh(mesh->xyz, mesh->nv, mesh->tri, mesh->nt);
        if (dist && dist->world > 1) throw NotImpl("multi-GPU sharding is not in this build");
        C->device = dist ? dist->device : 0;
        const bool structure_only = C->device == DH2_DEVICE_NONE;
        if (!structure_only) {
            int ndev = 0;
            if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) throw CudaError("no CUDA device");
            CK(cudaSetDevice(C->device));
        }
        auto t0 = std::chrono::steady_clock::now();
        Params prm;
        prm.kappa = p.kappa;
        prm.m = p.m;
        prm.leaf = p.leaf_size;
        prm.eta1 = p.eta1;
        prm.eta2 = p.eta2;
        C->st.build(mesh->xyz, mesh->nv, mesh->tri, mesh->nt, prm);
        auto tt = std::chrono::steady_clock::now();
        build_tables(C.get());
        C->host_tables_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tt).count();
        C->host_build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (structure_only) return;
        CK(cudaStreamCreateWithFlags(&C->own_stream, cudaStreamNonBlocking));
        C->stream = C->own_stream;
        CK(configure_kernels());
        upload_all(C.get(), mesh->xyz, mesh->nv, mesh->tri);
        run_setup(C.get());
        C->finish();
    });
    if (rc != DH2_OK) return rc;
    *out = C.release();
    return DH2_OK;
}

int dh2_setup_device(dh2_ctx* C) {
    if (!C) return fail(nullptr, DH2_EINVAL, "null context");
    return guarded(C, [&] {
        require_device(C);
        CK(cudaSetDevice(C->device));
        run_setup(C);
        C->recompressed = false;
        C->finish();
    });
}

int dh2_recompress(dh2_ctx* C, double eps, int32_t mode) {
    if (!C) return fail(nullptr, DH2_EINVAL, "null context");
    return guarded(C, [&] {
        if (!(eps >= 0.0) || mode < 0 || mode > 2) throw std::invalid_argument("invalid eps or mode");
        require_device(C);
        CK(cudaSetDevice(C->device));
        C->eps = eps;
        C->mode = mode;
        run_recompress(C, eps, mode);
        C->finish();
        // certified sums (host reduction of the per-pair device results)
        for (PassH* X : {&C->row, &C->col}) {
            X->disc.resize(X->bp.size());
            CK(cudaMemcpy(X->disc.data(), X->d_disc.p, X->disc.size() * sizeof(double), cudaMemcpyDeviceToHost));
        }
        std::vector<double> g2(C->st.blocks.size());
        CK(cudaMemcpy(g2.data(), C->d_normG2.p, g2.size() * sizeof(double), cudaMemcpyDeviceToHost));
        C->E_row = C->E_col = C->far2 = 0;
        for (double d : C->row.disc) C->E_row += d;
        for (double d : C->col.disc) C->E_col += d;
        for (double d : g2) C->far2 += d;
        C->recompressed = true;
    });
}

int dh2_matvec(dh2_ctx* C, int32_t which, const double* x, double* y, int32_t flags) {
    if (!C) return fail(nullptr, DH2_EINVAL, "null context");
    return guarded(C, [&] {
        if (!x || !y || (which != DH2_ORIG && which != DH2_RECOMP)) throw std::invalid_argument("invalid matvec arguments");
        if (which == DH2_RECOMP && !C->recompressed) throw StateError("RECOMP matvec before dh2_recompress");
        require_device(C);
        CK(cudaSetDevice(C->device));
        const size_t nb = (size_t)C->n * sizeof(double2);
        if (flags & DH2_DEVICE_PTRS) {
            run_matvec(C, which == DH2_RECOMP, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y));
        } else {
            CK(cudaMemcpyAsync(C->d_x.p, x, nb, cudaMemcpyHostToDevice, C->stream));
            run_matvec(C, which == DH2_RECOMP, C->d_x.p, C->d_y.p);
            CK(cudaMemcpyAsync(y, C->d_y.p, nb, cudaMemcpyDeviceToHost, C->stream));
        }
        C->finish();
    });
}

int dh2_storage(const dh2_ctx* C, int32_t which, dh2_storage_report* out) {
    if (!C || !out) return fail(nullptr, DH2_EINVAL, "null argument");
    dh2_ctx* Cm = const_cast<dh2_ctx*>(C);
    return guarded(Cm, [&] {
        if (which == DH2_RECOMP && !C->recompressed) throw StateError("RECOMP storage before dh2_recompress");
        if (which != DH2_ORIG && which != DH2_RECOMP) throw std::invalid_argument("invalid which");
        storage_report(C, which, out);
    });
}

int dh2_set_stream(dh2_ctx* C, void* stream) {
    if (!C) return fail(nullptr, DH2_EINVAL, "null context");
    C->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : C->own_stream;
    return DH2_OK;
}

int dh2_set_option(dh2_ctx* C, const char* name, int64_t value) {
    if (!C || !name) return fail(nullptr, DH2_EINVAL, "null argument");
    const std::string nm(name);
    if (nm == "adjoint_symmetry") {
        if (value != 0 && value != 1) return fail(C, DH2_EINVAL, "adjoint_symmetry must be 0 or 1");
        C->sym_opt = (int)value;
        return DH2_OK;
    }
    return fail(C, DH2_EINVAL, "unknown option " + nm);
}

int dh2_set_profiling(dh2_ctx* C, int32_t enable) {
    if (!C) return fail(nullptr, DH2_EINVAL, "null context");
    C->profiling = enable != 0;
    return DH2_OK;
}

int dh2_get_stats(const dh2_ctx* C, char* buf, int64_t* len) {
    if (!C || !len) return fail(nullptr, DH2_EINVAL, "null argument");
    std::ostringstream o;
    o.precision(17);
    const Structure& S = C->st;
    int64_t nrow = (int64_t)C->row.bp.size(), ncol = (int64_t)C->col.bp.size();
    o << "{\"n\": " << C->n << ", \"k\": " << C->k << ", \"depth\": " << S.ct.depth
      << ", \"clusters\": " << C->nclusters << ", \"blocks\": " << S.blocks.size() << ", \"near\": " << S.near.size()
      << ", \"row_pairs\": " << nrow << ", \"col_pairs\": " << ncol << ", \"basis_pairs\": " << C->bp_t.size()
      << ", \"host_build_ms\": " << C->host_build_ms << ", \"host_phases_ms\": {\"tree\": " << S.ms_tree
      << ", \"dirs\": " << S.ms_dirs << ", \"blocks\": " << S.ms_blocks << ", \"closure\": " << S.ms_closure
      << ", \"tables\": " << C->host_tables_ms << "}, \"launches_total\": " << C->launches_total
      << ", \"E_row\": " << C->E_row << ", \"E_col\": " << C->E_col << ", \"far2\": " << C->far2
      << ", \"device_bytes\": " << plan_bytes(C) << ", \"mirror_missing\": " << C->mirror_missing
      << ", \"adjoint_symmetry\": {\"available\": " << (C->sym_ok ? "true" : "false") << ", \"enabled\": " << C->sym_opt
      << ", \"used\": " << (C->sym_used ? "true" : "false") << ", \"why_not\": \"" << C->sym_why << "\"}"
      << ", \"kernels\": {";
    bool first = true;
    for (auto& kv : C->kstat) {
        if (!first) o << ", ";
        first = false;
        o << "\"" << kv.first << "\": {\"launches\": " << kv.second.launches << ", \"ms\": " << kv.second.ms
          << ", \"flops\": " << kv.second.flops << ", \"bytes\": " << kv.second.bytes << "}";
    }
    o << "}}";
    std::string s = o.str();
    if (!buf) {
        *len = (int64_t)s.size() + 1;
        return DH2_OK;
    }
    if (*len < (int64_t)s.size() + 1) return fail(const_cast<dh2_ctx*>(C), DH2_EINVAL, "buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return DH2_OK;
}

int dh2_export(const dh2_ctx* C, const char* name, void* buf, int64_t* nbytes) {
    if (!C || !name || !nbytes) return fail(nullptr, DH2_EINVAL, "null argument");
    dh2_ctx* Cm = const_cast<dh2_ctx*>(C);
    return guarded(Cm, [&] {
        static thread_local std::vector<int64_t> tmp64;
        static thread_local std::vector<double> tmpd;
        const Structure& S = C->st;
        const ClusterTree& T = S.ct;
        std::string nm(name);
        // optional element slice: "<name>@<offset>:<count>"
        size_t sl_off = 0, sl_cnt = 0;
        bool sliced = false;
        const size_t at = nm.find('@');
        if (at != std::string::npos) {
            const size_t colon = nm.find(':', at);
            if (colon == std::string::npos) throw std::invalid_argument("slice syntax is name@offset:count");
            sl_off = std::stoull(nm.substr(at + 1, colon - at - 1));
            sl_cnt = std::stoull(nm.substr(colon + 1));
            nm = nm.substr(0, at);
            sliced = true;
        }
        static thread_local std::vector<double2> tmpz;
        ExportItem it{nullptr, 0, false, 1};
        auto pairs_arr = [&](const std::vector<std::vector<Pair>>& P) {
            tmp64.clear();
            for (size_t l = 0; l < P.size(); ++l)
                for (auto& pr : P[l]) {
                    tmp64.push_back((int64_t)l);
                    tmp64.push_back(pr.t);
                    tmp64.push_back(pr.c);
                }
            return hv(tmp64);
        };
        const PassH* X = nullptr;
        std::string base = nm;
        if (nm.size() > 4 && nm.compare(nm.size() - 4, 4, "_row") == 0) {
            X = &C->row;
            base = nm.substr(0, nm.size() - 4);
        } else if (nm.size() > 4 && nm.compare(nm.size() - 4, 4, "_col") == 0) {
            X = &C->col;
            base = nm.substr(0, nm.size() - 4);
        }
        if (X) {
            if (base == "bp") it = hv(X->bp);
            else if (base == "child0") it = hv(X->child0);
            else if (base == "child1") it = hv(X->child1);
            else if (base == "Z_rows") it = hv(X->Z_rows);
            else if (base == "Z_off") it = hv(X->Z_off);
            else if (base == "kb") it = hv(X->kb);
            else if (base == "rowsb") it = hv(X->rowsb);
            else if (base == "C_off") it = hv(X->C_off);
            else if (base == "Q_off") it = hv(X->Q_off);
            else if (base == "sig_off") it = hv(X->sig_off);
            else if (base == "lev_ptr") it = hv(X->lev_ptr);
            else if (base == "Z" && X == &C->col && C->sym_used) {
                // column Zhat = conj(row Zhat at -c) (k_mirror_pass); materialised here on demand,
                // only for the requested element range
                require_device(C);
                CK(cudaSetDevice(C->device));
                const size_t lo = sliced ? sl_off : 0, hi = sliced ? sl_off + sl_cnt : (size_t)C->col.Z_total;
                if (hi > (size_t)C->col.Z_total) throw std::invalid_argument("export slice out of range for " + nm);
                if (!buf) {
                    *nbytes = (int64_t)((hi - lo) * sizeof(double2));
                    return;
                }
                tmpz.assign(hi - lo, double2{0.0, 0.0});
                const auto& off = C->col.Z_off;
                size_t p = std::upper_bound(off.begin(), off.end(), (int64_t)lo) - off.begin();
                p = p ? p - 1 : 0;
                for (; p < C->col.bp.size() && (size_t)off[p] < hi; ++p) {
                    const size_t a0 = std::max((size_t)off[p], lo);
                    const size_t a1 = std::min((size_t)off[p] + (size_t)C->col.Z_rows[p] * C->k, hi);
                    if (a1 <= a0) continue;
                    const int q = C->col2row[p];
                    CK(cudaMemcpy(tmpz.data() + (a0 - lo), C->row.d_Z.p + C->row.Z_off[q] + (a0 - off[p]),
                                  (a1 - a0) * sizeof(double2), cudaMemcpyDeviceToHost));
                    for (size_t i = a0; i < a1; ++i) tmpz[i - lo].y = -tmpz[i - lo].y;
                }
                it = hv(tmpz);
                sliced = false;  // tmpz holds exactly the requested range
            } else if (base == "Z") it = dv(X->d_Z);
            else if (base == "C") it = dv(X->d_C);
            else if (base == "Q") it = dv(X->d_Q);
            else if (base == "sigma") it = dv(X->d_sigma);
            else if (base == "rank") it = dv(X->d_rank);
            else if (base == "nsig") it = dv(X->d_nsig);
            else if (base == "disc") it = dv(X->d_disc);
            else if (base == "sweeps") it = dv(X->d_sweeps);
            else throw std::invalid_argument("unknown export name " + nm);
        } else if (nm == "perm") it = hv(T.perm);
        else if (nm == "c_begin") it = hv(T.begin);
        else if (nm == "c_end") it = hv(T.end);
        else if (nm == "c_level") it = hv(T.level);
        else if (nm == "c_lo") it = hv(T.lo);
        else if (nm == "c_hi") it = hv(T.hi);
        else if (nm == "mdir") it = hv(S.mdir);
        else if (nm == "dir_off") it = hv(C->dir_off);
        else if (nm == "dirs") it = hv(C->dirs_flat);
        else if (nm == "blocks") {
            tmp64.clear();
            for (auto& b : S.blocks) {
                tmp64.push_back(b.t);
                tmp64.push_back(b.s);
                tmp64.push_back(b.c);
            }
            it = hv(tmp64);
        } else if (nm == "near") {
            tmp64.clear();
            for (auto& b : S.near) {
                tmp64.push_back(b.first);
                tmp64.push_back(b.second);
            }
            it = hv(tmp64);
        } else if (nm == "row_pairs") it = pairs_arr(S.row_pairs);
        else if (nm == "col_pairs") it = pairs_arr(S.col_pairs);
        else if (nm == "basis_pairs") it = pairs_arr(S.basis_pairs);
        else if (nm == "bp_V_off") it = hv(C->bp_V_off);
        else if (nm == "bp_R_off") it = hv(C->bp_R_off);
        else if (nm == "bp_R_rows") it = hv(C->bp_R_rows);
        else if (nm == "bp_E_off") it = hv(C->bp_E_off);
        else if (nm == "blk_St_off") it = hv(C->blk_St_off);
        else if (nm == "blk_prow") it = hv(C->blk_prow);
        else if (nm == "blk_pcol") it = hv(C->blk_pcol);
        else if (nm == "blk_mirror") it = hv(C->blk_mirror);
        else if (nm == "VR") it = dv(C->d_VR);
        else if (nm == "E") it = dv(C->d_E);
        else if (nm == "S") it = dv(C->d_S);
        else if (nm == "St") it = dv(C->d_St);
        else if (nm == "omega") it = dv(C->d_omega);
        else if (nm == "normG2") it = dv(C->d_normG2);
        else throw std::invalid_argument("unknown export name " + nm);
        if (sliced) {
            if ((sl_off + sl_cnt) * it.elem > it.bytes) throw std::invalid_argument("export slice out of range for " + nm);
            it.p = static_cast<const char*>(it.p) + sl_off * it.elem;
            it.bytes = sl_cnt * it.elem;
        }
        if (!buf) {
            *nbytes = (int64_t)it.bytes;
            return;
        }
        if (*nbytes < (int64_t)it.bytes) throw std::invalid_argument("export buffer too small for " + nm);
        if (it.bytes == 0) return;
        if (it.device) {
            require_device(C);
            CK(cudaSetDevice(C->device));
            CK(cudaMemcpy(buf, it.p, it.bytes, cudaMemcpyDeviceToHost));
        } else {
            std::memcpy(buf, it.p, it.bytes);
        }
        *nbytes = (int64_t)it.bytes;
        (void)tmpd;
    });
}

int dh2_destroy(dh2_ctx* C) {
    if (!C) return DH2_OK;
    if (C->device != DH2_DEVICE_NONE) {
        cudaSetDevice(C->device);
        if (C->stream) cudaStreamSynchronize(C->stream);
    }
    delete C;
    return DH2_OK;
}

const char* dh2_last_error(const dh2_ctx* C) {
    if (C) return C->err.c_str();
    return g_last_error.c_str();
}

}  // extern "C"
