// C-ABI implementation of libdh2.so (include/dh2.h): host structure -> device tables ->
// level-batched sm_100a kernels.  No CPU fallback: every compute step runs on the GPU.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <numeric>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <exception>
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
#include "dh2_shard.h"

namespace dh2 {
cudaError_t configure_kernels();
}

using namespace dh2;

namespace {

std::string g_last_error;

}  // namespace

namespace {

inline uint64_t key(int64_t t, int64_t c) { return ((uint64_t)t << 32) | (uint64_t)c; }

// Adjoint symmetry of the single-layer DH^2 (W = V; column pass =
// row pass on G^*).  With antipodal direction sets (DESIGN R2/R4), V_{s,-c} =
// conj(V_{s,c}), E likewise, and the mirror block (s,t,-c) has S = S_b^T.  The column-pass
// matrix of (s,c), rows w_b R_tc S_b over t in col(s,c) plus inherited E Zhat'^*, is then the
// complex conjugate of the row-pass matrix of (s,-c), so Zhat', sigma', k', Q', F', C' are
// the conjugates of the row results at (s,-c).  This checks that the structure has exactly
// that correspondence (pairs, blocks, parents, children, bounds); otherwise two passes run.
void check_symmetry(Shard* C) {
    Structure& S = C->st;
    const int L = S.ct.depth;
    const PassH &R = C->row, &X = C->col;
    C->sym_ok = false;
    C->col2row.clear();
    if (C->mirror_missing) { C->sym_why = "blocks without an antipodal mirror"; return; }
    if (R.bp.size() != X.bp.size()) { C->sym_why = "row and column pair counts differ"; return; }

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
        const int nid = nc < 0 ? -1 : C->bp_find(C->bp_t[id], nc);
        const int q = nid < 0 ? -1 : R.bp2p[nid];
        if (q < 0) { C->sym_why = "column pair without a row pair at -c"; return; }
        c2r[p] = q;
    }
    // per-pair comparisons in parallel (read-only); the first failing pair in index order names the reason
    const int64_t npairs = (int64_t)X.bp.size();
    std::vector<const char*> why(npairs, nullptr);
    std::atomic<bool> bad{false};
#pragma omp parallel
    {
        std::vector<int> a, b, pa, pb;  // scratch, reused across pairs
#pragma omp for schedule(dynamic, 512)
        for (int64_t p = 0; p < npairs; ++p) {
            if (bad.load(std::memory_order_relaxed)) continue;
            const int q = c2r[p];
            const char* w = nullptr;
            if (X.Z_rows[p] != R.Z_rows[q] || X.total_rows[p] != R.total_rows[q] || X.kb[p] != R.kb[q] ||
                X.rowsb[p] != R.rowsb[q])
                w = "bounds differ";
            else if ((X.child0[p] < 0) != (R.child0[q] < 0))
                w = "leaf mismatch";
            else if (X.child0[p] >= 0 && (c2r[X.child0[p]] != R.child0[q] || c2r[X.child1[p]] != R.child1[q]))
                w = "children differ";
            if (!w) {
                a.clear();
                b.clear();
                for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) a.push_back(C->blk_mirror[X.blk[ib]]);
                for (int ib = R.blk_ptr[q]; ib < R.blk_ptr[q + 1]; ++ib) b.push_back(R.blk[ib]);
                std::sort(a.begin(), a.end());
                std::sort(b.begin(), b.end());
                if (a != b) w = "block sets differ";
            }
            if (!w) {
                pa.clear();
                pb.clear();
                for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) pa.push_back(c2r[X.par[ip]] * 2 + X.par_child[ip]);
                for (int ip = R.par_ptr[q]; ip < R.par_ptr[q + 1]; ++ip) pb.push_back(R.par[ip] * 2 + R.par_child[ip]);
                std::sort(pa.begin(), pa.end());
                std::sort(pb.begin(), pb.end());
                if (pa != pb) w = "parents differ";
            }
            if (w) {
                why[p] = w;
                bad.store(true, std::memory_order_relaxed);
            }
        }
    }
    if (bad.load()) {
        for (int64_t p = 0; p < npairs; ++p)
            if (why[p]) { C->sym_why = why[p]; return; }
    }
    C->col2row.swap(c2r);
    C->sym_ok = true;
    C->sym_why.clear();
}

// Ownership of clusters for sharding: cut level log2(world); the subtree of the
// r-th cluster of the cut level belongs to shard r.  Every active level must lie on or below the
// cut (the replicated top carries no recompression work); blocks are re-ordered by the owner of
// their row cluster (stable, so world == 1 keeps the structure's order).
void assign_owners(Shard* C) {
    Structure& S = C->st;
    const ClusterTree& T = S.ct;
    const int L = T.depth;
    C->cut = 0;
    while ((1 << C->cut) < C->world) ++C->cut;
    if ((1 << C->cut) != C->world) throw std::invalid_argument("world size must be a power of two");
    if (C->rank < 0 || C->rank >= C->world) throw std::invalid_argument("rank out of range");
    if (C->cut > L || (int)T.levels[C->cut].size() != C->world)
        throw NotImpl("the cluster tree has fewer than world clusters on level log2(world)");
    for (int l = 0; l < C->cut; ++l)
        if (!S.basis_pairs[l].empty())
            throw NotImpl("active pairs above the cut level log2(world) (direction split not implemented)");
    C->owner.assign(T.begin.size(), -1);
    for (int i = 0; i < C->world; ++i) C->owner[T.levels[C->cut][i]] = i;
    for (int l = C->cut + 1; l <= L; ++l)
        for (int64_t t : T.levels[l]) C->owner[t] = C->owner[T.parent[t]];
    if (C->world > 1) {
        const auto& own = C->owner;
        std::stable_sort(S.blocks.begin(), S.blocks.end(), [&](const Block& a, const Block& b) { return own[a.t] < own[b.t]; });
    }
    const int64_t top = T.levels[C->cut][C->rank];
    C->pos_lo = T.begin[top];
    C->pos_hi = T.end[top];
}

void build_tables(Shard* C) {
    Structure& S = C->st;
    const ClusterTree& T = S.ct;
    const int k = S.k, L = T.depth;
    C->n = (int)T.n;
    C->k = k;
    C->m = S.p.m;
    C->nclusters = (int)T.begin.size();
    using tclk = std::chrono::steady_clock;
    auto tmark = tclk::now();
    auto tick = [&](int i) {
        auto now = tclk::now();
        C->tab_ms[i] += std::chrono::duration<double, std::milli>(now - tmark).count();
        tmark = now;
    };
    assign_owners(C);
    const int me = C->rank, W = C->world;
    const auto& own = C->owner;
    // directions of the materialised levels
    C->dir_off.assign(L + 2, -1);
    for (int l = 0; l <= L; ++l) {
        if (S.basis_pairs[l].empty()) continue;
        C->dir_off[l] = (int64_t)C->dirs_flat.size() / 3;
        const auto& D = S.D(l);
        C->dirs_flat.insert(C->dirs_flat.end(), D.begin(), D.end());
    }
    // basis pairs (global ids, level by level)
    C->bp_lev_ptr.assign(L + 2, 0);
    for (int l = 0; l <= L; ++l) {
        C->bp_lev_ptr[l] = (int)C->bp_t.size();
        for (const Pair& pr : S.basis_pairs[l]) {
            int id = (int)C->bp_t.size();
            C->bp_t.push_back((int)pr.t);
            C->bp_c.push_back((int)pr.c);
            C->bp_level.push_back(l);
            C->bp_dir.push_back((int)(C->dir_off[l] + pr.c));
        }
    }
    C->bp_lev_ptr[L + 1] = (int)C->bp_t.size();
    const int nbp = (int)C->bp_t.size();
    // clusters are numbered level by level (BFS) and pairs sorted by (t, c) within a level, so
    // the pairs of one cluster are contiguous
    C->bp_cl.assign(C->nclusters + 1, 0);
    for (int id = 0; id < nbp; ++id) ++C->bp_cl[C->bp_t[id] + 1];
    for (int t = 0; t < C->nclusters; ++t) C->bp_cl[t + 1] += C->bp_cl[t];
    for (int id = 1; id < nbp; ++id)
        if (C->bp_t[id] < C->bp_t[id - 1]) throw std::logic_error("basis pairs not grouped by cluster");
    C->bp_child0.assign(nbp, -1);
    C->bp_child1.assign(nbp, -1);
    C->bp_sddir.assign(nbp, -1);
    C->bp_V_off.assign(nbp, -1);
    C->bp_R_off.assign(nbp, -1);
    C->bp_E_off.assign(nbp, -1);
    C->bp_R_rows.assign(nbp, 0);
    C->bp_own.assign(nbp, 0);
    C->leafV_lists.assign(L + 1, {});
    C->basis_lists.assign(L + 1, {});
    C->E_lists.assign(L + 1, {});
    C->basis_maxrows.assign(L + 1, 0);
    for (int id = 0; id < nbp; ++id) {
        int t = C->bp_t[id], l = C->bp_level[id];
        C->bp_own[id] = own[t] == me;
        if (!T.is_leaf(t)) {
            int64_t c2 = S.sd(l, C->bp_c[id]);
            C->bp_sddir[id] = (int)(C->dir_off[l + 1] + c2);
            C->bp_child0[id] = C->bp_at(T.child0[t], c2);
            C->bp_child1[id] = C->bp_at(T.child1[t], c2);
        }
    }
    // (t,-c) of every basis pair (antipodal direction sets, DESIGN R2/R4)
    C->bp_neg.assign(nbp, -1);
    for (int l = 0; l <= L; ++l) {
        if (S.basis_pairs[l].empty()) continue;
        const auto& D = S.D(l);
        const int nd = (int)D.size() / 3;
        std::map<std::tuple<double, double, double>, int> idx;
        for (int c = 0; c < nd; ++c) idx[{D[3 * c] + 0.0, D[3 * c + 1] + 0.0, D[3 * c + 2] + 0.0}] = c;
        std::vector<int> neg(nd, -1);
        for (int c = 0; c < nd; ++c) {
            auto it = idx.find({-D[3 * c] + 0.0, -D[3 * c + 1] + 0.0, -D[3 * c + 2] + 0.0});
            if (it != idx.end()) neg[c] = it->second;
        }
        for (int id = C->bp_lev_ptr[l]; id < C->bp_lev_ptr[l + 1]; ++id) {
            const int nc = neg[C->bp_c[id]];
            C->bp_neg[id] = nc < 0 ? -1 : C->bp_find(C->bp_t[id], nc);
        }
    }
    // basis-weight rows, bottom-up (Eq. 18): leaf min(#t, k) (R = V if #t <= k), inner min(r1 + r2, k)
    for (int l = L; l >= 0; --l)
        for (int id = C->bp_lev_ptr[l]; id < C->bp_lev_ptr[l + 1]; ++id) {
            const int t = C->bp_t[id];
            const int rows = T.is_leaf(t) ? (int)T.size(t) : C->bp_R_rows[C->bp_child0[id]] + C->bp_R_rows[C->bp_child1[id]];
            C->bp_R_rows[id] = std::min(rows, k);
        }
    auto r_by_qr = [&](int id) { return !T.is_leaf(C->bp_t[id]) || T.size(C->bp_t[id]) > k; };
    tick(0);
    // blocks (global ids; own range contiguous after assign_owners)
    const int nb = (int)S.blocks.size();
    C->b_lo = nb;
    C->b_hi = 0;
    for (int b = 0; b < nb; ++b) {
        const Block& B = S.blocks[b];
        int l = (int)T.level[B.t];
        C->blk_t.push_back((int)B.t);
        C->blk_s.push_back((int)B.s);
        C->blk_dir.push_back((int)(C->dir_off[l] + B.c));
        C->blk_bprow.push_back(C->bp_at(B.t, B.c));
        C->blk_bpcol.push_back(C->bp_at(B.s, B.c));
        C->blk_bpcs.push_back(C->bp_neg[C->blk_bpcol.back()]);
        if (own[B.t] == me) {
            C->b_lo = std::min(C->b_lo, b);
            C->b_hi = std::max(C->b_hi, b + 1);
        }
    }
    if (C->b_lo >= C->b_hi) C->b_lo = C->b_hi = 0;
    for (int b = C->b_lo; b < C->b_hi; ++b)
        if (own[S.blocks[b].t] != me) throw std::logic_error("own blocks not contiguous");
    // basis pairs needed here: own ones, plus the column pairs of own blocks owned elsewhere
    // (imported: R received if computed by QR, else R = V regenerated from the replicated mesh)
    std::vector<char> need(C->bp_own.begin(), C->bp_own.end());
    for (int b = C->b_lo; b < C->b_hi; ++b) {
        need[C->blk_bpcol[b]] = 1;
        if (C->blk_bpcs[b] >= 0) need[C->blk_bpcs[b]] = 1;  // column side under the adjoint symmetry
    }
    int64_t off = 0;
    for (int id = 0; id < nbp; ++id) {
        if (!need[id]) continue;
        const int t = C->bp_t[id], l = C->bp_level[id];
        if (T.is_leaf(t) && (C->bp_own[id] || !r_by_qr(id))) {  // V slab
            const int sz = (int)T.size(t);
            C->max_leaf = std::max(C->max_leaf, sz);
            C->bp_V_off[id] = off;
            off += (int64_t)sz * k;
            C->leafV_lists[l].push_back(id);
        }
        if (C->bp_own[id] && !T.is_leaf(t)) C->E_lists[l].push_back(id);
    }
    for (int l = L; l >= 0; --l)
        for (int id = C->bp_lev_ptr[l]; id < C->bp_lev_ptr[l + 1]; ++id) {
            if (!need[id]) continue;
            if (!r_by_qr(id)) {
                C->bp_R_off[id] = C->bp_V_off[id];  // R = V, P = I (Eq. 18)
                continue;
            }
            C->bp_R_off[id] = off;
            off += (int64_t)C->bp_R_rows[id] * k;
            if (C->bp_own[id]) {
                C->basis_lists[l].push_back(id);
                const int t = C->bp_t[id];
                const int rows = T.is_leaf(t) ? (int)T.size(t) : C->bp_R_rows[C->bp_child0[id]] + C->bp_R_rows[C->bp_child1[id]];
                C->basis_maxrows[l] = std::max(C->basis_maxrows[l], rows);
            }
        }
    C->VR_total = off;
    int64_t eoff = 0;
    for (int id = 0; id < nbp; ++id)
        if (C->bp_own[id] && C->bp_child0[id] >= 0) {
            C->bp_E_off[id] = eoff;
            eoff += 6LL * C->m * C->m;
        }
    C->E_total = eoff;
    tick(1);
    // passes (global pair ids; per-pair slabs only for the pairs this shard computes or imports);
    // the two sides are independent (sd() values are all cached by the basis-pair pass above)
    C->blk_prow.clear();
    C->blk_pcol.clear();
    std::exception_ptr side_err[2];
#pragma omp parallel for num_threads(2) schedule(static, 1)
    for (int side = 0; side < 2; ++side) try {
        PassH& X = side == 0 ? C->row : C->col;
        const auto& pairs = side == 0 ? S.row_pairs : S.col_pairs;
        X.bp2p.assign(nbp, -1);
        X.lev_ptr.assign(L + 2, 0);
        for (int l = 0; l <= L; ++l) {
            X.lev_ptr[l] = (int)X.bp.size();
            for (const Pair& pr : pairs[l]) {
                const int id = C->bp_at(pr.t, pr.c);
                X.bp2p[id] = (int)X.bp.size();
                X.bp.push_back(id);
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
                X.child0[p] = X.bp2p[C->bp_child0[id]];
                X.child1[p] = X.bp2p[C->bp_child1[id]];
                if (X.child0[p] < 0 || X.child1[p] < 0) throw std::logic_error("pass closure broken");
            }
        }
        // blocks CSR (blocks sorted by (t,s) per owner: per pair sorted by the other cluster)
        // (counting sort into the CSR, then each pair's few blocks by the other cluster)
        std::vector<int>& bpp = side == 0 ? C->blk_prow : C->blk_pcol;
        bpp.resize(nb);
        X.blk_ptr.assign(np + 1, 0);
        for (int b = 0; b < nb; ++b) {
            int p = X.bp2p[side == 0 ? C->blk_bprow[b] : C->blk_bpcol[b]];
            if (p < 0) throw std::logic_error("block pair missing from the pass");
            bpp[b] = p;
            ++X.blk_ptr[p + 1];
        }
        for (int p = 0; p < np; ++p) X.blk_ptr[p + 1] += X.blk_ptr[p];
        X.blk.assign(nb, 0);
        {
            std::vector<int> pos(X.blk_ptr.begin(), X.blk_ptr.end() - 1);
            for (int b = 0; b < nb; ++b) X.blk[pos[bpp[b]]++] = b;
        }
        for (int p = 0; p < np; ++p)
            std::sort(X.blk.begin() + X.blk_ptr[p], X.blk.begin() + X.blk_ptr[p + 1], [&](int a, int b) {
                const Block &A = S.blocks[a], &B = S.blocks[b];
                return side == 0 ? (A.s < B.s || (A.s == B.s && a < b)) : (A.t < B.t || (A.t == B.t && a < b));
            });
        // parents CSR: (t+, c+) -> children (t_i, sd(c+)), parents in increasing order
        X.par_ptr.assign(np + 1, 0);
        for (int p = 0; p < np; ++p) {
            if (X.child0[p] < 0) continue;
            ++X.par_ptr[X.child0[p] + 1];
            ++X.par_ptr[X.child1[p] + 1];
        }
        for (int p = 0; p < np; ++p) X.par_ptr[p + 1] += X.par_ptr[p];
        X.par.assign(X.par_ptr[np], 0);
        X.par_child.assign(X.par_ptr[np], 0);
        {
            std::vector<int> pos(X.par_ptr.begin(), X.par_ptr.end() - 1);
            for (int p = 0; p < np; ++p) {
                if (X.child0[p] < 0) continue;
                for (int ci = 0; ci < 2; ++ci) {
                    const int q = pos[ci ? X.child1[p] : X.child0[p]]++;
                    X.par[q] = p;
                    X.par_child[q] = ci;
                }
            }
        }
        // Zhat rows, top-down
        X.Z_rows.assign(np, 0);
        X.total_rows.assign(np, 0);
        X.lev_max_total.assign(L + 1, 0);
        X.lev_max_zrows.assign(L + 1, 0);
        X.lev_max_leafrows.assign(L + 1, 0);
        X.own_lo.assign(L + 1, 0);
        X.own_hi.assign(L + 1, 0);
        for (int l = 0; l <= L; ++l) {
            int lo = X.lev_ptr[l + 1], hi = X.lev_ptr[l];
            for (int p = X.lev_ptr[l]; p < X.lev_ptr[l + 1]; ++p) {
                int tot = 0;
                for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
                    int b = X.blk[ib];
                    tot += C->bp_R_rows[side == 0 ? C->blk_bpcol[b] : C->blk_bprow[b]];
                }
                for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) tot += X.Z_rows[X.par[ip]];
                X.total_rows[p] = tot;
                X.Z_rows[p] = std::min(tot, k);
                if (own[C->bp_t[X.bp[p]]] != me) continue;
                lo = std::min(lo, p);
                hi = std::max(hi, p + 1);
                X.lev_max_total[l] = std::max(X.lev_max_total[l], tot);
                X.lev_max_zrows[l] = std::max(X.lev_max_zrows[l], X.Z_rows[p]);
            }
            if (lo >= hi) lo = hi = X.lev_ptr[l];
            for (int p = lo; p < hi; ++p)
                if (own[C->bp_t[X.bp[p]]] != me) throw std::logic_error("own pairs of a level not contiguous");
            X.own_lo[l] = lo;
            X.own_hi[l] = hi;
        }
        // rank bounds, bottom-up
        X.rowsb.assign(np, 0);
        X.kb.assign(np, 0);
        for (int l = L; l >= 0; --l)
            for (int p = X.lev_ptr[l]; p < X.lev_ptr[l + 1]; ++p) {
                int t = C->bp_t[X.bp[p]];
                X.rowsb[p] = X.child0[p] < 0 ? (int)T.size(t) : X.kb[X.child0[p]] + X.kb[X.child1[p]];
                X.kb[p] = std::min(X.rowsb[p], X.Z_rows[p]);
                if (X.child0[p] < 0 && own[t] == me) X.lev_max_leafrows[l] = std::max(X.lev_max_leafrows[l], (int)T.size(t));
            }
        // slabs: own pairs (Z, C, Q, sigma); column pairs of own blocks owned elsewhere (C' only)
        std::vector<char> imp(np, 0);
        if (side == 1)
            for (int b = C->b_lo; b < C->b_hi; ++b)
                if (own[C->blk_s[b]] != me) imp[C->blk_pcol[b]] = 1;
        X.Z_off.assign(np, -1);
        X.C_off.assign(np, -1);
        X.Q_off.assign(np, -1);
        X.sig_off.assign(np, -1);
        for (int p = 0; p < np; ++p) {
            const bool mine = own[C->bp_t[X.bp[p]]] == me;
            if (mine) {
                X.Z_off[p] = X.Z_total;
                X.Z_total += (int64_t)X.Z_rows[p] * k;
                X.Q_off[p] = X.Q_total;
                X.Q_total += (int64_t)X.rowsb[p] * X.kb[p];
                X.sig_off[p] = X.sig_total;
                X.sig_total += X.kb[p];
            }
            if (mine || imp[p]) {
                X.C_off[p] = X.C_total;
                X.C_total += (int64_t)X.kb[p] * k;
            }
        }
        // leaf-cluster groups (contiguous pairs of one leaf cluster)
        X.lc_ptr.push_back(0);
        int lastt = -1;
        X.lc_lo = -1;
        for (int p = 0; p < np; ++p) {
            int t = C->bp_t[X.bp[p]];
            if (!T.is_leaf(t)) continue;
            if (t != lastt && !X.lc.empty()) X.lc_ptr.push_back((int)X.lc.size());
            if (t != lastt && own[t] == me) {
                const int g = (int)X.lc_ptr.size() - 1;
                if (X.lc_lo < 0) X.lc_lo = g;
                X.lc_hi = g + 1;
            }
            X.lc.push_back(p);
            lastt = t;
        }
        if (!X.lc.empty()) X.lc_ptr.push_back((int)X.lc.size());
        if (X.lc_lo < 0) X.lc_lo = X.lc_hi = 0;
    } catch (...) {
        side_err[side] = std::current_exception();
    }
    for (auto& e : side_err)
        if (e) std::rethrow_exception(e);
    tick(2);
    // antipodal mirror b' = (s, t, -c) of every block: S_{b'} = S_b^T exactly (DESIGN §total weights)
    {
        // block ids ordered by (t, s) (the structure's order unless re-ordered by owner)
        std::vector<int> ord(nb);
        std::iota(ord.begin(), ord.end(), 0);
        auto ts_less = [&](int a, int b) {
            const Block &A = S.blocks[a], &B = S.blocks[b];
            return A.t < B.t || (A.t == B.t && A.s < B.s);
        };
        if (!std::is_sorted(ord.begin(), ord.end(), ts_less)) std::sort(ord.begin(), ord.end(), ts_less);
        C->blk_mirror.assign(nb, -1);
        for (int b = 0; b < nb; ++b) {
            const Block& B = S.blocks[b];
            auto it = std::lower_bound(ord.begin(), ord.end(), 0, [&](int a, int) {
                const Block& A = S.blocks[a];
                return A.t < B.s || (A.t == B.s && A.s < B.t);
            });
            if (it == ord.end() || S.blocks[*it].t != B.s || S.blocks[*it].s != B.t) { ++C->mirror_missing; continue; }
            int l = (int)T.level[B.t];
            const auto& D = S.D(l);
            int64_t c2 = S.blocks[*it].c;
            bool neg = D[3 * c2] == -D[3 * B.c] && D[3 * c2 + 1] == -D[3 * B.c + 1] && D[3 * c2 + 2] == -D[3 * B.c + 2];
            if (neg) C->blk_mirror[b] = *it; else ++C->mirror_missing;
        }
    }
    tick(3);
    check_symmetry(C);
    if (C->sym_ok) {
        PassH &R = C->row, &X = C->col;
        const int np = (int)X.bp.size();
        X.C_off_own = X.C_off;
        X.Q_off_own = X.Q_off;
        X.sig_off_own = X.sig_off;
        X.C_off_alias.assign(np, -1);
        X.Q_off_alias.assign(np, -1);
        X.sig_off_alias.assign(np, -1);
        X.C_imp_total = 0;
        for (int p = 0; p < np; ++p) {
            if (X.C_off[p] < 0) continue;
            if (X.Q_off[p] >= 0) {  // own pair: the row pair at -c
                const int q = C->col2row[p];
                X.C_off_alias[p] = R.C_off[q];
                X.Q_off_alias[p] = R.Q_off[q];
                X.sig_off_alias[p] = R.sig_off[q];
            } else {  // imported C' (partition), after the row C pool
                X.C_off_alias[p] = R.C_total + X.C_imp_total;
                X.C_imp_total += (int64_t)X.kb[p] * k;
            }
        }
        R.C_extra = X.C_imp_total;
        X.alias = true;
        X.C_off = X.C_off_alias;
        X.Q_off = X.Q_off_alias;
        X.sig_off = X.sig_off_alias;
        // row basis pairs only (own), plus the (s,-c) of own blocks whose column cluster is elsewhere
        std::vector<char> need_sym(nbp, 0);
        for (int id = 0; id < nbp; ++id) need_sym[id] = C->bp_own[id] && R.bp2p[id] >= 0;
        for (int b = C->b_lo; b < C->b_hi; ++b) {
            if (C->blk_bpcs[b] < 0) throw std::logic_error("column pair without (s,-c) on a symmetric structure");
            need_sym[C->blk_bpcs[b]] = 1;
        }
        C->leafV_lists_sym.assign(L + 1, {});
        C->basis_lists_sym.assign(L + 1, {});
        C->E_lists_sym.assign(L + 1, {});
        for (int l = 0; l <= L; ++l) {
            for (int id : C->leafV_lists[l])
                if (need_sym[id]) C->leafV_lists_sym[l].push_back(id);
            for (int id : C->basis_lists[l])
                if (R.bp2p[id] >= 0) C->basis_lists_sym[l].push_back(id);
            for (int id : C->E_lists[l])
                if (R.bp2p[id] >= 0) C->E_lists_sym[l].push_back(id);
        }
    }
    tick(4);
    if (W > 1 && !C->sym_ok)
        throw NotImpl("sharding needs the adjoint-symmetric structure (" + C->sym_why + ")");
    C->blk_St_off.assign(nb, -1);
    for (int b = C->b_lo; b < C->b_hi; ++b) {
        C->blk_St_off[b] = C->St_total;
        C->St_total += (int64_t)C->row.kb[C->blk_prow[b]] * C->col.kb[C->blk_pcol[b]];
    }
    // exchange lists: for a block (t,s,c) with owner(t) != owner(s), owner(s)
    // sends R_sc (if computed by QR) and the column results C'_sc, k'_sc (and xh'_sc in matvec)
    C->R_send.assign(W, {});
    C->R_recv.assign(W, {});
    C->C_send.assign(W, {});
    C->C_recv.assign(W, {});
    for (int b = 0; b < nb; ++b) {
        const int rt = own[C->blk_t[b]], rs = own[C->blk_s[b]];
        if (rt == rs || (rt != me && rs != me)) continue;
        const int bp = C->blk_bpcs[b], p = C->blk_pcol[b];  // R of (s,-c): the column side is its conjugate
        if (rs == me) {
            if (r_by_qr(bp)) C->R_send[rt].push_back(bp);
            C->C_send[rt].push_back(p);
        } else {
            if (r_by_qr(bp)) C->R_recv[rs].push_back(bp);
            C->C_recv[rs].push_back(p);
        }
    }
    for (auto* v : {&C->R_send, &C->R_recv, &C->C_send, &C->C_recv})
        for (auto& l : *v) {
            std::sort(l.begin(), l.end());
            l.erase(std::unique(l.begin(), l.end()), l.end());
        }
    tick(5);
}

void upload_pass(Shard* C, PassH& X, PassD& D, bool alloc_Z) {
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
    if (alloc_Z && !C->lean.on) X.d_Z.alloc(X.Z_total);
    if (!X.alias) {  // (aliased column factors live in the row pools)
        if (!C->lean.on) {  // lean plan: C, Q in growable pools (lean_alloc)
            X.d_C.alloc(X.C_total + X.C_extra);
            X.d_Q.alloc(X.Q_total);
        }
        X.d_sigma.alloc(X.sig_total);
        // slots past a pair's nsig (pivoted-QR rank stop, N1) are never written: zero, not pool garbage
        if (X.sig_total) CK(cudaMemsetAsync(X.d_sigma.p, 0, X.sig_total * sizeof(double), s));
    }
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

size_t plan_bytes(const Shard* C) {
    if (C->lean.on) return (size_t)lean_bytes(C);
    size_t b = 0;
    b += (size_t)C->VR_total * 16 + (size_t)C->E_total * 16 + (size_t)(C->b_hi - C->b_lo) * C->k * C->k * 16;
    b += (size_t)C->St_total * 16;
    for (const PassH* X : {&C->row, &C->col})
        if (X->alias)
            b += 0;  // column factors read from the row pools (imports counted in row C_extra)
        else
            b += (size_t)((X == &C->col && C->sym_ok ? 0 : X->Z_total) + X->C_total + X->C_extra + X->Q_total) * 16 +
                 (size_t)X->sig_total * 8;
    b += (size_t)C->n * 7 * 32 + (size_t)C->nclusters * sizeof(GridD);
    b += cq_scratch_bytes_bound(C->k);
    return b;
}

// The full plan materialises V, S and every factor; when it does not fit (or when forced), the
// memory-lean chunked plan is used instead (dh2_lean.cu), with the smallest number of chunks whose
// estimate fits.
void choose_plan(Shard* C) {
    size_t freeb = 0, totb = 0;
    CK(cudaMemGetInfo(&freeb, &totb));
    freeb += pool_reusable(C->device);
    const size_t margin = (size_t)2 << 30;
    if (C->lean.on) {
        if ((size_t)lean_bytes(C) + margin > freeb)
            throw NoMem("lean device memory plan needs " + std::to_string((size_t)lean_bytes(C) >> 20) + " MiB, free " +
                        std::to_string(freeb >> 20) + " MiB");
        return;
    }
    const size_t need = plan_bytes(C);
    if (!C->lean_required && need + (size_t)256 * 1024 * 1024 <= freeb) return;
    const std::string full = "device memory plan needs " + std::to_string(need >> 20) + " MiB, free " + std::to_string(freeb >> 20) + " MiB";
    if (!C->sym_ok) throw NoMem(full + " (the memory-lean plan needs the adjoint symmetry)");
    const int ntop = (int)C->st.ct.levels[std::max(0, C->st.first_level)].size();
    for (int G = 1;; G *= 2) {  // (the estimate guesses the ranks: keep 15 % in reserve)
        lean_plan(C, G);
        if ((size_t)lean_bytes(C) + margin <= (size_t)(0.85 * freeb)) return;
        if (G >= ntop) break;
    }
    throw NoMem(full + "; the memory-lean plan needs " + std::to_string((size_t)lean_bytes(C) >> 20) + " MiB with " +
                std::to_string(C->lean.G) + " chunks");
}

void upload_all(Shard* C, const double* xyz, int64_t nv, const int64_t* tri) {
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    choose_plan(C);
    if (xyz) {  // (a re-layout keeps the device mesh)
        C->d_xyz.upload(std::vector<double>(xyz, xyz + 3 * nv), s);
        C->d_tri.upload(std::vector<int64_t>(tri, tri + 3 * C->n), s);
    }
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
    {
        // mirror reads only where the mirror block is this shard's (else the strided S_b read)
        std::vector<int> mir(C->blk_mirror);
        for (int& b : mir)
            if (b < C->b_lo || b >= C->b_hi) b = -1;
        C->d_blk_mirror.upload(mir, s);
    }
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
        if (C->sym_ok) {
            C->d_leafV_list_sym.push_back(up_list(C->leafV_lists_sym[l]));
            C->d_basis_list_sym.push_back(up_list(C->basis_lists_sym[l]));
            C->d_E_list_sym.push_back(up_list(C->E_lists_sym[l]));
        }
    }
    C->d_blk_bpcs.upload(C->blk_bpcs, s);
    C->d_qp.alloc((size_t)C->n * 7);
    C->d_grid.alloc(C->nclusters);
    C->d_VR.alloc(C->VR_total);
    C->d_E.alloc(C->E_total);
    const size_t nb = C->st.blocks.size();
    if (!C->lean.on) {  // (lean: S per chunk, S~ once the ranks are known)
        C->d_S.alloc((size_t)(C->b_hi - C->b_lo) * C->k * C->k);  // own blocks only
        C->d_St.alloc(C->St_total);
    }
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
    P.blk_bpcs = C->d_blk_bpcs.p;
    P.blk_prow = C->d_blk_prow.p;
    P.blk_pcol = C->d_blk_pcol.p;
    P.blk_St_off = C->d_blk_St_off.p;
    {  // S slots: own blocks in order (slot b - b_lo)
        std::vector<int> slot(nb, 0);
        for (int b = C->b_lo; b < C->b_hi; ++b) slot[b] = b - C->b_lo;
        C->d_blk_slot.upload(slot, s);
    }
    P.blk_slot = C->d_blk_slot.p;
    P.S = C->d_S.p;
    P.St = C->d_St.p;
    P.omega = C->d_omega.p;
    P.normG2 = C->d_normG2.p;
    upload_pass(C, C->row, P.row, true);
    upload_pass(C, C->col, P.col, !C->sym_ok);  // column Zhat only when two passes can run
    if (C->col.alias) {
        P.col.C = P.row.C;
        P.col.Q = P.row.Q;
        P.col.sigma = P.row.sigma;
    }
    P.col_conj = C->col.alias ? 1 : 0;
    if (C->sym_ok) C->d_col2row.upload(C->col2row, s);
    P.col2row = C->d_col2row.p;
    // set-up of the row basis pairs only when the column side can be read by conjugation
    P.sym = (C->sym_ok && C->sym_opt) ? 1 : 0;
    P.qr_wy = C->qr_wy_init;
    P.qr_flag = C->qr_flag_init;
    P.trunc_mode = C->trunc_mode_init;
    P.qr_cq = C->qr_cq_init;
    P.t64_threads = C->t64_threads_init;
    P.bw_variant = C->bw_variant_init;
    P.mv_fwd_warp = C->mv_fwd_warp_init;
    P.qr_cq_tw = C->qr_cq_tw_init;
    P.qr_cq_tw_leaf = C->qr_cq_tw_leaf_init;
    P.qr_cq64 = C->qr_cq64_init;
    P.qr_cq64_tw = C->qr_cq64_tw_init;
    if (P.k <= 128) {
        C->d_cq.alloc(cq_scratch_elems(P));
        P.cq_scr = C->d_cq.p;
    } else {
        P.cq_scr = nullptr;
    }
    if (C->lean.on) lean_alloc(C);
}

// Device set-up (§2): quadrature points, grids, leaf V, E factors, S.
void run_setup(Shard* C) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const int L = C->st.ct.depth;
    const int k = C->k;
    C->timed("setup_quad", 2, [&] { launch_quad(P, s); });
    C->timed("setup_grid", 1, [&] { launch_grid(P, s); });
    // adjoint symmetry: V and E of the row basis pairs only (the column side is read conjugated)
    const bool sym = P.sym && !C->col_data;
    C->sym_setup = sym;
    for (int l = 0; l <= L; ++l) {
        const auto& lv = sym ? C->leafV_lists_sym[l] : C->leafV_lists[l];
        int nl = C->lean.on ? 0 : (int)lv.size();  // lean plan: leaf V per chunk inside the recompression
        if (nl) {
            C->timed("setup_leafV", 1, [&] { launch_leafV(P, sym ? C->d_leafV_list_sym[l] : C->d_leafV_list[l], nl, C->max_leaf, s); });
            double ent = 0;
            for (int id : lv) ent += (double)C->st.ct.size(C->bp_t[id]) * k;
            auto& st = C->kstat["setup_leafV"];
            st.flops += ent * 7 * 6;
            st.bytes += ent * 16 + ent / k * 7 * 32;
        }
        int ne = (int)(sym ? C->E_lists_sym[l] : C->E_lists[l]).size();
        if (ne) {
            C->timed("setup_E", 1, [&] { launch_E(P, sym ? C->d_E_list_sym[l] : C->d_E_list[l], ne, s); });
            C->kstat["setup_E"].bytes += (double)ne * 6 * C->m * C->m * 16;
        }
    }
    if (!sym) C->col_data = true;
    if (C->lean.on) return;  // S_b per chunk inside the recompression
    const int nb = C->b_hi - C->b_lo;
    C->timed("setup_S", 1, [&] { launch_S(P, C->b_lo, nb, s); });
    auto& st = C->kstat["setup_S"];
    double ent = (double)nb * k * k;
    st.flops += ent * 20;
    st.bytes += ent * 16;
}

// Householder QR (R only) of a complex M x N matrix, K = min(M, N): 4 x LAPACK's real count
// 2(2MNK - (M+N)K^2 + 2K^3/3), i.e. 8(MN^2 - N^3/3) for M >= N (a complex multiply-add = 8 flops)
inline double qr_flops(double M, double N) {
    double K = std::min(M, N);
    return 16.0 * (M * N * K - (M + N) * K * K / 2.0 + K * K * K / 3.0);
}

// Column factors aliased to the conjugate row factors (adjoint symmetry) or in their own storage
// (two passes requested on a symmetric structure; one shard).
void set_col_alias(Shard* C, bool alias) {
    PassH& X = C->col;
    PlanD& P = C->P;
    cudaStream_t s = C->stream;
    CK(cudaStreamSynchronize(s));
    if (alias) {
        X.C_off = X.C_off_alias;
        X.Q_off = X.Q_off_alias;
        X.sig_off = X.sig_off_alias;
        P.col.C = P.row.C;
        P.col.Q = P.row.Q;
        P.col.sigma = P.row.sigma;
    } else {
        if (C->world > 1) throw NotImpl("sharded recompression needs adjoint_symmetry = 1");
        X.C_off = X.C_off_own;
        X.Q_off = X.Q_off_own;
        X.sig_off = X.sig_off_own;
        if (!X.d_C.p && X.C_total) X.d_C.alloc(X.C_total);
        if (!X.d_Q.p && X.Q_total) X.d_Q.alloc(X.Q_total);
        if (!X.d_sigma.p && X.sig_total) {
            X.d_sigma.alloc(X.sig_total);
            CK(cudaMemsetAsync(X.d_sigma.p, 0, X.sig_total * sizeof(double), s));
        }
        P.col.C = X.d_C.p;
        P.col.Q = X.d_Q.p;
        P.col.sigma = X.d_sigma.p;
    }
    X.d_C_off.upload(X.C_off, s);
    X.d_Q_off.upload(X.Q_off, s);
    X.d_sig_off.upload(X.sig_off, s);
    P.col.C_off = X.d_C_off.p;
    P.col.Q_off = X.d_Q_off.p;
    P.col.sig_off = X.d_sig_off.p;
    P.col_conj = alias ? 1 : 0;
    X.alias = alias;
}

// Phase b: basis weights of this shard's basis pairs, bottom-up (Eq. 18).
void run_basis(Shard* C) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    const int L = T.depth, k = C->k, m = C->m;
    const bool sym = P.sym != 0;  // row basis pairs only (adjoint symmetry)
    for (int l = L; l >= 0; --l) {
        const auto& lst = sym ? C->basis_lists_sym[l] : C->basis_lists[l];
        int nb = (int)lst.size();
        if (!nb) continue;
        C->timed("basis@" + std::to_string(l), 1, [&] { launch_basis(P, sym ? C->d_basis_list_sym[l] : C->d_basis_list[l], nb, C->basis_maxrows[l], s); });
        double fl = 0;
        for (int id : lst) {
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
}

}  // namespace

namespace dh2 {
// Whether a leaf level folds its total weights into the truncation (dh2_set_option
// "fuse_leaf_weights"): 1 = wherever a fused kernel applies -- the split path's k_trunc_zqr
// (k <= 64, #t <= 32) or k_truncate_fused (#t <= 64, any k); 2 = only k_truncate_fused for k > 64
// (C4/C5 leaves).
bool fuse_leaf_level(const Shard* C, int leafrows, int maxz, int np) {
    if (!C->fuse_leaf || C->force_ws) return false;
    const PlanD& P = C->P;
    if (C->fuse_leaf == 1 && C->split_trunc && P.k <= 64 && leafrows <= 32) {
        const TruncLaunch TL = plan_truncate(P, np, leafrows, maxz, true, false);
        return !TL.use_ws;
    }
    return (C->fuse_leaf == 1 || P.k > 64) && leafrows <= 64 && trunc_fused_smem(P, leafrows) <= (size_t)P.smem_optin;
}

// Truncation of the pairs [p0, p0 + np) of level l (all leaves or all inner pairs): kernel choice
// (split warp-Jacobi path for leaves <= 32, shared-memory CTA per pair, or the global-workspace
// persistent grid), rank read-back (sizes the next level) and the executed-flop model.
void truncate_level(Shard* C, PassH& X, bool row, int l, int p0, int np, int maxrows, int maxz, bool all_leaf, bool fused,
                    double eps, int mode, const int* mirror) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    const int k = C->k, m = C->m;
    const std::string cls = std::string(row ? "truncate_row@" : "truncate_col@") + std::to_string(l);
    bool any_leaf = false, any_inner = false;
    for (int p = p0; p < p0 + np; ++p) (X.child0[p] < 0 ? any_leaf : any_inner) = true;
    if (any_leaf && any_inner) {
        // a level mixing leaf and inner clusters (sizes straddling the leaf size): one launch per
        // kind on pair lists, each sized by its own pairs
        std::vector<int> lists[2];
        int mr[2] = {0, 0}, mz[2] = {0, 0};
        for (int p = p0; p < p0 + np; ++p) {
            const int kind = X.child0[p] < 0 ? 0 : 1;
            lists[kind].push_back(p);
            mr[kind] = std::max(mr[kind], kind == 0 ? (int)T.size(C->bp_t[X.bp[p]]) : X.rank[X.child0[p]] + X.rank[X.child1[p]]);
            mz[kind] = std::max(mz[kind], X.Z_rows[p]);
        }
        std::vector<int> both(lists[0]);
        both.insert(both.end(), lists[1].begin(), lists[1].end());
        CK(cudaStreamSynchronize(s));
        C->d_plist.upload(both, s);
        for (int kind = 0; kind < 2; ++kind) {
            const int n = (int)lists[kind].size();
            const TruncLaunch TL = plan_truncate(P, n, mr[kind], mz[kind], kind == 0, C->force_ws != 0);
            if (TL.use_ws) {
                const size_t need = (size_t)TL.grid * TL.ws_stride;
                if (C->d_ws.n < need) {
                    CK(cudaStreamSynchronize(s));
                    C->d_ws.alloc(need);
                }
                ++C->ws_launches;
            }
            const int* pl = C->d_plist.p + (kind ? lists[0].size() : 0);
            C->timed(cls, 1, [&] { launch_truncate(P, row, 0, n, TL, kind == 0, eps, mode, C->d_ws.p, s, pl); });
        }
    } else {
    const TruncLaunch TL = plan_truncate(P, np, maxrows, maxz, all_leaf, C->force_ws != 0);
    const bool split = C->split_trunc && all_leaf && maxrows <= 32 && !TL.use_ws && (!fused || P.k <= 64);
    // leaves of 33..64 (C4/C5) and, with k > 64, inner levels of k1 + k2 <= 64 rows: QR kernel, then
    // Jacobi + epilogue at three pairs per SM
    const bool split64 = C->split_trunc64 && !TL.use_ws && !TL.append && !fused && maxrows <= 64 &&
                         ((all_leaf && maxrows > 32) || (!all_leaf && P.k > 64 && C->split_trunc64_inner));
    if (split64) {
        const size_t need = trunc_split64_scratch_bytes(np, all_leaf, P.k);
        if (C->d_tscr.n < need) {
            CK(cudaStreamSynchronize(s));
            C->d_tscr.alloc(need);
        }
        C->timed(cls, 2, [&] { launch_truncate_split64(P, row, p0, np, TL, all_leaf, eps, mode, C->d_tscr.p, s); });
    } else if (fused && !split) {  // leaf total weights folded into one CTA per pair (k_truncate_fused)
        C->timed(cls, 1, [&] { launch_truncate_fused(P, row, p0, np, maxrows, eps, mode, mirror, s); });
    } else if (split) {
        const size_t need = trunc_split_scratch_bytes(np);
        if (C->d_tscr.n < need) {
            CK(cudaStreamSynchronize(s));
            C->d_tscr.alloc(need);
        }
        C->timed(cls, 3, [&] { launch_truncate_split(P, row, p0, np, TL, eps, mode, C->d_tscr.p, fused, C->fuse_direct, mirror, s); });
    }
    if (TL.use_ws && !fused) {
        const size_t need = (size_t)TL.grid * TL.ws_stride;
        if (C->d_ws.n < need) {
            CK(cudaStreamSynchronize(s));
            C->d_ws.alloc(need);
        }
        ++C->ws_launches;
    }
    if (!split && !split64 && !fused) C->timed(cls, 1, [&] { launch_truncate(P, row, p0, np, TL, all_leaf, eps, mode, C->d_ws.p, s); });
    }
    CK(cudaMemcpyAsync(X.rank.data() + p0, X.d_rank.p + p0, np * sizeof(int), cudaMemcpyDeviceToHost, s));
    if ((int)C->sweeps_h.size() < np) C->sweeps_h.resize(np);
    CK(cudaMemcpyAsync(C->sweeps_h.data(), X.d_sweeps.p + p0, np * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int p = p0; p < p0 + np; ++p)
        if (X.rank[p] < 0)
            throw NumericError("non-finite singular values in the truncation of level " + std::to_string(l) + " (pair " +
                               std::to_string(p) + "): non-finite input from an earlier phase");
    for (int i = 0; i < np; ++i)  // every Jacobi loop stops after 60 sweeps; reaching it means no convergence
        if (C->sweeps_h[i] >= 60)
            throw NumericError("one-sided Jacobi SVD did not converge in 60 sweeps (truncation of level " + std::to_string(l) +
                               ", pair " + std::to_string(p0 + i) + ")");
    double fl = 0;
    for (int p = p0; p < p0 + np; ++p) {
        double rows = X.child0[p] < 0 ? (double)T.size(C->bp_t[X.bp[p]]) : X.rank[X.child0[p]] + X.rank[X.child1[p]];
        double zr = X.Z_rows[p];
        if (X.child0[p] >= 0) fl += 8.0 * 3 * rows * k * m;
        if (fused) {  // stack rows (as total weights), stack V^*, structured QR appends
            const double tot = X.total_rows[p];
            for (int ib = X.blk_ptr[p]; ib < X.blk_ptr[p + 1]; ++ib) {
                int b = X.blk[ib];
                fl += 8.0 * C->bp_R_rows[row ? C->blk_bpcol[b] : C->blk_bprow[b]] * (double)k * k;
            }
            for (int ip = X.par_ptr[p]; ip < X.par_ptr[p + 1]; ++ip) fl += 8.0 * 3 * X.Z_rows[X.par[ip]] * (double)k * m;
            fl += 8.0 * tot * rows * k + 8.0 * tot * rows * rows;
            zr = std::min(tot, rows);
        } else {
            fl += 8.0 * rows * zr * k;  // M
        }
        double n = std::min(rows, zr);
        if (rows < zr) fl += qr_flops(zr, rows);
        fl += 8.0 * 10.0 * rows * n * n;  // SVD, C_svd = 10 model (DESIGN §flop model)
        fl += 8.0 * X.rank[p] * rows * k;  // C
    }
    C->kstat[cls].flops += fl;
}
}  // namespace dh2

namespace {

// Phases c-e: block weights, total weights (top-down) and truncation (bottom-up) of the row
// pass over this shard's pairs; the column pass by adjoint symmetry (or a second pass, 1 shard).
void run_weights_truncate(Shard* C, double eps, int mode) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const ClusterTree& T = C->st.ct;
    const int L = T.depth, k = C->k, m = C->m;
    C->timed("block_weights", 1, [&] { launch_block_weights(P, C->b_lo, C->b_hi - C->b_lo, mode, C->d_blk_mirror.p, s); });
    {
        double fl = 0;
        for (int b = C->b_lo; b < C->b_hi; ++b) {
            double rt = C->bp_R_rows[C->blk_bprow[b]], rs = C->bp_R_rows[C->blk_bpcol[b]];
            fl += 8.0 * (rt * k * k + rt * rs * k);
        }
        C->kstat["block_weights"].flops += fl;
    }
    const bool sym = C->sym_ok && C->sym_opt;
    if (!sym && C->world > 1) throw NotImpl("sharded recompression needs adjoint_symmetry = 1");
    if (!sym && !C->col.d_Z.p && C->col.Z_total) {  // two passes requested on a symmetric structure
        C->col.d_Z.alloc(C->col.Z_total);
        C->P.col.Z = C->col.d_Z.p;
    }
    if (C->sym_ok && C->col.alias != sym) set_col_alias(C, sym);
    C->sym_used = sym;
    C->fused_levels[0].clear();
    C->fused_levels[1].clear();
    C->fused_append = 0;
    for (int side = 0; side < 2; ++side) {
        PassH& X = side == 0 ? C->row : C->col;
        const bool row = side == 0;
        if (!row && sym) {
            // column pass = conjugate of the row pass at -c (check_symmetry)
            X.rank.assign(X.bp.size(), 0);
            double by = 0;
            for (int l = 0; l <= L; ++l) {
                const int p0 = X.own_lo[l], np = X.own_hi[l] - p0;
                if (!np) continue;
                C->timed("mirror_col", 1, [&] { launch_mirror_pass(P, C->d_col2row.p, p0, np, s); });
                for (int p = p0; p < p0 + np; ++p) {
                    const int kk = X.rank[p] = C->row.rank[C->col2row[p]];
                    by += 2.0 * 16.0 * ((double)kk * k + (double)X.rowsb[p] * kk);
                }
            }
            C->kstat["mirror_col"].bytes += by;
            C->fused_levels[1] = C->fused_levels[0];  // column Zhat mirrors the row Zhat
            continue;
        }
        // leaf levels truncated by the split path with k <= 64 fold their total weights into the
        // split QR (k_trunc_zqr): Zhat of such a level is never formed
        auto level_kind = [&](int l, bool& all_leaf, bool& any_leaf) {
            all_leaf = true;
            any_leaf = false;
            for (int p = X.own_lo[l]; p < X.own_hi[l]; ++p) {
                all_leaf = all_leaf && X.child0[p] < 0;
                any_leaf = any_leaf || X.child0[p] < 0;
            }
        };
        std::vector<char> fused(L + 1, 0);
        for (int l = 0; l <= L; ++l) {
            const int np = X.own_hi[l] - X.own_lo[l];
            bool all_leaf, any_leaf;
            level_kind(l, all_leaf, any_leaf);
            if (!np || !all_leaf || !fuse_leaf_level(C, X.lev_max_leafrows[l], X.lev_max_zrows[l], np)) continue;
            fused[l] = 1;
            C->fused_levels[side].push_back(l);
            for (int p = X.own_lo[l]; p < X.own_hi[l]; ++p) C->fused_append += X.total_rows[p] > C->fuse_direct;
        }
        // total weights, top-down
        for (int l = 0; l <= L; ++l) {
            int p0 = X.own_lo[l], np = X.own_hi[l] - p0;
            if (!np || fused[l]) continue;
            bool all_leaf, any_leaf;
            level_kind(l, all_leaf, any_leaf);
            C->timed(std::string(row ? "total_weights_row@" : "total_weights_col@") + std::to_string(l), 1,
                     [&] { launch_total_weights(P, row, p0, np, C->d_blk_mirror.p, s, all_leaf); });
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
            int p0 = X.own_lo[l], np = X.own_hi[l] - p0;
            if (!np) continue;
            int maxrows = X.lev_max_leafrows[l];
            for (int p = p0; p < p0 + np; ++p)
                if (X.child0[p] >= 0) maxrows = std::max(maxrows, X.rank[X.child0[p]] + X.rank[X.child1[p]]);
            bool all_leaf, any_leaf;
            level_kind(l, all_leaf, any_leaf);  // (mixed levels: one launch per kind, truncate_level)
            truncate_level(C, X, row, l, p0, np, maxrows, X.lev_max_zrows[l], all_leaf, fused[l] != 0, eps, mode,
                           C->d_blk_mirror.p);
        }
    }
}

// Phase f: projection of this shard's blocks, S~_b = C_tc S_b C'^*_sc.
void run_project(Shard* C) {
    const PlanD& P = C->P;
    const int k = C->k;
    int maxkrow = 0;
    for (int l = 0; l < (int)C->row.own_lo.size(); ++l)
        for (int p = C->row.own_lo[l]; p < C->row.own_hi[l]; ++p) maxkrow = std::max(maxkrow, C->row.rank[p]);
    C->timed("project", 1, [&] { launch_project(P, C->b_lo, C->b_hi - C->b_lo, maxkrow, C->d_blk_mirror.p, C->stream); });
    double fl = 0;
    for (int b = C->b_lo; b < C->b_hi; ++b) {
        double kt = C->row.rank[C->blk_prow[b]], ks = C->col.rank[C->blk_pcol[b]];
        fl += 8.0 * (kt * k * k + kt * ks * k);
    }
    C->kstat["project"].flops += fl;
}

// certified sums of this shard: discarded squares of its own row/column pairs, ||G_b||^2 of its blocks
void local_sums(Shard* C, double out[3]) {
    out[0] = out[1] = out[2] = 0.0;
    for (int side = 0; side < 2; ++side) {
        PassH& X = side == 0 ? C->row : C->col;
        X.disc.assign(X.bp.size(), 0.0);
        for (int l = 0; l < (int)X.own_lo.size(); ++l) {
            const int p0 = X.own_lo[l], np = X.own_hi[l] - p0;
            if (np) CK(cudaMemcpy(X.disc.data() + p0, X.d_disc.p + p0, np * sizeof(double), cudaMemcpyDeviceToHost));
        }
        for (double d : X.disc) out[side] += d;
    }
    std::vector<double> g2(C->b_hi - C->b_lo);
    if (!g2.empty())
        CK(cudaMemcpy(g2.data(), C->d_normG2.p + C->b_lo, g2.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (double d : g2) out[2] += d;
}

// Matvec, part 1: x (original order) -> cluster order, forward transformation of this shard's
// column pairs (xh'_sc = B_sc^* x|_s, nested through the transfers), bottom-up.
void run_mv_forward(Shard* C, bool recomp, const double2* x) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const int L = C->st.ct.depth, n = C->n;
    C->timed("matvec", 1, [&] { launch_permute(P.perm, x, C->d_xp.p, n, true, s); });
    for (int l = L; l >= 0; --l) {
        int p0 = C->col.own_lo[l], np = C->col.own_hi[l] - p0;
        if (np) C->timed("matvec", 1, [&] { launch_mv_forward(P, recomp, p0, np, C->d_xp.p, C->d_xh.p, s); });
    }
}

// Matvec, part 2 (after the xh' exchange): couplings, backward transformation and leaf output
// of this shard's row pairs into the cluster-ordered yp (own position range).
void run_mv_rest(Shard* C, bool recomp) {
    const PlanD& P = C->P;
    cudaStream_t s = C->stream;
    const int L = C->st.ct.depth, n = C->n;
    for (int l = 0; l <= L; ++l) {
        int p0 = C->row.own_lo[l], np = C->row.own_hi[l] - p0;
        if (np) C->timed("matvec", 1, [&] { launch_mv_couple(P, recomp, p0, np, C->d_xh.p, C->d_yh.p, s); });
    }
    for (int l = 0; l <= L; ++l) {
        int p0 = C->row.own_lo[l], np = C->row.own_hi[l] - p0;
        if (np) C->timed("matvec", 1, [&] { launch_mv_backward(P, recomp, p0, np, C->d_yh.p, s); });
    }
    CK(cudaMemsetAsync(C->d_yp.p, 0, sizeof(double2) * n, s));
    C->timed("matvec", 1, [&] {
        launch_mv_leaf_out(P, recomp, C->row.d_lc.p, C->row.d_lc_ptr.p, C->row.lc_lo, C->row.lc_hi - C->row.lc_lo, C->d_yh.p,
                           C->d_yp.p, s);
    });
}

// Matvec, part 3 (after the yp gather): cluster order -> original order.
void run_mv_out(Shard* C, double2* y) {
    C->timed("matvec", 1, [&] { launch_permute(C->P.perm, C->d_yp.p, y, C->n, false, C->stream); });
}

void require_device(const Shard* C) {
    if (C->device == DH2_DEVICE_NONE) throw StateError("structure-only context (device = DH2_DEVICE_NONE) has no device data");
}

// Storage of this shard's part (DESIGN R21): own pairs, own blocks, nearfield
// blocks whose row cluster it owns.  v = {row basis, col basis, couplings, nearfield, sum of
// ranks, number of ranks, max rank} (bytes; 16 B per complex entry).
void storage_partial(const Shard* C, int which, double v[7]) {
    const Structure& S = C->st;
    const ClusterTree& T = S.ct;
    const int k = C->k, me = C->rank;
    const bool rc = which == DH2_RECOMP;
    for (int i = 0; i < 7; ++i) v[i] = 0.0;
    for (auto& pr : S.near) {
        const int o = C->owner[pr.first];
        if (o == me || (o < 0 && me == 0)) v[3] += (double)T.size(pr.first) * T.size(pr.second) * 16.0;
    }
    for (int side = 0; side < 2; ++side) {
        const PassH& X = side == 0 ? C->row : C->col;
        double tot = 0;
        for (int l = 0; l < (int)X.own_lo.size(); ++l)
            for (int p = X.own_lo[l]; p < X.own_hi[l]; ++p) {
                int t = C->bp_t[X.bp[p]];
                if (X.child0[p] < 0)
                    tot += (double)T.size(t) * (rc ? X.rank[p] : k);
                else if (rc)
                    tot += (double)(X.rank[X.child0[p]] + X.rank[X.child1[p]]) * X.rank[p];
                else
                    tot += 2.0 * k * k;
                if (rc) {
                    v[4] += X.rank[p];
                    v[5] += 1;
                    v[6] = std::max(v[6], (double)X.rank[p]);
                }
            }
        v[side] = tot * 16.0;
    }
    for (int b = C->b_lo; b < C->b_hi; ++b)
        v[2] += rc ? (double)C->row.rank[C->blk_prow[b]] * C->col.rank[C->blk_pcol[b]] * 16.0 : (double)k * k * 16.0;
    if (!rc) {
        v[4] = k;
        v[5] = 1;
        v[6] = k;
    }
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

// Internal export of one shard's host/device arrays (names: DESIGN.md §12).
void export_shard(const Shard* C, const char* name, void* buf, int64_t* nbytes) {
        static thread_local std::vector<int64_t> tmp64;
        static thread_local std::vector<int> tmp32;
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
        bool conj_out = false;
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
            else if (C->lean.on && X == &C->row && (base == "kb" || base == "rowsb" || base == "C_off" || base == "Q_off")) {
                // lean plan: the current layout (compact after the truncation)
                const LeanState& Ln = C->lean;
                it = base == "kb" ? hv(Ln.kb_cur) : base == "rowsb" ? hv(Ln.rowsb_cur) : base == "C_off" ? hv(Ln.C_off_cur) : hv(Ln.Q_off_cur);
            } else if (base == "kb") it = hv(X->kb);
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
            else if (C->lean.on && (base == "C" || base == "Q")) {
                // lean plan: compact Q/F and the persistent C (direct pairs) at the start of the pools
                const LeanState& Ln = C->lean;
                const bool q = base == "Q";
                it = {q ? Ln.Qpool.ptr() : Ln.Cpool.ptr(), (size_t)(q ? Ln.Q_used : Ln.C_used) * sizeof(double2), true,
                      sizeof(double2)};
                conj_out = X == &C->col;
            } else if (X == &C->col && X->alias && (base == "C" || base == "Q" || base == "sigma")) {
                // aliased column factors: conjugates of the row storage at (s,-c) (offsets C_off_col, ...)
                if (base == "sigma") {
                    it = dv(C->row.d_sigma);
                } else {
                    it = dv(base == "C" ? C->row.d_C : C->row.d_Q);
                    conj_out = true;
                }
            } else if (base == "C") it = dv(X->d_C);
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
        } else if (nm == "near_values") {  // this shard's assembled nearfield blocks (dh2_nearfield_assemble)
            if (!C->near.on) throw StateError("near_values before dh2_nearfield_assemble");
            it = {C->near.d_val.p, (size_t)C->near.values * sizeof(double2), true, sizeof(double2)};
        } else if (nm == "near_off") {
            if (!C->near.on) throw StateError("near_off before dh2_nearfield_assemble");
            it = hv(C->near.off);
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
        else if (nm == "bp_neg") it = hv(C->bp_neg);
        else if (nm == "lean_p_lo") it = hv(C->lean.p_lo);
        else if (nm == "lean_p_hi") it = hv(C->lean.p_hi);
        else if (nm == "lean_blk_ptr") it = hv(C->lean.blk_ptr);
        else if (nm == "lean_blk") it = hv(C->lean.blk);
        else if (nm == "lean_qr_ptr") it = hv(C->lean.qr_ptr);
        else if (nm == "lean_qr") it = hv(C->lean.qr);
        else if (nm == "lean_lvd") it = hv(C->lean.lvd);
        else if (nm == "lean_lvb") it = hv(C->lean.lvb);
        else if (nm == "lean_keep") it = hv(C->lean.keep);
        else if (nm == "lean_keepC") it = hv(C->lean.keepC);
        else if (nm == "lean_slot") it = hv(C->lean_slot);
        else if (nm == "lean_mirror") it = hv(C->lean_mirror);
        else if (nm == "blk_bpcs") it = hv(C->blk_bpcs);
        else if (nm == "owner") {
            tmp32.assign(C->owner.begin(), C->owner.end());
            it = hv(tmp32);
        } else if (nm == "own_range") {
            tmp32 = {C->b_lo, C->b_hi, (int)C->pos_lo, (int)C->pos_hi};
            it = hv(tmp32);
        } else if (nm == "xR_send" || nm == "xR_recv" || nm == "xC_send" || nm == "xC_recv") {
            const auto& L = nm == "xR_send" ? C->R_send : nm == "xR_recv" ? C->R_recv : nm == "xC_send" ? C->C_send : C->C_recv;
            tmp32.clear();
            for (const auto& v : L) {
                tmp32.push_back((int)v.size());
                tmp32.insert(tmp32.end(), v.begin(), v.end());
            }
            it = hv(tmp32);
        } else if (nm == "VR") it = dv(C->d_VR);
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
        if (conj_out) {
            double2* z = static_cast<double2*>(buf);
            for (size_t i = 0; i < it.bytes / sizeof(double2); ++i) z[i].y = -z[i].y;
        }
        *nbytes = (int64_t)it.bytes;
        (void)tmpd;
}

}  // namespace

// ============================================================== context (one or more shards)
// A context holds the shards this process runs: 1 (single GPU, or one rank of an NCCL job) or,
// in the virtual mode (world > 1 without an NCCL id), all `world` shards of the partition on one
// device, run phase by phase with device-to-device exchanges.  Both modes execute the same
// shard code and exchange the same items; only the transport differs.
struct dh2_ctx {
    std::vector<std::unique_ptr<Shard>> sh;
    std::string err;
    int world = 1, rank = 0;
    bool virt = false;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool recompressed = false;
    double E_row = 0, E_col = 0, far2 = 0;
    double exch_bytes = 0;  // bytes moved by the last recompress + matvec exchanges (this process)
    // NCCL transport
    void* comm = nullptr;
    DevBuf<double2> sendbuf, recvbuf;
    DevBuf<int> isend, irecv;
    DevBuf<double> red;
    // cached segment lists: key = (kind, a, b)
    struct Seg {
        DevBuf<int64_t> soff, doff, len;
        int n = 0;
        std::vector<int64_t> peer_cnt;  // NCCL: elements per peer (pack order = peer order)
        int64_t total = 0;
    };
    std::map<std::tuple<int, int, int>, std::unique_ptr<Seg>> segs;
    ~dh2_ctx();
};

namespace {

// ---------------------------------------------------------------- NCCL, loaded at run time
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = std::string("dlopen libnccl.so.2: ") + dlerror();
        return api;
    }
    auto sym = [&](const char* nm) { return dlsym(h, nm); };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv && api.AllReduce &&
             api.GroupStart && api.GroupEnd && api.GetErrorString;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    return api;
}

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#define NK(x)                                                                                           \
    do {                                                                                                \
        ncclResult_t r_ = (x);                                                                          \
        if (r_ != ncclSuccess) throw NcclError(std::string(#x) + ": " + nccl().GetErrorString(r_));     \
    } while (0)

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
    } catch (const NcclError& e) {
        return fail(C, DH2_ENCCL, e.what());
    } catch (const StateError& e) {
        return fail(C, DH2_ESTATE, e.what());
    } catch (const NotImpl& e) {
        return fail(C, DH2_ENOTIMPL, e.what());
    } catch (const NoMem& e) {
        return fail(C, DH2_ENOMEM, e.what());
    } catch (const NumericError& e) {
        return fail(C, DH2_ENUMERIC, e.what());
    } catch (const MismatchError& e) {
        return fail(C, DH2_EMISMATCH, e.what());
    } catch (const std::bad_alloc& e) {
        return fail(C, DH2_ENOMEM, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(C, DH2_ECUDA, std::string("internal error: ") + e.what());
    }
}

// ---------------------------------------------------------------- exchanges
enum XKind { X_R = 0, X_C = 1, X_RANK = 2, X_XH = 3 };

// items exchanged from shard `from` to shard `to`, as seen by shard S (S is one of them)
const std::vector<int>& items(const Shard* S, XKind kind, int peer, bool send) {
    if (kind == X_R) return send ? S->R_send[peer] : S->R_recv[peer];
    return send ? S->C_send[peer] : S->C_recv[peer];
}

// (offset, length) of one item in the shard's pool of that kind
std::pair<int64_t, int64_t> item_seg(const Shard* S, XKind kind, int id) {
    const int k = S->k;
    switch (kind) {
        case X_R: return {S->bp_R_off[id], (int64_t)S->bp_R_rows[id] * k};
        case X_C: return {S->col.C_off[id], (int64_t)S->col.kb[id] * k};
        case X_RANK: return {id, 1};
        default: return {(int64_t)id * k, k};
    }
}

void upload_seg(dh2_ctx::Seg& g, const std::vector<int64_t>& so, const std::vector<int64_t>& d, const std::vector<int64_t>& ln,
                cudaStream_t s) {
    g.soff.upload(so, s);
    g.doff.upload(d, s);
    g.len.upload(ln, s);
    g.n = (int)so.size();
}

double2* pool2(Shard* S, XKind kind) { return kind == X_R ? S->d_VR.p : kind == X_C ? S->P.col.C : S->d_xh.p; }

// one exchange of `kind` among all shards (virtual) or with all peers (NCCL)
void exchange(dh2_ctx* X, XKind kind) {
    cudaStream_t s = X->stream;
    const int W = X->world;
    if (W == 1) return;
    if (X->virt) {
        for (int a = 0; a < W; ++a)
            for (int b = 0; b < W; ++b) {
                if (a == b) continue;
                Shard *A = X->sh[a].get(), *B = X->sh[b].get();
                const auto& ia = items(A, kind, b, true);
                if (ia.empty()) continue;
                auto& slot = X->segs[{(int)kind, a, b}];
                if (!slot) {
                    const auto& ib = items(B, kind, a, false);
                    if (ia != ib) throw std::logic_error("exchange lists of two shards disagree");
                    slot.reset(new dh2_ctx::Seg());
                    std::vector<int64_t> so, d, ln;
                    for (int id : ia) {
                        auto sa = item_seg(A, kind, id), sb = item_seg(B, kind, id);
                        so.push_back(sa.first);
                        d.push_back(sb.first);
                        ln.push_back(sa.second);
                        slot->total += sa.second;
                    }
                    upload_seg(*slot, so, d, ln, s);
                }
                if (kind == X_RANK)
                    launch_copy_segments_i(A->col.d_rank.p, B->col.d_rank.p, slot->soff.p, slot->doff.p, slot->len.p, slot->n, s);
                else
                    launch_copy_segments(pool2(A, kind), pool2(B, kind), slot->soff.p, slot->doff.p, slot->len.p, slot->n, s);
                X->exch_bytes += (double)slot->total * (kind == X_RANK ? 4 : 16);
                CK(cudaGetLastError());
            }
        return;
    }
    // NCCL: pack -> grouped send/recv with every peer -> unpack
    Shard* S = X->sh[0].get();
    const int me = X->rank;
    auto build = [&](bool send) {
        auto& slot = X->segs[{(int)kind, send ? 0 : 1, -1}];
        if (slot) return slot.get();
        slot.reset(new dh2_ctx::Seg());
        std::vector<int64_t> so, d, ln;
        slot->peer_cnt.assign(W, 0);
        int64_t pos = 0;
        for (int peer = 0; peer < W; ++peer) {
            if (peer == me) continue;
            for (int id : items(S, kind, peer, send)) {
                auto sg = item_seg(S, kind, id);
                so.push_back(send ? sg.first : pos);
                d.push_back(send ? pos : sg.first);
                ln.push_back(sg.second);
                pos += sg.second;
                slot->peer_cnt[peer] += sg.second;
            }
        }
        slot->total = pos;
        upload_seg(*slot, so, d, ln, s);
        return slot.get();
    };
    dh2_ctx::Seg* out = build(true);
    dh2_ctx::Seg* in = build(false);
    const bool ints = kind == X_RANK;
    const size_t esz = ints ? sizeof(int) : sizeof(double2);
    const bool grow = ints ? (X->isend.n < (size_t)out->total || X->irecv.n < (size_t)in->total)
                           : (X->sendbuf.n < (size_t)out->total || X->recvbuf.n < (size_t)in->total);
    if (grow) CK(cudaStreamSynchronize(s));  // earlier sends/receives may still use the old buffers
    if (ints) {
        if (X->isend.n < (size_t)out->total) X->isend.alloc(out->total);
        if (X->irecv.n < (size_t)in->total) X->irecv.alloc(in->total);
        launch_copy_segments_i(S->col.d_rank.p, X->isend.p, out->soff.p, out->doff.p, out->len.p, out->n, s);
    } else {
        if (X->sendbuf.n < (size_t)out->total) X->sendbuf.alloc(out->total);
        if (X->recvbuf.n < (size_t)in->total) X->recvbuf.alloc(in->total);
        launch_copy_segments(pool2(S, kind), X->sendbuf.p, out->soff.p, out->doff.p, out->len.p, out->n, s);
    }
    CK(cudaGetLastError());
    char* sb = ints ? (char*)X->isend.p : (char*)X->sendbuf.p;
    char* rb = ints ? (char*)X->irecv.p : (char*)X->recvbuf.p;
    ncclComm_t comm = (ncclComm_t)X->comm;
    NK(nccl().GroupStart());
    int64_t so = 0, ro = 0;
    for (int peer = 0; peer < W; ++peer) {
        if (peer == me) continue;
        if (out->peer_cnt[peer]) NK(nccl().Send(sb + so * esz, out->peer_cnt[peer] * esz, ncclUint8, peer, comm, s));
        if (in->peer_cnt[peer]) NK(nccl().Recv(rb + ro * esz, in->peer_cnt[peer] * esz, ncclUint8, peer, comm, s));
        so += out->peer_cnt[peer];
        ro += in->peer_cnt[peer];
    }
    NK(nccl().GroupEnd());
    if (ints)
        launch_copy_segments_i(X->irecv.p, S->col.d_rank.p, in->soff.p, in->doff.p, in->len.p, in->n, s);
    else
        launch_copy_segments(X->recvbuf.p, pool2(S, kind), in->soff.p, in->doff.p, in->len.p, in->n, s);
    CK(cudaGetLastError());
    X->exch_bytes += (double)(out->total + in->total) * esz;
}

// gather the cluster-ordered output slices of all shards (every rank / shard 0 gets all of yp)
void gather_y(dh2_ctx* X) {
    const int W = X->world;
    if (W == 1) return;
    cudaStream_t s = X->stream;
    Shard* S0 = X->sh[0].get();
    const ClusterTree& T = S0->st.ct;
    auto range = [&](int r) {
        const int64_t t = T.levels[S0->cut][r];
        return std::make_pair(T.begin[t], T.end[t]);
    };
    if (X->virt) {
        for (int r = 1; r < W; ++r) {
            auto g = range(r);
            CK(cudaMemcpyAsync(S0->d_yp.p + g.first, X->sh[r]->d_yp.p + g.first, (g.second - g.first) * sizeof(double2),
                               cudaMemcpyDeviceToDevice, s));
        }
        return;
    }
    ncclComm_t comm = (ncclComm_t)X->comm;
    auto mine = range(X->rank);
    NK(nccl().GroupStart());
    for (int peer = 0; peer < W; ++peer) {
        if (peer == X->rank) continue;
        auto g = range(peer);
        NK(nccl().Send(S0->d_yp.p + mine.first, (mine.second - mine.first) * sizeof(double2), ncclUint8, peer, comm, s));
        NK(nccl().Recv(S0->d_yp.p + g.first, (g.second - g.first) * sizeof(double2), ncclUint8, peer, comm, s));
    }
    NK(nccl().GroupEnd());
}

// sum (or max) of a few doubles over all shards / ranks
void reduce_doubles(dh2_ctx* X, std::vector<double>& v, bool max_op) {
    if (X->world == 1 || X->virt) return;  // virtual: the caller already combined the shards
    if (X->red.n < v.size()) X->red.alloc(v.size());
    CK(cudaMemcpyAsync(X->red.p, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, X->stream));
    NK(nccl().AllReduce(X->red.p, X->red.p, v.size(), ncclFloat64, max_op ? ncclMax : ncclSum, (ncclComm_t)X->comm, X->stream));
    CK(cudaMemcpyAsync(v.data(), X->red.p, v.size() * sizeof(double), cudaMemcpyDeviceToHost, X->stream));
    CK(cudaStreamSynchronize(X->stream));
}

void finish_all(dh2_ctx* X) {
    for (auto& S : X->sh) S->finish();
}

void require_device(const dh2_ctx* X) { require_device(X->sh[0].get()); }

uint64_t fnv1a(const void* data, size_t n, uint64_t h) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 1099511628211ull;
    }
    return h;
}

// DH2_EMISMATCH: the arguments' hash, min- and max-reduced over the ranks, must agree (NCCL mode;
// the virtual mode runs every shard from the same call)
void check_same_args(dh2_ctx* X, uint64_t h, const char* what) {
    if (X->world == 1 || X->virt || !X->comm) return;
    DevBuf<uint64_t> d;
    d.alloc(2);
    const uint64_t v[2] = {h, ~h};  // max of ~h = ~(min of h)
    CK(cudaMemcpyAsync(d.p, v, sizeof(v), cudaMemcpyHostToDevice, X->stream));
    NK(nccl().AllReduce(d.p, d.p, 2, ncclUint64, ncclMax, (ncclComm_t)X->comm, X->stream));
    uint64_t r[2];
    CK(cudaMemcpyAsync(r, d.p, sizeof(r), cudaMemcpyDeviceToHost, X->stream));
    CK(cudaStreamSynchronize(X->stream));
    if (r[0] != h || ~r[1] != h) throw MismatchError(std::string(what) + " differ between ranks");
}

void do_recompress(dh2_ctx* X, double eps, int mode) {
    if (X->sh[0]->lean.on) {  // memory-lean chunked plan (every shard of a context chooses alike)
        // host wall clock per phase (issue + the phase's own synchronisations; stats "lean_wall_ms")
        auto& W = X->sh[0]->lean_wall_ms;
        W.assign(6, 0.0);
        auto tw = std::chrono::steady_clock::now();
        auto mark = [&](int i) {
            auto now = std::chrono::steady_clock::now();
            W[i] += std::chrono::duration<double, std::milli>(now - tw).count();
            tw = now;
        };
        for (auto& S : X->sh) lean_begin(S.get());
        mark(0);
        for (auto& S : X->sh) lean_basis(S.get());
        exchange(X, X_R);  // R of the (s,-c) that other shards' blocks reference
        mark(1);
        for (auto& S : X->sh) lean_weights_truncate(S.get(), eps, mode);
        exchange(X, X_RANK);
        mark(2);
        for (auto& S : X->sh) lean_columns(S.get());
        // the compact C layout depends on the ranks: segment lists of X_C are rebuilt every time
        for (auto it = X->segs.begin(); it != X->segs.end();)
            it = std::get<0>(it->first) == (int)X_C ? X->segs.erase(it) : std::next(it);
        exchange(X, X_C);
        mark(3);
        for (auto& S : X->sh) lean_project(S.get());
        mark(4);
        finish_all(X);
        mark(5);
        std::vector<double> sums(3, 0.0);
        for (auto& S : X->sh) {
            double v[3];
            local_sums(S.get(), v);
            for (int i = 0; i < 3; ++i) sums[i] += v[i];
            lean_finish(S.get());
        }
        reduce_doubles(X, sums, false);
        X->E_row = sums[0];
        X->E_col = sums[1];
        X->far2 = sums[2];
        return;
    }
    for (auto& S : X->sh) {
        // adjoint symmetry: row basis pairs only; the two-pass mode needs the column-only V/E too
        const bool sym = S->sym_ok && S->sym_opt;
        if (!sym && !S->col_data) {
            S->P.sym = 0;
            run_setup(S.get());
        }
        S->P.sym = sym ? 1 : 0;
    }
    for (auto& S : X->sh) run_basis(S.get());
    exchange(X, X_R);  // R_sc of column pairs referenced across shards (after phase b)
    for (auto& S : X->sh) run_weights_truncate(S.get(), eps, mode);
    exchange(X, X_C);  // C'_sc and k'_sc (after the column truncation)
    exchange(X, X_RANK);
    if (X->world > 1) {
        CK(cudaStreamSynchronize(X->stream));
        for (auto& S : X->sh) {  // host copies of the imported column ranks (projection flops, storage)
            std::vector<int> all(S->col.bp.size());
            CK(cudaMemcpy(all.data(), S->col.d_rank.p, all.size() * sizeof(int), cudaMemcpyDeviceToHost));
            for (int peer = 0; peer < X->world; ++peer)
                for (int p : S->C_recv[peer]) S->col.rank[p] = all[p];
        }
    }
    for (auto& S : X->sh) run_project(S.get());
    finish_all(X);
    std::vector<double> sums(3, 0.0);
    for (auto& S : X->sh) {
        double v[3];
        local_sums(S.get(), v);
        for (int i = 0; i < 3; ++i) sums[i] += v[i];
    }
    reduce_doubles(X, sums, false);
    X->E_row = sums[0];
    X->E_col = sums[1];
    X->far2 = sums[2];
}

void do_matvec(dh2_ctx* X, bool recomp, const double2* x, double2* y, bool add_near) {
    if (!recomp && X->sh[0]->lean.on)
        throw NotImpl("ORIG matvec on the memory-lean plan (V and S are not resident)");
    if (add_near)
        for (auto& S : X->sh)
            if (!S->near.on) throw StateError("DH2_ADD_NEAR before dh2_nearfield_assemble");
    for (auto& S : X->sh) run_mv_forward(S.get(), recomp, x);
    exchange(X, X_XH);  // xh'_sc of column pairs referenced across shards
    for (auto& S : X->sh) {
        run_mv_rest(S.get(), recomp);
        if (add_near) near_matvec(S.get());  // own rows, x_p holds all of x on every shard
    }
    gather_y(X);
    run_mv_out(X->sh[0].get(), y);
    if (!X->virt)
        for (size_t i = 1; i < X->sh.size(); ++i) run_mv_out(X->sh[i].get(), y);
}

}  // namespace

dh2_ctx::~dh2_ctx() {
    for (auto& S : sh)
        if (S->device != DH2_DEVICE_NONE && S->stream) {
            cudaSetDevice(S->device);
            cudaStreamSynchronize(S->stream);
        }
    segs.clear();
    sh.clear();
    if (comm && nccl().ok) nccl().CommDestroy((ncclComm_t)comm);
}

// ============================================================== C ABI
extern "C" {

int dh2_nccl_unique_id(void* uid) {
    if (!uid) return fail(nullptr, DH2_EINVAL, "null argument");
    NcclApi& api = nccl();
    if (!api.ok) return fail(nullptr, DH2_ENCCL, api.why);
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, DH2_ENCCL, api.GetErrorString(r));
    std::memcpy(uid, &id, sizeof(id));
    return DH2_OK;
}

int dh2_build_interp(const dh2_mesh* mesh, const dh2_params* params, const dh2_dist* dist, dh2_ctx** out) {
    if (out) *out = nullptr;
    if (!mesh || !params || !out) return fail(nullptr, DH2_EINVAL, "null argument");
    std::unique_ptr<dh2_ctx> X(new dh2_ctx());
    int rc = guarded(X.get(), [&] {
        const dh2_params& p = *params;
        if (!(p.kappa >= 0.0) || p.m < 1 || p.leaf_size < 1 || !(p.eta1 > 0.0) || !(p.eta2 > 0.0))
            throw std::invalid_argument("invalid parameters");
        if (p.quad != 7) throw std::invalid_argument("quad must be 7 (Radon's degree-5 rule)");
        if (p.m > MMAX) throw NotImpl("m > " + std::to_string(MMAX) + " (grid tables are sized for m <= MMAX)");
        if (mesh->nt > (int64_t)1 << 30) throw std::invalid_argument("mesh too large");
        validate_mesh(mesh->xyz, mesh->nv, mesh->tri, mesh->nt);
        X->world = dist ? std::max(1, (int)dist->world) : 1;
        X->rank = dist ? (int)dist->rank : 0;
        X->device = dist ? dist->device : 0;
        X->virt = X->world > 1 && (!dist || !dist->nccl_uid);
        if (X->rank < 0 || X->rank >= X->world) throw std::invalid_argument("rank out of range");
        const bool structure_only = X->device == DH2_DEVICE_NONE;
        if (!structure_only) {
            int ndev = 0;
            if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) throw CudaError("no CUDA device");
            CK(cudaSetDevice(X->device));
        }
        auto t0 = std::chrono::steady_clock::now();
        Params prm;
        prm.kappa = p.kappa;
        prm.m = p.m;
        prm.leaf = p.leaf_size;
        prm.eta1 = p.eta1;
        prm.eta2 = p.eta2;
        const int nsh = X->virt ? X->world : 1;
        for (int i = 0; i < nsh; ++i) {
            X->sh.emplace_back(new Shard());
            Shard* S = X->sh.back().get();
            S->device = X->device;
            S->world = X->world;
            S->rank = X->virt ? i : X->rank;
            if (i == 0)
                S->st.build(mesh->xyz, mesh->nv, mesh->tri, mesh->nt, prm);
            else
                S->st = X->sh[0]->st;  // replicated host structure
            auto tt = std::chrono::steady_clock::now();
            build_tables(S);
            S->host_tables_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tt).count();
            S->host_build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        }
        if (structure_only) return;
        if (X->world > 1 && !X->virt) {
            NcclApi& api = nccl();
            if (!api.ok) throw NcclError(api.why);
            ncclUniqueId id;
            std::memcpy(&id, dist->nccl_uid, sizeof(id));
            ncclComm_t comm;
            setenv("NCCL_DEBUG", "INFO", 0);  // communicator set-up in the log (rank count, transports), unless set
            fprintf(stderr, "dh2: ncclCommInitRank rank %d of %d on device %d\n", X->rank, X->world, X->device);
            NK(api.CommInitRank(&comm, X->world, id, X->rank));
            X->comm = comm;
        }
        CK(configure_kernels());
        pool_setup(X->device);
        int optin = 0, nsm = 0;
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, X->device));
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, X->device));
        for (auto& S : X->sh) {
            if (!X->stream) {
                CK(cudaStreamCreateWithFlags(&S->own_stream, cudaStreamNonBlocking));
                X->stream = S->own_stream;
            }
            S->stream = X->stream;  // all shards of a context issue on one stream
        }
        {
            // every shard of a partition takes the same kind of plan (the exchanged C layouts differ):
            // the lean one if any shard's full plan does not fit its GPU (virtual mode: all of them
            // together on this GPU; NCCL: the maximum over the ranks)
            size_t freeb = 0, totb = 0;
            CK(cudaMemGetInfo(&freeb, &totb));
            freeb += pool_reusable(X->device);
            double need = 0.0;
            for (auto& S : X->sh) need = X->virt ? need + plan_bytes(S.get()) : std::max(need, (double)plan_bytes(S.get()));
            std::vector<double> v{need + (double)(256 << 20) > (double)freeb ? 1.0 : 0.0};
            reduce_doubles(X.get(), v, true);
            if (X->world > 1 && v[0] > 0.0)
                for (auto& S : X->sh) S->lean_required = true;
        }
        for (auto& S : X->sh) {
            S->P.smem_optin = optin - 1024;  // margin for the kernels' static shared memory
            S->P.num_sms = nsm;
            upload_all(S.get(), mesh->xyz, mesh->nv, mesh->tri);
            run_setup(S.get());
        }
        finish_all(X.get());
        // every rank must have passed the same mesh and parameters
        uint64_t h = fnv1a(mesh->xyz, sizeof(double) * 3 * (size_t)mesh->nv, 1469598103934665603ull);
        h = fnv1a(mesh->tri, sizeof(int64_t) * 3 * (size_t)mesh->nt, h);
        const double pv[5] = {p.kappa, (double)p.m, (double)p.leaf_size, p.eta1, p.eta2};
        check_same_args(X.get(), fnv1a(pv, sizeof(pv), h), "dh2_build_interp (mesh or parameters)");
    });
    if (rc != DH2_OK) return rc;
    *out = X.release();
    return DH2_OK;
}

int dh2_setup_device(dh2_ctx* X) {
    if (!X) return fail(nullptr, DH2_EINVAL, "null context");
    return guarded(X, [&] {
        require_device(X);
        CK(cudaSetDevice(X->device));
        for (auto& S : X->sh) {
            run_setup(S.get());
            S->recompressed = false;
        }
        X->recompressed = false;
        finish_all(X);
    });
}

int dh2_recompress(dh2_ctx* X, double eps, int32_t mode) {
    if (!X) return fail(nullptr, DH2_EINVAL, "null context");
    return guarded(X, [&] {
        if (!(eps >= 0.0) || mode < 0 || mode > 2) throw std::invalid_argument("invalid eps or mode");
        require_device(X);
        CK(cudaSetDevice(X->device));
        for (auto& S : X->sh) {
            S->eps = eps;
            S->mode = mode;
        }
        X->exch_bytes = 0;
        {
            const double a[2] = {eps, (double)mode};
            check_same_args(X, fnv1a(a, sizeof(a), 1469598103934665603ull), "dh2_recompress (eps or mode)");
        }
        // a failure part-way leaves the factors inconsistent: RECOMP is unavailable until a
        // recompression completes
        for (auto& S : X->sh) S->recompressed = false;
        X->recompressed = false;
        do_recompress(X, eps, mode);
        for (auto& S : X->sh) S->recompressed = true;
        X->recompressed = true;
    });
}

int dh2_matvec(dh2_ctx* X, int32_t which, const double* x, double* y, int32_t flags) {
    if (!X) return fail(nullptr, DH2_EINVAL, "null context");
    return guarded(X, [&] {
        if (!x || !y || (which != DH2_ORIG && which != DH2_RECOMP)) throw std::invalid_argument("invalid matvec arguments");
        if (which == DH2_RECOMP && !X->recompressed) throw StateError("RECOMP matvec before dh2_recompress");
        require_device(X);
        CK(cudaSetDevice(X->device));
        Shard* S0 = X->sh[0].get();
        const size_t nb = (size_t)S0->n * sizeof(double2);
        if (flags & DH2_DEVICE_PTRS) {
            do_matvec(X, which == DH2_RECOMP, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y),
                      flags & DH2_ADD_NEAR);
        } else {
            CK(cudaMemcpyAsync(S0->d_x.p, x, nb, cudaMemcpyHostToDevice, X->stream));
            do_matvec(X, which == DH2_RECOMP, S0->d_x.p, S0->d_y.p, flags & DH2_ADD_NEAR);
            CK(cudaMemcpyAsync(y, S0->d_y.p, nb, cudaMemcpyDeviceToHost, X->stream));
        }
        finish_all(X);
    });
}

int dh2_nearfield_assemble(dh2_ctx* X, int32_t nq_singular, int32_t nq_regular) {
    if (!X) return fail(nullptr, DH2_EINVAL, "null context");
    return guarded(X, [&] {
        require_device(X);
        CK(cudaSetDevice(X->device));
        for (auto& S : X->sh) near_assemble(S.get(), nq_singular, nq_regular);
        finish_all(X);
    });
}

int dh2_storage(const dh2_ctx* C, int32_t which, dh2_storage_report* out) {
    if (!C || !out) return fail(nullptr, DH2_EINVAL, "null argument");
    dh2_ctx* X = const_cast<dh2_ctx*>(C);
    return guarded(X, [&] {
        if (which == DH2_RECOMP && !X->recompressed) throw StateError("RECOMP storage before dh2_recompress");
        if (which != DH2_ORIG && which != DH2_RECOMP) throw std::invalid_argument("invalid which");
        std::vector<double> sum(6, 0.0), mx(1, 0.0);
        for (auto& S : X->sh) {
            double v[7];
            storage_partial(S.get(), which, v);
            for (int i = 0; i < 6; ++i) sum[i] += v[i];
            mx[0] = std::max(mx[0], v[6]);
        }
        if (which == DH2_ORIG) sum[4] = sum[5] = 1;  // the interpolation rank k, counted once
        if (X->sh[0]->device != DH2_DEVICE_NONE) {
            reduce_doubles(X, sum, false);
            reduce_doubles(X, mx, true);
        }
        if (which == DH2_ORIG) {
            sum[4] = X->sh[0]->k;
            sum[5] = 1;
        }
        const double n = X->sh[0]->n;
        out->n = X->sh[0]->n;
        out->row_basis_bytes = sum[0];
        out->col_basis_bytes = sum[1];
        out->coupling_bytes = sum[2];
        out->nearfield_bytes = sum[3];
        out->kb_per_dof_basis = (sum[0] + sum[1]) / n / 1024.0;
        out->kb_per_dof_matrix = (sum[0] + sum[1] + sum[2] + sum[3]) / n / 1024.0;
        out->max_rank = (int32_t)mx[0];
        out->mean_rank = sum[5] > 0 ? sum[4] / sum[5] : 0.0;
    });
}

int dh2_set_stream(dh2_ctx* X, void* stream) {
    if (!X) return fail(nullptr, DH2_EINVAL, "null context");
    X->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : X->sh[0]->own_stream;
    for (auto& S : X->sh) S->stream = X->stream;
    return DH2_OK;
}

int dh2_set_option(dh2_ctx* X, const char* name, int64_t value) {
    if (!X || !name) return fail(nullptr, DH2_EINVAL, "null argument");
    const std::string nm(name);
    if (nm == "truncate_workspace") {  // 1: force the global-workspace truncation path (tests)
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "truncate_workspace must be 0 or 1");
        for (auto& S : X->sh) S->force_ws = (int)value;
        return DH2_OK;
    }
    if (nm == "fuse_leaf_weights") {  // leaf Zhat folded into the truncation, never stored (fuse_leaf_level)
        if (value < 0 || value > 2) return fail(X, DH2_EINVAL, "fuse_leaf_weights must be 0, 1 or 2");
        for (auto& S : X->sh) S->fuse_leaf = (int)value;
        return DH2_OK;
    }
    if (nm == "fuse_direct_rows") {  // fused leaf QR: stacks up to this height form M^* directly (tests: 0)
        if (value < 0 || value > 64) return fail(X, DH2_EINVAL, "fuse_direct_rows must be in [0, 64]");
        for (auto& S : X->sh) S->fuse_direct = (int)value;
        return DH2_OK;
    }
    if (nm == "qr_wy") {  // 0: column-by-column chunk appends (A/B and tests)
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "qr_wy must be 0 or 1");
        for (auto& S : X->sh) S->P.qr_wy = S->qr_wy_init = (int)value;
        return DH2_OK;
    }
    if (nm == "near_tma") {  // nearfield matvec: 1 = TMA bulk-copy ring (default), 0 = direct global loads (A/B)
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, nm + " must be 0 or 1");
        for (auto& S : X->sh) S->near_tma = (int)value;
        return DH2_OK;
    }
    if (nm == "mv_forward_warp") {  // matvec, leaf forward transform: 1 = warp per coefficient (default), 0 = thread per coefficient
        if (value < 0 || value > 2) return fail(X, DH2_EINVAL, nm + " must be 0, 1 or 2");
        for (auto& S : X->sh) S->P.mv_fwd_warp = S->mv_fwd_warp_init = (int)value;
        return DH2_OK;
    }
    if (nm == "bw_variant") {  // block weights at k > 64: 1 = unrolled loads + register-blocked norm GEMM
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, nm + " must be 0 or 1");
        for (auto& S : X->sh) S->P.bw_variant = S->bw_variant_init = (int)value;
        return DH2_OK;
    }
    if (nm == "trunc64_threads") {
        if (value != 64 && value != 128 && value != 256) return fail(X, DH2_EINVAL, "trunc64_threads must be 64, 128 or 256");
        for (auto& S : X->sh) S->P.t64_threads = S->t64_threads_init = (int)value;
        return DH2_OK;
    }
    if (nm == "truncate_split64") {  // 0: leaves of 33..64 truncated by one kernel (k_truncate)
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "truncate_split64 must be 0 or 1");
        for (auto& S : X->sh) S->split_trunc64 = (int)value;
        return DH2_OK;
    }
    if (nm == "truncate_split64_inner") {  // 0: inner levels (k > 64, <= 64 rows) truncated by one kernel
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "truncate_split64_inner must be 0 or 1");
        for (auto& S : X->sh) S->split_trunc64_inner = (int)value;
        return DH2_OK;
    }
    if (nm == "qr_cq64" || nm == "qr_cq64_tw") {  // k <= 64: 0 CTA-cooperative, 1 (3: rows by thread-column FMAs) column-per-thread
        if (value != 0 && value != 1 && value != 3) return fail(X, DH2_EINVAL, nm + " must be 0, 1 or 3");
        for (auto& S : X->sh) {
            if (nm == "qr_cq64")
                S->P.qr_cq64 = S->qr_cq64_init = (int)value;
            else
                S->P.qr_cq64_tw = S->qr_cq64_tw_init = (int)value;
        }
        return DH2_OK;
    }
    if (nm == "qr_cq" || nm == "qr_cq_tw" || nm == "qr_cq_tw_leaf") {  // 0: k > 64 basis (total) weights by the CTA-cooperative appends
        if (value < 0 || value > 3) return fail(X, DH2_EINVAL, nm + " must be 0..3 (variant)");
        for (auto& S : X->sh) {
            if (nm == "qr_cq")
                S->P.qr_cq = S->qr_cq_init = (int)value;
            else if (nm == "qr_cq_tw")
                S->P.qr_cq_tw = S->qr_cq_tw_init = (int)value;
            else
                S->P.qr_cq_tw_leaf = S->qr_cq_tw_leaf_init = (int)value;
        }
        return DH2_OK;
    }
    if (nm == "trunc_direct") {  // 1: the leaf truncation factorises M^* = Zhat V^* directly (no streamed appends)
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "trunc_direct must be 0 or 1");
        for (auto& S : X->sh) S->P.trunc_mode = S->trunc_mode_init = (int)value;
        return DH2_OK;
    }
    if (nm == "qr_flag") {  // 0: one block barrier per reflection in the chunk appends (A/B and tests)
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "qr_flag must be 0 or 1");
        for (auto& S : X->sh) S->P.qr_flag = S->qr_flag_init = (int)value;
        return DH2_OK;
    }
    if (nm == "truncate_split") {  // 0: the one-kernel truncation also for leaves <= 32 (tests)
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "truncate_split must be 0 or 1");
        for (auto& S : X->sh) S->split_trunc = (int)value;
        return DH2_OK;
    }
    if (nm == "lean_chunks") {  // > 0: re-lay the context out on the memory-lean chunked plan with that many chunks
        if (value < 1 || value > (1 << 20)) return fail(X, DH2_EINVAL, "lean_chunks must be >= 1");
        return guarded(X, [&] {
            if (X->world > 1 && !X->virt) throw NotImpl("lean_chunks on an NCCL context: the planner chooses per rank");
            for (auto& Sp : X->sh) {
            Shard* S = Sp.get();
            if (S->device == DH2_DEVICE_NONE) {  // structure-only context: the host plan alone (tests)
                lean_plan(S, (int)value);
                continue;
            }
            if (!S->sym_ok || !S->sym_opt) throw NotImpl("the memory-lean plan needs adjoint_symmetry = 1");
            CK(cudaSetDevice(S->device));
            CK(cudaStreamSynchronize(S->stream));
            // release the full plan's pools, then lay out and set up the lean plan
            S->d_VR.free();
            S->d_E.free();
            S->d_S.free();
            S->d_St.free();
            for (PassH* P : {&S->row, &S->col}) {
                P->d_Z.free();
                P->d_C.free();
                P->d_Q.free();
            }
            lean_plan(S, (int)value);
            upload_all(S, nullptr, 0, nullptr);
            run_setup(S);
            S->finish();
            S->recompressed = false;
            }
            X->segs.clear();  // exchange segments refer to the previous layout
            X->recompressed = false;
        });
    }
    if (nm == "adjoint_symmetry") {
        if (value != 0 && value != 1) return fail(X, DH2_EINVAL, "adjoint_symmetry must be 0 or 1");
        if (value == 0 && X->sh[0]->lean.on) return fail(X, DH2_ENOTIMPL, "the memory-lean plan needs adjoint_symmetry = 1");
        if (value == 0 && X->world > 1) return fail(X, DH2_ENOTIMPL, "sharded recompression needs adjoint_symmetry = 1");
        for (auto& S : X->sh) S->sym_opt = (int)value;
        return DH2_OK;
    }
    return fail(X, DH2_EINVAL, "unknown option " + nm);
}

int dh2_set_profiling(dh2_ctx* X, int32_t enable) {
    if (!X) return fail(nullptr, DH2_EINVAL, "null context");
    for (auto& S : X->sh) S->profiling = enable != 0;
    return DH2_OK;
}

int dh2_get_stats(const dh2_ctx* C, char* buf, int64_t* len) {
    if (!C || !len) return fail(nullptr, DH2_EINVAL, "null argument");
    const Shard* S0 = C->sh[0].get();
    const Structure& S = S0->st;
    std::map<std::string, KStat> ks;
    int64_t launches = 0, ws = 0;
    size_t devb = 0;
    for (auto& sh : C->sh) {
        for (auto& kv : sh->kstat) {
            KStat& a = ks[kv.first];
            a.launches += kv.second.launches;
            a.ms += kv.second.ms;
            a.flops += kv.second.flops;
            a.bytes += kv.second.bytes;
        }
        launches += sh->launches_total;
        ws += sh->ws_launches;
        devb += plan_bytes(sh.get());
    }
    std::ostringstream o;
    o.precision(17);
    int64_t nrow = (int64_t)S0->row.bp.size(), ncol = (int64_t)S0->col.bp.size();
    o << "{\"n\": " << S0->n << ", \"k\": " << S0->k << ", \"depth\": " << S.ct.depth
      << ", \"clusters\": " << S0->nclusters << ", \"blocks\": " << S.blocks.size() << ", \"near\": " << S.near.size()
      << ", \"row_pairs\": " << nrow << ", \"col_pairs\": " << ncol << ", \"basis_pairs\": " << S0->bp_t.size()
      << ", \"world\": " << C->world << ", \"rank\": " << C->rank << ", \"shards_here\": " << C->sh.size()
      << ", \"transport\": \"" << (C->world == 1 ? "none" : C->virt ? "virtual" : "nccl") << "\""
      << ", \"own_blocks\": " << (S0->b_hi - S0->b_lo) << ", \"exchange_bytes\": " << C->exch_bytes
      << ", \"host_build_ms\": " << S0->host_build_ms << ", \"host_phases_ms\": {\"tree\": " << S.ms_tree
      << ", \"dirs\": " << S.ms_dirs << ", \"blocks\": " << S.ms_blocks << ", \"closure\": " << S.ms_closure
      << ", \"tables\": " << S0->host_tables_ms << ", \"tables_split\": [" << S0->tab_ms[0] << ", " << S0->tab_ms[1]
      << ", " << S0->tab_ms[2] << ", " << S0->tab_ms[3] << ", " << S0->tab_ms[4] << ", " << S0->tab_ms[5]
      << "]}, \"launches_total\": " << launches
      << ", \"E_row\": " << C->E_row << ", \"E_col\": " << C->E_col << ", \"far2\": " << C->far2
      << ", \"device_bytes\": " << devb << ", \"shard_device_bytes\": [";
    for (size_t i = 0; i < C->sh.size(); ++i) o << (i ? ", " : "") << plan_bytes(C->sh[i].get());
    o << "], \"mirror_missing\": " << S0->mirror_missing
      << ", \"truncate_ws_launches\": " << ws;
    {
        const LeanState& Ln = S0->lean;
        o << ", \"lean\": {\"on\": " << (Ln.on ? "true" : "false") << ", \"chunks\": " << Ln.G << ", \"l0\": " << Ln.l0
          << ", \"VR_persist_bytes\": " << 16.0 * Ln.VR_persist << ", \"VR_scratch_bytes\": " << 16.0 * Ln.VR_scratch
          << ", \"Z_scratch_bytes\": " << 16.0 * Ln.Z_scratch << ", \"S_slots\": " << Ln.S_slots
          << ", \"C_pool_mapped\": " << Ln.Cpool.mapped_bytes() << ", \"Q_pool_mapped\": " << Ln.Qpool.mapped_bytes()
          << ", \"C_compact_bytes\": " << 16.0 * Ln.C_used << ", \"Q_compact_bytes\": " << 16.0 * Ln.Q_used
          << ", \"compact_items\": " << Ln.compact_items << ", \"device_used_peak\": " << Ln.peak_bytes
          << ", \"plan_bytes\": " << (Ln.on ? lean_bytes(S0) : 0.0) << ", \"wall_ms\": {";
        static const char* wn[6] = {"begin", "basis", "weights_truncate", "columns", "project", "finish"};
        for (size_t i = 0; i < S0->lean_wall_ms.size() && i < 6; ++i)
            o << (i ? ", " : "") << "\"" << wn[i] << "\": " << S0->lean_wall_ms[i];
        o << "}}";
    }
    {
        int64_t nb = 0, nv = 0, ns = 0;
        double ne = 0;
        bool on = true;
        for (auto& sh : C->sh)
            nb += sh->near.nblk, nv += sh->near.values, ns += sh->near.nsing, ne += sh->near.evals, on = on && sh->near.on;
        o << ", \"nearfield\": {\"assembled\": " << (on ? "true" : "false") << ", \"blocks\": " << nb
          << ", \"values\": " << nv << ", \"touching_entries\": " << ns << ", \"kernel_evals\": " << ne
          << ", \"nq_singular\": " << S0->near.nq_sing
          << ", \"nq_regular\": " << S0->near.nq_reg << "}";
    }
    for (int side = 0; side < 2; ++side) {
        o << (side ? ", \"fused_leaf_levels_col\": [" : ", \"fused_leaf_levels_row\": [");
        for (size_t i = 0; i < S0->fused_levels[side].size(); ++i) o << (i ? ", " : "") << S0->fused_levels[side][i];
        o << "]";
    }
    o << ", \"fused_append_pairs\": " << S0->fused_append
      << ", \"adjoint_symmetry\": {\"available\": " << (S0->sym_ok ? "true" : "false") << ", \"enabled\": " << S0->sym_opt
      << ", \"used\": " << (S0->sym_used ? "true" : "false") << ", \"row_only_setup\": " << (S0->sym_setup ? "true" : "false")
      << ", \"why_not\": \"" << S0->sym_why << "\"}"
      << ", \"kernels\": {";
    bool first = true;
    for (auto& kv : ks) {
        if (!first) o << ", ";
        first = false;
        o << "\"" << kv.first << "\": {\"launches\": " << kv.second.launches << ", \"ms\": " << kv.second.ms
          << ", \"flops\": " << kv.second.flops << ", \"bytes\": " << kv.second.bytes << "}";
    }
    o << "}}";
    (void)ws;
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
    dh2_ctx* X = const_cast<dh2_ctx*>(C);
    return guarded(X, [&] {
        const std::string nm(name);
        if (X->sh.size() > 1 && (nm == "rank_row" || nm == "rank_col")) {
            // merged over the virtual shards: each pair's rank from the shard that owns it
            static thread_local std::vector<int> merged;
            const bool row = nm == "rank_row";
            const PassH& X0 = row ? X->sh[0]->row : X->sh[0]->col;
            merged.assign(X0.bp.size(), 0);
            for (auto& S : X->sh) {
                const PassH& P = row ? S->row : S->col;
                for (int l = 0; l < (int)P.own_lo.size(); ++l)
                    for (int p = P.own_lo[l]; p < P.own_hi[l]; ++p) merged[p] = P.rank[p];
            }
            const int64_t bytes = (int64_t)merged.size() * sizeof(int);
            if (!buf) {
                *nbytes = bytes;
                return;
            }
            if (*nbytes < bytes) throw std::invalid_argument("export buffer too small for " + nm);
            std::memcpy(buf, merged.data(), bytes);
            *nbytes = bytes;
            return;
        }
        export_shard(X->sh[0].get(), name, buf, nbytes);
    });
}

int dh2_export_shard(const dh2_ctx* C, int32_t shard, const char* name, void* buf, int64_t* nbytes) {
    if (!C || !name || !nbytes) return fail(nullptr, DH2_EINVAL, "null argument");
    dh2_ctx* X = const_cast<dh2_ctx*>(C);
    return guarded(X, [&] {
        if (shard < 0 || shard >= (int)X->sh.size()) throw std::invalid_argument("shard index out of range");
        export_shard(X->sh[shard].get(), name, buf, nbytes);
    });
}

int dh2_destroy(dh2_ctx* C) {
    if (!C) return DH2_OK;
    delete C;
    return DH2_OK;
}

const char* dh2_last_error(const dh2_ctx* C) {
    if (C) return C->err.c_str();
    return g_last_error.c_str();
}

}  // extern "C"
