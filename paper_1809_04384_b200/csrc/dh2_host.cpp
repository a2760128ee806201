// Host structures of the DH^2 matrix — see dh2_host.h.  Every formula cites PAPER.md.
#include "dh2_host.h"

#include <algorithm>
#include <iterator>
#include <chrono>
#include <cmath>
#include <numeric>
#include <stdexcept>

namespace dh2 {

static inline double norm3(double a, double b, double c) { return std::sqrt((a * a + b * b) + c * c); }

void validate_mesh(const double* xyz, int64_t nv, const int64_t* tri, int64_t nt) {
    if (nv < 3 || nt < 1 || !xyz || !tri) throw std::invalid_argument("empty mesh");
    for (int64_t i = 0; i < nt; ++i) {
        for (int j = 0; j < 3; ++j)
            if (tri[3 * i + j] < 0 || tri[3 * i + j] >= nv) throw std::invalid_argument("triangle index out of range");
        const double* a = xyz + 3 * tri[3 * i];
        const double* b = xyz + 3 * tri[3 * i + 1];
        const double* c = xyz + 3 * tri[3 * i + 2];
        double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double cr0 = e1[1] * e2[2] - e1[2] * e2[1];
        double cr1 = e1[2] * e2[0] - e1[0] * e2[2];
        double cr2 = e1[0] * e2[1] - e1[1] * e2[0];
        if (!(norm3(cr0, cr1, cr2) > 0.0)) throw std::invalid_argument("triangle with area <= 0");
    }
}

// Cluster tree: median split along the longest axis of the tight box (DESIGN
// reading R-cluster), ties of the axis to the lowest axis, of the centroid to the triangle
// index; the first child receives ceil(#t/2); split while #t > leaf; BFS numbering.
void Structure::build_tree(const double* xyz, const int64_t* tri, int64_t nt) {
    ClusterTree& T = ct;
    T.n = nt;
    std::vector<double> cen(3 * nt);
    for (int64_t i = 0; i < nt; ++i)
        for (int a = 0; a < 3; ++a)
            cen[3 * i + a] = ((xyz[3 * tri[3 * i] + a] + xyz[3 * tri[3 * i + 1] + a]) + xyz[3 * tri[3 * i + 2] + a]) / 3.0;
    T.perm.resize(nt);
    std::iota(T.perm.begin(), T.perm.end(), 0);
    T.begin = {0};
    T.end = {nt};
    T.level = {0};
    T.parent = {-1};
    T.child0 = {-1};
    T.child1 = {-1};
    for (size_t t = 0; t < T.begin.size(); ++t) {
        int64_t b = T.begin[t], e = T.end[t];
        double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t p = b; p < e; ++p)
            for (int v = 0; v < 3; ++v)
                for (int a = 0; a < 3; ++a) {
                    double x = xyz[3 * tri[3 * T.perm[p] + v] + a];
                    lo[a] = std::min(lo[a], x);
                    hi[a] = std::max(hi[a], x);
                }
        for (int a = 0; a < 3; ++a) {
            T.lo.push_back(lo[a]);
            T.hi.push_back(hi[a]);
        }
        int64_t cnt = e - b;
        if (cnt > p.leaf) {
            double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
            int axis = 0;
            for (int a = 1; a < 3; ++a)
                if (ext[a] > ext[axis]) axis = a;
            auto key_less = [&](int64_t i, int64_t j) {
                double ki = cen[3 * i + axis], kj = cen[3 * j + axis];
                return ki < kj || (ki == kj && i < j);
            };
            // median split: the key order is total (ties by index), so partitioning at the median
            // gives the halves of the sorted order; a half that becomes a leaf keeps the sorted
            // order (the order of a cluster that is split again is irrelevant: it is re-partitioned)
            int64_t half = (cnt + 1) / 2;
            std::nth_element(T.perm.begin() + b, T.perm.begin() + b + half, T.perm.begin() + e, key_less);
            if (half <= p.leaf) std::sort(T.perm.begin() + b, T.perm.begin() + b + half, key_less);
            if (cnt - half <= p.leaf) std::sort(T.perm.begin() + b + half, T.perm.begin() + e, key_less);
            int64_t c0 = (int64_t)T.begin.size();
            int64_t rng[2][2] = {{b, b + half}, {b + half, e}};
            for (auto& r : rng) {
                T.begin.push_back(r[0]);
                T.end.push_back(r[1]);
                T.level.push_back(T.level[t] + 1);
                T.parent.push_back((int64_t)t);
                T.child0.push_back(-1);
                T.child1.push_back(-1);
            }
            T.child0[t] = c0;
            T.child1[t] = c0 + 1;
        }
    }
    int64_t nc = (int64_t)T.begin.size();
    T.depth = 0;
    for (int64_t t = 0; t < nc; ++t) T.depth = std::max<int>(T.depth, (int)T.level[t]);
    T.levels.assign(T.depth + 1, {});
    T.diam.resize(nc);
    T.mid.resize(3 * nc);
    for (int64_t t = 0; t < nc; ++t) {
        T.levels[T.level[t]].push_back(t);
        double e0 = T.hi[3 * t] - T.lo[3 * t], e1 = T.hi[3 * t + 1] - T.lo[3 * t + 1], e2 = T.hi[3 * t + 2] - T.lo[3 * t + 2];
        T.diam[t] = norm3(e0, e1, e2);  // diam(B_t)
        for (int a = 0; a < 3; ++a) T.mid[3 * t + a] = 0.5 * (T.lo[3 * t + a] + T.hi[3 * t + a]);
    }
}

// Remark 2.4: D_l = {0} if kappa d_l <= eta1; else m = ceil(sqrt2 kappa d_l/eta1) and
// the 6 m^2 normalised centres of the squares of the faces of [-1,1]^3 (DESIGN reading Q2),
// faces -x,+x,-y,+y,-z,+z, centres (2i+1-m)/m on the two remaining axes in increasing order.
const std::vector<double>& Structure::D(int l) {
    if (dirs_ready[l]) return dirs[l];
    std::vector<double>& out = dirs[l];
    int md = mdir[l];
    if (md == 0) {
        out = {0.0, 0.0, 0.0};
    } else {
        out.reserve((size_t)18 * md * md);
        for (int a = 0; a < 3; ++a) {
            int u = a == 0 ? 1 : 0, w = a == 2 ? 1 : 2;
            for (int sgn = -1; sgn <= 1; sgn += 2)
                for (int iu = 0; iu < md; ++iu)
                    for (int iv = 0; iv < md; ++iv) {
                        double q[3];
                        q[a] = (double)sgn;
                        q[u] = (double)(2 * iu + 1 - md) / md;
                        q[w] = (double)(2 * iv + 1 - md) / md;
                        double nr = norm3(q[0], q[1], q[2]);
                        out.push_back(q[0] / nr);
                        out.push_back(q[1] / nr);
                        out.push_back(q[2] / nr);
                    }
        }
    }
    build_tiles(l);
    dirs_ready[l] = 1;
    return out;
}

// Search index of D_l for nearest(): the m x m squares of each face grouped in T x T tiles
// (T ~ sqrt m), each with the mean of its directions and the largest distance to one of them.
void Structure::build_tiles(int l) {
    if ((int)tiles.size() <= l) tiles.resize(l + 1);
    DirTiles& X = tiles[l];
    X = DirTiles{};
    const int md = mdir[l];
    if (md < 4) return;  // <= 54 directions: exhaustive search
    const std::vector<double>& Dl = dirs[l];
    const int T = std::max(2, (int)std::lround(std::sqrt((double)md)));
    const int nt = (md + T - 1) / T;
    X.ptr.push_back(0);
    for (int f = 0; f < 6; ++f)
        for (int tu = 0; tu < nt; ++tu)
            for (int tv = 0; tv < nt; ++tv) {
                double cen[3] = {0.0, 0.0, 0.0};
                const size_t first = X.member.size();
                for (int iu = tu * T; iu < std::min(md, (tu + 1) * T); ++iu)
                    for (int iv = tv * T; iv < std::min(md, (tv + 1) * T); ++iv) {
                        const int64_t c = ((int64_t)f * md + iu) * md + iv;  // order of D(l)
                        X.member.push_back(c);
                        for (int a = 0; a < 3; ++a) cen[a] += Dl[3 * c + a];
                    }
                const double cnt = (double)(X.member.size() - first);
                double r = 0.0;
                for (int a = 0; a < 3; ++a) cen[a] /= cnt;
                for (size_t i = first; i < X.member.size(); ++i) {
                    const int64_t c = X.member[i];
                    r = std::max(r, norm3(Dl[3 * c] - cen[0], Dl[3 * c + 1] - cen[1], Dl[3 * c + 2] - cen[2]));
                }
                X.centre.insert(X.centre.end(), cen, cen + 3);
                X.radius.push_back(r);
                X.ptr.push_back((int64_t)X.member.size());
            }
}

// Best approximation of y in D_l with the symmetric tie rule (DESIGN reading Q4):
// candidates |y-c|^2 <= min + 1e-12, maximise s<c,w>, s = sign<y,w>, w = (1,sqrt2,sqrt3)/sqrt6.
int64_t Structure::nearest(int l, const double y[3]) {
    const std::vector<double>& Dl = D(l);
    int64_t nd = (int64_t)Dl.size() / 3;
    if (nd == 1) return 0;
    static const double wr[3] = {1.0, std::sqrt(2.0), std::sqrt(3.0)};
    const double wn = norm3(wr[0], wr[1], wr[2]);
    const double w[3] = {wr[0] / wn, wr[1] / wn, wr[2] / wn};
    auto dist2 = [&](int64_t c) {
        double d0 = y[0] - Dl[3 * c], d1 = y[1] - Dl[3 * c + 1], d2 = y[2] - Dl[3 * c + 2];
        return (d0 * d0 + d1 * d1) + d2 * d2;
    };
    // Candidate set: every direction (exhaustive), or, with the tile index, the members of every
    // tile that can hold a direction within sqrt(U + 1e-12) of y, U = the smallest distance^2 in
    // the tile whose centre is nearest to y (triangle inequality |y - c| >= |y - centre| - radius,
    // with a 1e-7 margin for rounding).  That set contains the minimiser and every direction of
    // the tie window below, so mn, the window and the choice are those of the exhaustive search.
    thread_local std::vector<int64_t> cand;
    thread_local std::vector<double> e;
    cand.clear();
    const DirTiles* X = (int)tiles.size() > l && !tiles[l].ptr.empty() ? &tiles[l] : nullptr;
    if (X) {
        const int64_t ntl = (int64_t)X->radius.size();
        e.resize(ntl);  // squared distances to the tile centres
        int64_t tb = 0;
        for (int64_t i = 0; i < ntl; ++i) {
            const double d0 = y[0] - X->centre[3 * i], d1 = y[1] - X->centre[3 * i + 1], d2 = y[2] - X->centre[3 * i + 2];
            e[i] = (d0 * d0 + d1 * d1) + d2 * d2;
            if (e[i] < e[tb]) tb = i;
        }
        double U = INFINITY;
        for (int64_t q = X->ptr[tb]; q < X->ptr[tb + 1]; ++q) U = std::min(U, dist2(X->member[q]));
        const double rad = std::sqrt(U + 1e-12) + 1e-7;
        for (int64_t i = 0; i < ntl; ++i) {
            const double lim = rad + X->radius[i];  // |y - centre| <= rad + radius
            if (e[i] <= lim * lim * (1.0 + 1e-12))
                cand.insert(cand.end(), X->member.begin() + X->ptr[i], X->member.begin() + X->ptr[i + 1]);
        }
        std::sort(cand.begin(), cand.end());
    }
    const int64_t ncand = X ? (int64_t)cand.size() : nd;
    auto at = [&](int64_t i) { return X ? cand[i] : i; };
    double mn = INFINITY;
    for (int64_t i = 0; i < ncand; ++i) {
        double dd = dist2(at(i));
        if (dd < mn) mn = dd;
    }
    const double thr = mn + 1e-12;
    const double yw = (y[0] * w[0] + y[1] * w[1]) + y[2] * w[2];
    const double s = yw >= 0.0 ? 1.0 : -1.0;
    int64_t best = -1;
    double bscore = -INFINITY;
    for (int64_t i = 0; i < ncand; ++i) {
        const int64_t c = at(i);
        double dd = dist2(c);
        if (dd <= thr) {
            double sc = s * ((Dl[3 * c] * w[0] + Dl[3 * c + 1] * w[1]) + Dl[3 * c + 2] * w[2]);
            if (best < 0 || sc > bscore) {
                best = c;
                bscore = sc;
            }
        }
    }
    return best;
}

// sd_l(c) = nearest direction of D_{l+1} to c.
int64_t Structure::sd(int l, int64_t c) {
    std::vector<int64_t>& cache = sd_cache[l];
    if ((int64_t)cache.size() <= c) cache.resize(D(l).size() / 3, -1);
    if (cache[c] < 0) {
        const std::vector<double>& Dl = D(l);
        double y[3] = {Dl[3 * c], Dl[3 * c + 1], Dl[3 * c + 2]};
        cache[c] = nearest(l + 1, y);
    }
    return cache[c];
}

// Minimal block tree (Def. 2.5): level-synchronous recursion from (root, root);
// admissible (Eq. 3b, 3c) -> L+ with c_ts; else children if both have some; else L-.
void Structure::build_blocks() {
    ClusterTree& T = ct;
    std::vector<std::pair<int64_t, int64_t>> front = {{0, 0}};
    int lvl = 0;
    while (!front.empty()) {
        std::vector<std::pair<int64_t, int64_t>> next;
        std::vector<Block> adm;
        for (auto& ts : front) {
            int64_t t = ts.first, s = ts.second;
            double g[3];
            for (int a = 0; a < 3; ++a)
                g[a] = std::max(0.0, std::max(T.lo[3 * t + a] - T.hi[3 * s + a], T.lo[3 * s + a] - T.hi[3 * t + a]));
            double dist = norm3(g[0], g[1], g[2]);
            double dmax = std::max(T.diam[t], T.diam[s]);
            bool ok = (dmax <= p.eta2 * dist) && (p.kappa * (dmax * dmax) <= p.eta2 * dist);
            if (ok) {
                adm.push_back({t, s, -1});
            } else if (!T.is_leaf(t) && !T.is_leaf(s)) {
                int64_t tc[2] = {T.child0[t], T.child1[t]}, sc[2] = {T.child0[s], T.child1[s]};
                for (int i = 0; i < 2; ++i)
                    for (int j = 0; j < 2; ++j) next.push_back({tc[i], sc[j]});
            } else {
                near.push_back({t, s});
            }
        }
        if (!adm.empty()) {
            D(lvl);
#pragma omp parallel for schedule(dynamic, 64)
            for (int64_t i = 0; i < (int64_t)adm.size(); ++i) {
                int64_t t = adm[i].t, s = adm[i].s;
                double dv[3];
                for (int a = 0; a < 3; ++a) dv[a] = T.mid[3 * t + a] - T.mid[3 * s + a];
                double nr = norm3(dv[0], dv[1], dv[2]);
                double y[3] = {dv[0] / nr, dv[1] / nr, dv[2] / nr};
                adm[i].c = nearest(lvl, y);
            }
            blocks.insert(blocks.end(), adm.begin(), adm.end());
        }
        front.swap(next);
        ++lvl;
    }
    std::sort(blocks.begin(), blocks.end(), [](const Block& a, const Block& b) { return a.t < b.t || (a.t == b.t && a.s < b.s); });
    std::sort(near.begin(), near.end());
}

// Sort by (t, c) and drop duplicates: counting sort by cluster (a level's clusters are a
// contiguous BFS range), then each cluster's few directions.
static void sort_unique_pairs(std::vector<Pair>& v) {
    if (v.empty()) return;
    int64_t t0 = v[0].t, t1 = v[0].t;
    for (auto& pr : v) {
        t0 = std::min(t0, pr.t);
        t1 = std::max(t1, pr.t);
    }
    std::vector<int64_t> cnt(t1 - t0 + 2, 0);
    for (auto& pr : v) ++cnt[pr.t - t0 + 1];
    for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
    std::vector<Pair> out(v.size());
    {
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (auto& pr : v) out[pos[pr.t - t0]++] = pr;
    }
    size_t w = 0;
    for (size_t g = 0; g + 1 < cnt.size(); ++g) {
        auto a = out.begin() + cnt[g], b = out.begin() + cnt[g + 1];
        std::sort(a, b);
        for (auto it = a; it != b; ++it)
            if (w == 0 || !(out[w - 1] == *it)) out[w++] = *it;
    }
    out.resize(w);
    v.swap(out);
}

// Active pairs: (t, c_b) of every admissible block plus the closure (t', sd_t(c)).
std::vector<std::vector<Pair>> Structure::closure(bool row) {
    ClusterTree& T = ct;
    std::vector<std::vector<Pair>> pairs(T.depth + 1);
    for (auto& b : blocks) {
        int64_t t = row ? b.t : b.s;
        pairs[T.level[t]].push_back({t, b.c});
    }
    for (int l = 0; l <= T.depth; ++l) {
        auto& v = pairs[l];
        sort_unique_pairs(v);
        if (l == T.depth) break;
        // sd_l of every direction used on this level, computed in parallel into the cache
        // (D(l), D(l+1) and the cache are materialised first: nearest() then only reads)
        if (!v.empty()) {
            D(l);
            D(l + 1);
            std::vector<int64_t>& cache = sd_cache[l];
            if (cache.size() < D(l).size() / 3) cache.resize(D(l).size() / 3, -1);
            std::vector<int64_t> todo;
            for (auto& pr : v)
                if (!T.is_leaf(pr.t) && cache[pr.c] < 0 && (todo.empty() || todo.back() != pr.c)) todo.push_back(pr.c);
            std::sort(todo.begin(), todo.end());
            todo.erase(std::unique(todo.begin(), todo.end()), todo.end());
            const std::vector<double>& Dl = D(l);
#pragma omp parallel for schedule(dynamic, 16)
            for (int64_t i = 0; i < (int64_t)todo.size(); ++i) {
                const int64_t c = todo[i];
                double y[3] = {Dl[3 * c], Dl[3 * c + 1], Dl[3 * c + 2]};
                cache[c] = nearest(l + 1, y);
            }
        }
        for (auto& pr : v) {
            if (T.is_leaf(pr.t)) continue;
            int64_t c2 = sd(l, pr.c);
            pairs[l + 1].push_back({T.child0[pr.t], c2});
            pairs[l + 1].push_back({T.child1[pr.t], c2});
        }
    }
    return pairs;
}

void Structure::build(const double* xyz, int64_t nv, const int64_t* tri, int64_t nt, const Params& prm) {
    (void)nv;
    p = prm;
    k = p.m * p.m * p.m;
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    auto t0 = clk::now();
    build_tree(xyz, tri, nt);
    auto t1 = clk::now();
    ms_tree = ms(t0, t1);
    int L = ct.depth;
    d_level.assign(L + 1, 0.0);
    mdir.assign(L + 1, 0);
    for (int l = 0; l <= L; ++l) {
        double d = 0.0;
        for (int64_t t : ct.levels[l]) d = std::max(d, ct.diam[t]);
        d_level[l] = d;
        if (p.kappa * d <= p.eta1)
            mdir[l] = 0;
        else
            mdir[l] = (int)std::ceil(((std::sqrt(2.0) * p.kappa) * d) / p.eta1);
    }
    dirs.assign(L + 1, {});
    dirs_ready.assign(L + 1, 0);
    sd_cache.assign(L + 1, {});
    tiles.assign(L + 1, {});
    auto t2 = clk::now();
    ms_dirs = ms(t1, t2);
    build_blocks();
    auto t3 = clk::now();
    ms_blocks = ms(t2, t3);
    row_pairs = closure(true);
    col_pairs = closure(false);
    basis_pairs.assign(L + 1, {});
    for (int l = 0; l <= L; ++l) {
        auto& v = basis_pairs[l];  // union of the two sorted, duplicate-free lists
        v.reserve(row_pairs[l].size() + col_pairs[l].size());
        std::set_union(row_pairs[l].begin(), row_pairs[l].end(), col_pairs[l].begin(), col_pairs[l].end(), std::back_inserter(v));
        if (!v.empty() && first_level < 0) first_level = l;
    }
    // make sure every level that hosts pairs has its direction set materialised
    for (int l = 0; l <= L; ++l)
        if (!basis_pairs[l].empty()) D(l);
    ms_closure = ms(t3, clk::now());
}

}  // namespace dh2
