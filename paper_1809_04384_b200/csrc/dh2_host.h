// Host-side structures of the DH^2 matrix (§2): cluster tree, boxes,
// directions and sd maps, block tree, row/column pair closure, and the per-level
// schedules the device kernels consume.  Pure C++17; compiled with
// -ffp-contract=off so every floating-point decision follows the written order.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace dh2 {

struct Params {
    double kappa = 0.0;
    int m = 4;
    int leaf = 32;
    double eta1 = 1.0, eta2 = 10.0;
};

// Cluster tree (Def. 2.1) in BFS numbering; cluster t covers perm[begin[t], end[t]).
struct ClusterTree {
    int64_t n = 0;
    std::vector<int64_t> perm;  // position -> original triangle index
    std::vector<int64_t> begin, end, level, parent, child0, child1;
    std::vector<double> lo, hi;  // 3 per cluster (tight boxes)
    std::vector<double> diam, mid;
    int depth = 0;
    std::vector<std::vector<int64_t>> levels;
    bool is_leaf(int64_t t) const { return child0[t] < 0; }
    int64_t size(int64_t t) const { return end[t] - begin[t]; }
};

struct Pair {
    int64_t t;  // cluster
    int64_t c;  // direction index within D_level(t)
    bool operator<(const Pair& o) const { return t < o.t || (t == o.t && c < o.c); }
    bool operator==(const Pair& o) const { return t == o.t && c == o.c; }
};

struct Block {
    int64_t t, s, c;
};

struct Structure {
    Params p;
    int k = 0;
    ClusterTree ct;
    std::vector<double> d_level;
    std::vector<int> mdir;                 // 0 => D_l = {0}
    std::vector<std::vector<double>> dirs;  // 3 per direction; generated lazily (empty if unused)
    std::vector<char> dirs_ready;
    std::vector<std::vector<int64_t>> sd_cache;  // per level, -1 = not computed
    // per level: the directions grouped by tiles of adjacent face squares (search index of
    // nearest(); built with D(l); empty for small sets, which are searched exhaustively)
    struct DirTiles {
        std::vector<double> centre, radius;    // per tile: centre (3), max distance to a member
        std::vector<int64_t> ptr, member;      // members of tile i: member[ptr[i] .. ptr[i+1])
    };
    std::vector<DirTiles> tiles;
    std::vector<Block> blocks;                   // admissible leaves L+, sorted by (t, s)
    std::vector<std::pair<int64_t, int64_t>> near;  // inadmissible leaves L-
    std::vector<std::vector<Pair>> row_pairs, col_pairs, basis_pairs;  // per level, sorted
    int first_level = -1;  // first level with any pair
    double ms_tree = 0, ms_dirs = 0, ms_blocks = 0, ms_closure = 0;  // host phase timings

    void build(const double* xyz, int64_t nv, const int64_t* tri, int64_t nt, const Params& prm);
    const std::vector<double>& D(int level);
    int64_t sd(int level, int64_t c);
    int64_t nearest(int level, const double y[3]);

   private:
    void build_tree(const double* xyz, const int64_t* tri, int64_t nt);
    void build_blocks();
    void build_tiles(int level);
    std::vector<std::vector<Pair>> closure(bool row);
};

// Throws std::runtime_error on invalid input.
void validate_mesh(const double* xyz, int64_t nv, const int64_t* tri, int64_t nt);

}  // namespace dh2
