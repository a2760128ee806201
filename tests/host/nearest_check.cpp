// nearest() with its tile index (dh2_host.cpp) against the exhaustive search of P:396-403 with the
// tie rule of DESIGN reading R4, written out here: random, small-integer (tie-prone) and
// direction-set inputs on every level of two wavenumbers.  Built and run by tests/test_host_nearest.py.
#include "dh2_host.h"
#include <cstdlib>
#include <cstdio>
#include <cmath>
#include <random>
#include <vector>
static int64_t brute(const std::vector<double>& Dl, const double y[3]) {
    int64_t nd = (int64_t)Dl.size() / 3;
    if (nd == 1) return 0;
    static const double wr[3] = {1.0, std::sqrt(2.0), std::sqrt(3.0)};
    const double wn = std::sqrt((wr[0] * wr[0] + wr[1] * wr[1]) + wr[2] * wr[2]);
    const double w[3] = {wr[0] / wn, wr[1] / wn, wr[2] / wn};
    double mn = INFINITY;
    for (int64_t c = 0; c < nd; ++c) {
        double d0 = y[0] - Dl[3 * c], d1 = y[1] - Dl[3 * c + 1], d2 = y[2] - Dl[3 * c + 2];
        double dd = (d0 * d0 + d1 * d1) + d2 * d2;
        if (dd < mn) mn = dd;
    }
    const double thr = mn + 1e-12;
    const double yw = (y[0] * w[0] + y[1] * w[1]) + y[2] * w[2];
    const double s = yw >= 0.0 ? 1.0 : -1.0;
    int64_t best = -1;
    double bscore = -INFINITY;
    for (int64_t c = 0; c < nd; ++c) {
        double d0 = y[0] - Dl[3 * c], d1 = y[1] - Dl[3 * c + 1], d2 = y[2] - Dl[3 * c + 2];
        double dd = (d0 * d0 + d1 * d1) + d2 * d2;
        if (dd <= thr) {
            double sc = s * ((Dl[3 * c] * w[0] + Dl[3 * c + 1] * w[1]) + Dl[3 * c + 2] * w[2]);
            if (best < 0 || sc > bscore) { best = c; bscore = sc; }
        }
    }
    return best;
}
int main(int argc, char** argv) {
    if (argc < 5) return 2;
    const int64_t nv = atoll(argv[3]), nt = atoll(argv[4]);
    FILE* f = fopen(argv[1], "rb"); std::vector<double> xyz(nv * 3); if(fread(xyz.data(), 8, xyz.size(), f) != xyz.size()) return 1; fclose(f);
    f = fopen(argv[2], "rb"); std::vector<int64_t> tri(nt * 3); if(fread(tri.data(), 8, tri.size(), f) != tri.size()) return 1; fclose(f);
    std::mt19937_64 g(1);
    std::normal_distribution<double> N(0, 1);
    std::uniform_int_distribution<int> U(-3, 3);
    long bad = 0, tot = 0;
    for (double kappa : {16.0, 43.0}) {
        dh2::Params p; p.kappa = kappa; p.m = 4; p.leaf = 32; p.eta1 = 1; p.eta2 = 10;
        dh2::Structure S;
        S.build(xyz.data(), nv, tri.data(), nt, p);
        for (int l = 0; l <= S.ct.depth; ++l) {
            const auto& Dl = S.D(l);
            int64_t nd = Dl.size() / 3;
            if (nd > 12000) continue;
            auto check = [&](double y[3]) {
                ++tot;
                int64_t a = S.nearest(l, y), b = brute(Dl, y);
                if (a != b) { if (bad < 10) printf("MISMATCH kappa %g level %d y %.17g %.17g %.17g: %ld vs %ld\n", kappa, l, y[0], y[1], y[2], (long)a, (long)b); ++bad; }
            };
            for (int i = 0; i < 600; ++i) {
                double y[3] = {N(g), N(g), N(g)};
                double n = std::sqrt((y[0] * y[0] + y[1] * y[1]) + y[2] * y[2]);
                for (int a = 0; a < 3; ++a) y[a] /= n;
                check(y);
            }
            // symmetric / tie-prone inputs: small-integer vectors, the directions themselves, their negatives,
            // the directions of the coarser and finer levels (sd maps)
            for (int i = 0; i < 600; ++i) {
                double y[3] = {(double)U(g), (double)U(g), (double)U(g)};
                double n = std::sqrt((y[0] * y[0] + y[1] * y[1]) + y[2] * y[2]);
                if (n == 0) continue;
                for (int a = 0; a < 3; ++a) y[a] /= n;
                check(y);
            }
            for (int64_t c = 0; c < nd; ++c) {
                double y[3] = {Dl[3 * c], Dl[3 * c + 1], Dl[3 * c + 2]};
                check(y);
                double z[3] = {-y[0], -y[1], -y[2]};
                check(z);
            }
            for (int l2 : {l - 1, l + 1}) {
                if (l2 < 0 || l2 > S.ct.depth || S.D(l2).size() / 3 > 12000) continue;
                const auto& D2 = S.D(l2);
                for (size_t c = 0; c < D2.size() / 3; ++c) { double y[3] = {D2[3 * c], D2[3 * c + 1], D2[3 * c + 2]}; check(y); }
            }
        }
    }
    printf("checked %ld mismatches %ld\n", tot, bad);
    return bad != 0;
}
