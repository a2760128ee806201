"""Named workload configurations.

C1..C5 are BASELINE.json configs[0..4]; P0..P3 are the tiny
parity configurations of SURVEY.md §8(c) that exercise nesting (C1 has admissible
blocks on the leaf level only); P4/P5 run the C4/C5 order m = 5 (k = 125) and eps = 1e-6
at oracle-friendly sizes.  q is the per-face refinement: sphere n = 8 q^2,
cube n = 12 q^2.  eta1 = 1 (directions), eta2 = 10 (admissibility) as BASELINE.json
states.
"""

CONFIGS = {
    # tiny parity configs (tests only)
    "P0": dict(mesh="sphere", q=8, kappa=0.0, m=3, leaf=16, eta1=1.0, eta2=10.0, eps=1e-4),
    "P1": dict(mesh="sphere", q=8, kappa=4.0, m=3, leaf=8, eta1=1.0, eta2=10.0, eps=1e-4),
    "P2": dict(mesh="sphere", q=16, kappa=8.0, m=3, leaf=16, eta1=1.0, eta2=10.0, eps=1e-4),
    "P3": dict(mesh="cube", q=8, kappa=5.0, m=3, leaf=16, eta1=1.0, eta2=10.0, eps=1e-4),
    # k = 125 (m = 5) at the C4/C5 tolerance eps = 1e-6: cube (flat boxes) and sphere
    "P4": dict(mesh="cube", q=8, kappa=5.0, m=5, leaf=16, eta1=1.0, eta2=10.0, eps=1e-6),
    "P5": dict(mesh="sphere", q=16, kappa=6.0, m=5, leaf=16, eta1=1.0, eta2=10.0, eps=1e-6),
    # the C5 leaf shape (cube, flat leaves of 48 triangles) at k = 125
    "P6": dict(mesh="cube", q=8, kappa=5.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
    # three active levels of that shape: regression case of DESIGN reading N2 (numerically zero columns)
    "P7": dict(mesh="cube", q=16, kappa=14.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
    # an open sphere (every 37th triangle removed, n = 498) with leaf 15: tree levels mixing leaf and
    # inner clusters (median splits of sizes that are no power-of-two multiple)
    "P8": dict(mesh="sphere_cut", q=8, cut_every=37, cut_offset=5, kappa=4.0, m=3, leaf=15, eta1=1.0, eta2=10.0,
               eps=1e-4),
    # the PAPER's parameter setting (NEXT-3; eta1 = 10 for the directions, eta2 = 1 for
    # admissibility, m = 4, leaf 32 in Table 3): many blocks per (t,c) (sigma up to 47 / 28), so Z^*
    # stacks 1,000+ rows ("wide Z") -- P9 at desk scale (m = 3), P11 = the shape of Table 3's first
    # row (sphere n = 8192, kappa = 16)
    "P9": dict(mesh="sphere", q=16, kappa=4.0, m=3, leaf=16, eta1=10.0, eta2=1.0, eps=1e-4),
    "P11": dict(mesh="sphere", q=32, kappa=16.0, m=4, leaf=32, eta1=10.0, eta2=1.0, eps=1e-4),
    # BASELINE.json configs
    "C1": dict(mesh="sphere", q=8, kappa=4.0, m=3, leaf=16, eta1=1.0, eta2=10.0, eps=1e-4),
    "C2": dict(mesh="sphere", q=32, kappa=16.0, m=4, leaf=32, eta1=1.0, eta2=10.0, eps=1e-4),
    "C3": dict(mesh="sphere", q=64, kappa=32.0, m=4, leaf=32, eta1=1.0, eta2=10.0, eps=1e-5),
    "C4": dict(mesh="sphere", q=128, kappa=64.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
    "C5": dict(mesh="cube", q=128, kappa=115.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
    # C4 / C5 scaled down to one GPU's memory (same order m = 5, leaf 64, eps = 1e-6 and kappa h ~ 0.9):
    # the full C4/C5 need the partitioned or memory-lean path
    "C4s": dict(mesh="sphere", q=32, kappa=16.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
    "C5s": dict(mesh="cube", q=32, kappa=29.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
    # the largest scale-downs that fit one GPU (155 / 96 GB device plans)
    "C4q": dict(mesh="sphere", q=64, kappa=32.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
    "C5q": dict(mesh="cube", q=48, kappa=43.0, m=5, leaf=64, eta1=1.0, eta2=10.0, eps=1e-6),
}


def get_config(name):
    cfg = dict(CONFIGS[name])
    cfg["name"] = name
    return cfg
