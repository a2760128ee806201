"""Pins of the oracle host structures (§2) — closed forms and invariants."""
import math

import numpy as np
import pytest

from synth import get_config, mesh_for
from oracle.structure import (ClusterTree, DH2Structure, admissible, box_dist, direction_set,
                              nearest_direction)


def _structure(name, **over):
    cfg = get_config(name)
    cfg.update(over)
    xyz, tri = mesh_for(cfg)
    return DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])


@pytest.fixture(scope="module", params=["P1", "P3", "C1"])
def st(request):
    return _structure(request.param)


def test_cluster_tree_partition(st):
    ct = st.ct
    assert sorted(ct.perm.tolist()) == list(range(st.n))
    for t in range(ct.nclusters):
        if ct.is_leaf(t):
            assert 1 <= ct.size(t) <= st.leaf
        else:
            c0, c1 = ct.children[t]
            assert ct.begin[c0] == ct.begin[t] and ct.end[c0] == ct.begin[c1] and ct.end[c1] == ct.end[t]
            assert ct.size(c0) == (ct.size(t) + 1) // 2  # first child gets ceil(n/2)
            assert ct.level[c0] == ct.level[t] + 1
        # tight box contains all vertices of all triangles of t (supp phi_i in B_t)
        v = st.xyz[st.tri[ct.indices(t)]].reshape(-1, 3)
        assert np.all(v >= ct.lo[t]) and np.all(v <= ct.hi[t])
        assert np.array_equal(v.min(axis=0), ct.lo[t]) and np.array_equal(v.max(axis=0), ct.hi[t])


def test_single_triangle_tree():
    xyz = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])
    ct = ClusterTree(xyz, np.array([[0, 1, 2]]), 4)
    assert ct.nclusters == 1 and ct.is_leaf(0)
    assert np.array_equal(ct.lo[0], [0, 0, 0]) and np.array_equal(ct.hi[0], [1, 1, 0])


def test_block_partition(st):
    """The leaves of the block tree partition I x I."""
    ct = st.ct
    tot = 0
    cover = np.zeros((st.n, st.n), dtype=np.int32)
    for t, s, _ in st.blocks:
        assert ct.level[t] == ct.level[s]
        cover[np.ix_(ct.indices(t), ct.indices(s))] += 1
        tot += ct.size(t) * ct.size(s)
    for t, s in st.near:
        assert ct.level[t] == ct.level[s]
        cover[np.ix_(ct.indices(t), ct.indices(s))] += 1
        tot += ct.size(t) * ct.size(s)
    assert tot == st.n * st.n
    assert cover.min() == 1 and cover.max() == 1


def test_admissibility_examples():
    # SPEC blocktree examples: [0,1]^3 vs [3,4]^3
    lo_t, hi_t = np.zeros(3), np.ones(3)
    lo_s, hi_s = 3 * np.ones(3), 4 * np.ones(3)
    d = box_dist(lo_t, hi_t, lo_s, hi_s)
    assert abs(d - 2 * math.sqrt(3)) < 1e-15
    diam = math.sqrt(3)
    assert admissible(diam, diam, d, 1.0, 1.0)
    assert not admissible(diam, diam, d, 10.0, 1.0)  # parabolic (3c) fails
    assert not admissible(diam, diam, box_dist(lo_t, hi_t, lo_t, hi_t), 1.0, 1.0)


def test_admissible_blocks_satisfy_eq3(st):
    """Every admissible leaf satisfies (3a), (3b), (3c) with its c_ts."""
    ct = st.ct
    for t, s, c in st.blocks:
        l = ct.level[t]
        dmax = max(ct.diam[t], ct.diam[s])
        dist = box_dist(ct.lo[t], ct.hi[t], ct.lo[s], ct.hi[s])
        assert dmax <= st.eta2 * dist and st.kappa * dmax * dmax <= st.eta2 * dist
        y = ct.mid[t] - ct.mid[s]
        y = y / np.linalg.norm(y)
        cvec = st.dirs[l][c]
        if np.any(cvec != 0):
            assert st.kappa * np.linalg.norm(y - cvec) <= st.eta1 / dmax * (1 + 1e-12)


def test_direction_set_counts():
    # SPEC directions example: kappa=10, d=2, eta1=10 -> m = ceil(2 sqrt 2) = 3, 54 directions
    D, md = direction_set(2.0, 10.0, 10.0)
    assert md == 3 and D.shape == (54, 3)
    assert np.allclose(np.linalg.norm(D, axis=1), 1.0, atol=1e-15)
    D0, md0 = direction_set(0.5, 2.0, 1.0)  # kappa d <= eta1 -> {0}
    assert md0 == 0 and np.array_equal(D0, np.zeros((1, 3)))
    # antipodal: -c is in the set, at the mirrored index order
    Dn = {tuple(v) for v in D}
    assert all(tuple(-v) in Dn for v in D)


def test_direction_coverage_eq12(st):
    """Eq. 12: min_c |y - c| <= eta1/(kappa d_l) for every unit y (10^4 samples per level)."""
    rng = np.random.default_rng(7)
    Y = rng.normal(size=(10000, 3))
    Y /= np.linalg.norm(Y, axis=1)[:, None]
    for l, D in enumerate(st.dirs):
        if st.mdir[l] == 0:
            continue
        dmin = np.min(np.linalg.norm(Y[:, None, :] - D[None, :, :], axis=2), axis=1)
        assert dmin.max() <= st.eta1 / (st.kappa * st.d_level[l])


def test_nearest_direction_brute_force():
    D, _ = direction_set(1.3, 9.0, 1.0)
    rng = np.random.default_rng(3)
    Y = rng.normal(size=(200, 3))
    Y /= np.linalg.norm(Y, axis=1)[:, None]
    idx = nearest_direction(D, Y)
    d = np.linalg.norm(Y[:, None, :] - D[None, :, :], axis=2)
    assert np.allclose(d[np.arange(len(Y)), idx], d.min(axis=1), rtol=0, atol=1e-12)
    # a stored direction maps to itself
    assert np.array_equal(nearest_direction(D, D), np.arange(D.shape[0]))


def test_antipodal_symmetry(st):
    """With the symmetric tie rule (Q4): (t,s,c) in L+  <=>  (s,t,-c) in L+, sd(-c) = -sd(c)."""
    ct = st.ct
    blocks = {(int(t), int(s)): int(c) for t, s, c in st.blocks}
    for (t, s), c in blocks.items():
        l = ct.level[t]
        assert (s, t) in blocks
        c2 = blocks[(s, t)]
        assert np.array_equal(st.dirs[l][c2], -st.dirs[l][c]) or st.mdir[l] == 0
    for l in range(ct.depth):
        if st.mdir[l] == 0 or st.mdir[l + 1] == 0:
            continue
        D = st.dirs[l]
        neg = {tuple(v): i for i, v in enumerate(D)}
        for c in range(0, D.shape[0], 7):
            cn = neg[tuple(-D[c])]
            assert np.array_equal(st.dirs[l + 1][st.sd(l, cn)], -st.dirs[l + 1][st.sd(l, c)])


def test_pair_closure(st):
    """Every non-leaf active pair (t,c) has its children (t', sd(c)) active (Eq. 11 needs them)."""
    ct = st.ct
    for pairs in (st.row_pairs, st.col_pairs):
        for l in range(ct.depth):
            nxt = set(pairs[l + 1])
            for (t, c) in pairs[l]:
                if not ct.is_leaf(t):
                    for ch in ct.children[t]:
                        assert (int(ch), st.sd(l, c)) in nxt
    direct = {(int(t), int(c)) for t, _, c in st.blocks}
    assert all(p in set(st.row_pairs[int(ct.level[p[0]])]) for p in direct)


def test_c1_counts_match_survey():
    """C1 structure counts: 528 admissible, 496 inadmissible blocks, 512 row pairs."""
    s = _structure("C1")
    assert len(s.blocks) == 528 and len(s.near) == 496
    assert sum(len(p) for p in s.row_pairs) == 512
    assert sum(len(p) for p in s.basis_pairs) == 1024
    assert s.ct.depth == 5


def test_kappa0_is_h2():
    """kappa = 0: D_l = {0} on every level, (3c) vacuous -> standard H^2 (SURVEY §8(c) special case)."""
    s = _structure("P0")
    assert all(m == 0 for m in s.mdir)
    assert np.all(s.blocks[:, 2] == 0)
