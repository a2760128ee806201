"""Pins of the nearfield oracle (oracle/nearfield.py; NEXT-4).

* every Sauter-Schwab transformation integrates polynomials in (u, v) exactly (a wrong region
  map, a missing region or a wrong Jacobian power fails this);
* at kappa = 0 the entries converge, as n_q grows, to the Laplace Galerkin integral whose inner
  integral is the closed-form potential of a flat triangle (Wilton et al.'s edge formula) and
  whose outer integral is adaptive (QUADPACK): identical, edge- and vertex-adjacent and regular
  coplanar pairs;
* at kappa > 0 the Sauter-Schwab values converge with n_q (the Helmholtz remainder is bounded).
"""
import numpy as np
import pytest
from scipy import integrate

from oracle import nearfield as nf


def laplace_potential(P, x):
    """int_tau 1/|x-y| dy for x in the plane of the flat triangle P (edge formula, in-plane)."""
    n = np.cross(P[1] - P[0], P[2] - P[0])
    n /= np.linalg.norm(n)
    tot = 0.0
    for a in range(3):
        p, q = P[a], P[(a + 1) % 3]
        s = (q - p) / np.linalg.norm(q - p)
        d = np.dot(p - x, np.cross(s, n))
        if abs(d) < 1e-14:
            continue
        tot += d * (np.arcsinh(np.dot(q - x, s) / abs(d)) - np.arcsinh(np.dot(p - x, s) / abs(d)))
    return tot


def laplace_reference(Pi, Pj):
    A = nf.area(Pi)

    def f(u2, u1):
        return laplace_potential(Pj, Pi[0] + u1 * (Pi[1] - Pi[0]) + u2 * (Pi[2] - Pi[1]))

    v, _ = integrate.dblquad(f, 0, 1, 0, lambda u1: u1, epsabs=1e-13, epsrel=1e-10)
    return 2 * A * v / (4 * np.pi)


XYZ = np.array([[0.0, 0, 0], [1.0, 0.1, 0], [0.3, 0.9, 0], [1.2, 1.1, 0], [-0.8, 0.2, 0], [-0.5, -0.7, 0],
                [3.0, 0.5, 0], [4.0, 0.6, 0], [3.3, 1.4, 0]])


@pytest.mark.parametrize("case", ["identical", "edge", "vertex"])
def test_transformations_exact_on_polynomials(case):
    u1, u2, w = nf.duffy_rule(8)
    U1, V1 = np.meshgrid(u1, u1, indexing="ij")
    U2, V2 = np.meshgrid(u2, u2, indexing="ij")
    W = np.outer(w, w)
    polys = [lambda a, b, c, d: 1.0 + 0 * a, lambda a, b, c, d: a * d,
             lambda a, b, c, d: a ** 2 * b + c * d ** 2 - a * b * c * d,
             lambda a, b, c, d: (a - c) ** 2 + (b - d) ** 2 + 3 * b * c]
    for f in polys:
        exact = np.sum(W * f(U1, U2, V1, V2))
        assert abs(nf.singular_reference(case, f, 5) - exact) <= 1e-14
    assert abs(nf.singular_reference(case, polys[0], 5) - 0.25) <= 1e-15  # |T|^2


@pytest.mark.parametrize("ti,tj,case", [((0, 1, 2), (0, 1, 2), "identical"), ((0, 1, 2), (1, 3, 2), "edge"),
                                        ((0, 1, 2), (2, 4, 0), "edge"), ((0, 1, 2), (0, 4, 5), "vertex"),
                                        ((0, 1, 2), (6, 7, 8), "regular")])
def test_laplace_against_closed_form_potential(ti, tj, case):
    ti, tj = np.array(ti), np.array(tj)
    assert nf.classify(ti, tj)[0] == case
    ref = laplace_reference(XYZ[ti], XYZ[tj])
    err = lambda **kw: abs(nf.entry(XYZ[ti], XYZ[tj], ti, tj, 0.0, **kw) - ref) / abs(ref)
    if case == "regular":
        assert err(nq_reg=3) < 1e-5 and err(nq_reg=6) < 1e-10
    else:
        e3, e5, e8 = err(nq_sing=3), err(nq_sing=5), err(nq_sing=8)
        assert e5 < 1e-5 and e8 < 1e-8 and e8 < e5 < e3, (e3, e5, e8)


def test_classify_orders_put_shared_vertices_first():
    assert nf.classify((4, 7, 9), (9, 4, 7)) == ("identical", (0, 1, 2), (1, 2, 0))
    case, oi, oj = nf.classify((4, 7, 9), (9, 2, 7))
    assert case == "edge" and [(4, 7, 9)[a] for a in oi[:2]] == [(9, 2, 7)[b] for b in oj[:2]] == [7, 9]
    case, oi, oj = nf.classify((4, 7, 9), (1, 2, 7))
    assert case == "vertex" and (4, 7, 9)[oi[0]] == (1, 2, 7)[oj[0]] == 7
    assert nf.classify((1, 2, 3), (4, 5, 6))[0] == "regular"


def test_helmholtz_converges_with_order():
    kappa = 6.0
    P = XYZ * 0.15
    for ti, tj in [((0, 1, 2), (0, 1, 2)), ((0, 1, 2), (1, 3, 2)), ((0, 1, 2), (0, 4, 5))]:
        v5 = nf.entry(P[list(ti)], P[list(tj)], ti, tj, kappa, nq_sing=5)
        v10 = nf.entry(P[list(ti)], P[list(tj)], ti, tj, kappa, nq_sing=10)
        assert abs(v5 - v10) / abs(v10) < 1e-5
        # the Laplace part dominates; the difference is the smooth remainder, O(kappa |tau|^2)
        l10 = nf.entry(P[list(ti)], P[list(tj)], ti, tj, 0.0, nq_sing=10)
        assert abs(v10 - l10) < kappa * 4 * nf.area(P[list(ti)]) * nf.area(P[list(tj)]) / (4 * np.pi)


def test_near_block_matches_entrywise():
    from synth import get_config, mesh_for
    from oracle.structure import DH2Structure
    cfg = get_config("C1")
    xyz, tri = mesh_for(cfg)
    st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    t, s = st.near[0]
    ct = st.ct
    rows = ct.perm[ct.begin[t]: ct.begin[t] + ct.size(t)]
    cols = ct.perm[ct.begin[s]: ct.begin[s] + ct.size(s)]
    B = nf.near_block(xyz, tri, rows, cols, cfg["kappa"])
    for a in (0, 3, len(rows) - 1):
        for b in (0, 5, len(cols) - 1):
            i, j = rows[a], cols[b]
            assert abs(B[a, b] - nf.entry(xyz[tri[i]], xyz[tri[j]], tri[i], tri[j], cfg["kappa"])) <= 1e-15 * abs(B).max()


def test_near_and_far_blocks_partition_the_matrix():
    """L+ and L- tile I x I exactly once (Def. 2.5), so G = G_far + N has every entry once;
    every touching pair of triangles lies in L- (the boxes of touching triangles intersect)."""
    from synth import get_config, mesh_for
    from oracle.structure import DH2Structure
    for name in ("P1", "P3"):
        cfg = get_config(name)
        xyz, tri = mesh_for(cfg)
        st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
        ct, n = st.ct, len(tri)
        cover = np.zeros((n, n), dtype=np.int32)
        rng = lambda t: ct.perm[ct.begin[t]: ct.begin[t] + ct.size(t)]  # noqa: E731
        for t, s, _c in st.blocks:
            cover[np.ix_(rng(int(t)), rng(int(s)))] += 1
        near = np.zeros((n, n), dtype=bool)
        for t, s in st.near:
            cover[np.ix_(rng(int(t)), rng(int(s)))] += 1
            near[np.ix_(rng(int(t)), rng(int(s)))] = True
        assert (cover == 1).all()
        touch = (tri[:, None, :, None] == tri[None, :, None, :]).any(axis=(2, 3))
        assert near[touch].all()
