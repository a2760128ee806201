"""Pins of the oracle's directional interpolation (§2): textbook identities,
closed forms and brute force."""
import math

import numpy as np
import pytest

from synth import get_config, mesh_for
from oracle.interp import (QUAD_BARY, QUAD_W, Grid, Interpolation, cheb_ref, kernel_g, kernel_gc,
                           lagrange_1d, triangle_quadrature)
from oracle.structure import DH2Structure


def _gl_triangle(f, v, order=12):
    """Independent reference: Gauss-Legendre on the square, Duffy-collapsed onto triangle v."""
    x, w = np.polynomial.legendre.leggauss(order)
    x = 0.5 * (x + 1.0)
    w = 0.5 * w
    U, Wu = np.meshgrid(x, x, indexing="ij")
    WW = np.outer(w, w)
    l1 = U
    l2 = Wu * (1.0 - U)
    jac = (1.0 - U)
    area2 = np.linalg.norm(np.cross(v[1] - v[0], v[2] - v[0]))
    P = (v[0][None, None, :] * (1 - l1 - l2)[..., None] + v[1][None, None, :] * l1[..., None]
         + v[2][None, None, :] * l2[..., None])
    return np.sum(WW * jac * f(P.reshape(-1, 3)).reshape(P.shape[:2])) * area2


def test_chebyshev_points_first_kind():
    z = cheb_ref(4)
    assert np.allclose(z, np.cos(np.pi * np.array([1, 3, 5, 7]) / 8))
    assert np.allclose(cheb_ref(1), [0.0], atol=1e-16)


@pytest.mark.parametrize("m", [1, 2, 3, 4, 5])
def test_lagrange_delta_and_partition_of_unity(m):
    z = cheb_ref(m)
    L = lagrange_1d(z, z)
    assert np.allclose(L, np.eye(m), atol=1e-14)
    x = np.linspace(-1, 1, 17)
    assert np.allclose(lagrange_1d(z, x).sum(axis=1), 1.0, atol=1e-13)


def test_tensor_lagrange_reproduces_polynomials():
    rng = np.random.default_rng(1)
    g = Grid([-0.3, 0.1, 0.2], [0.5, 0.4, 0.9], 4)
    P = g.points()
    assert np.allclose(g.lagrange(P), np.eye(64), atol=1e-13)
    # p of degree < m per axis is reproduced exactly
    coef = rng.normal(size=(4, 4, 4))
    p = lambda X: np.polynomial.polynomial.polyval3d(X[:, 0], X[:, 1], X[:, 2], coef)
    X = rng.uniform([-0.3, 0.1, 0.2], [0.5, 0.4, 0.9], size=(50, 3))
    assert np.allclose(g.lagrange(X) @ p(P), p(X), rtol=1e-12, atol=1e-12)


def test_directional_interpolant_reproduces_plane_wave_times_polynomial():
    """I_tc[f] = sum_nu f(xi_nu) exp(-i k <xi_nu,c>) L_tc,nu reproduces f = exp(i k <x,c>) p(x)
    exactly for p of degree < m per axis (BASELINE north_star pin)."""
    rng = np.random.default_rng(2)
    kappa = 17.0
    c = np.array([0.3, -0.5, 0.8])
    c /= np.linalg.norm(c)
    g = Grid([0.1, 0.2, -0.4], [0.6, 0.3, 0.1], 3)
    coef = rng.normal(size=(3, 3, 3)) + 1j * rng.normal(size=(3, 3, 3))
    f = lambda X: np.exp(1j * kappa * X @ c) * np.polynomial.polynomial.polyval3d(X[:, 0], X[:, 1], X[:, 2], coef)
    P = g.points()
    X = rng.uniform([0.1, 0.2, -0.4], [0.6, 0.3, 0.1], size=(40, 3))
    Ltc = np.exp(1j * kappa * X @ c)[:, None] * g.lagrange(X)  # modified Lagrange
    approx = Ltc @ (f(P) * np.exp(-1j * kappa * P @ c))
    assert np.allclose(approx, f(X), rtol=1e-12, atol=1e-12)


def test_flat_axis_collapse():
    g = Grid([0.0, 0.0, 0.5], [1.0, 2.0, 0.5], 3)
    assert list(g.flat) == [False, False, True]
    X = np.array([[0.3, 0.7, 0.5], [0.9, 0.1, 0.5]])
    L = g.lagrange(X).reshape(2, 3, 3, 3)  # (pt, jz, jy, jx)
    assert np.all(L[:, 1:, :, :] == 0)
    assert np.allclose(L[:, 0].sum(axis=(1, 2)), 1.0)


def test_radon_rule_exact_degree5():
    """sum_q w_q lam1^a lam2^b lam3^c = 2 a! b! c! / (a+b+c+2)! for a+b+c <= 5 (w normalised)."""
    for a in range(6):
        for b in range(6 - a):
            for c in range(6 - a - b):
                val = np.sum(QUAD_W * QUAD_BARY[:, 0] ** a * QUAD_BARY[:, 1] ** b * QUAD_BARY[:, 2] ** c)
                exact = 2.0 * math.factorial(a) * math.factorial(b) * math.factorial(c) / math.factorial(a + b + c + 2)
                assert abs(val - exact) <= 1e-15
    assert abs(QUAD_W.sum() - 1.0) <= 1e-15


@pytest.fixture(scope="module")
def p1():
    cfg = get_config("P1")
    xyz, tri = mesh_for(cfg)
    st = DH2Structure(xyz, tri, cfg["kappa"], cfg["m"], cfg["leaf"], cfg["eta1"], cfg["eta2"])
    return st, Interpolation(st)


def test_leaf_V_closed_forms(p1):
    st, ip = p1
    t = int(st.ct.levels[st.ct.depth][0])
    idx = st.ct.indices(t)
    # m = 1, c = 0: V = area (SPEC interpolation example)
    st1 = DH2Structure(st.xyz, st.tri, 0.0, 1, st.leaf, 1.0, 10.0)
    ip1 = Interpolation(st1)
    t1 = int(st1.ct.levels[st1.ct.depth][0])
    v = st1.xyz[st1.tri[st1.ct.indices(t1)]]
    area = 0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1)
    assert np.allclose(ip1.leaf_V(t1, 0)[:, 0], area, rtol=1e-14)
    # kappa = 0 -> real; c = 0, m <= 2: degree <= 3 integrand, against an independent Gauss-Duffy rule
    st2 = DH2Structure(st.xyz, st.tri, 0.0, 2, st.leaf, 1.0, 10.0)
    ip2 = Interpolation(st2)
    t2 = int(st2.ct.levels[st2.ct.depth][0])
    V2 = ip2.leaf_V(t2, 0)
    assert np.all(V2.imag == 0)
    g2 = ip2.grids[t2]
    for r, i in enumerate(st2.ct.indices(t2)[:4]):
        verts = st2.xyz[st2.tri[i]]
        for nu in range(8):
            ref = _gl_triangle(lambda X: g2.lagrange(X)[:, nu], verts)
            assert abs(V2[r, nu] - ref) <= 1e-14 * max(1.0, abs(ref)) + 1e-17


def test_leaf_V_plane_wave_times_polynomial(p1):
    """V_tc a_p = quadrature of exp(i k <x,c>) p(x) with a_p = p(xi_nu), p of degree < m per axis."""
    st, ip = p1
    rng = np.random.default_rng(5)
    l = st.ct.depth
    t, c = st.row_pairs[l][3]
    g = ip.grids[t]
    coef = rng.normal(size=(3, 3, 3))
    p = lambda X: np.polynomial.polynomial.polyval3d(X[:, 0], X[:, 1], X[:, 2], coef)
    V = ip.leaf_V(t, c)
    cvec = st.dirs[l][c]
    pts, w = triangle_quadrature(st.xyz, st.tri, st.ct.indices(t))
    ref = np.sum(w * np.exp(1j * st.kappa * pts @ cvec) * p(pts.reshape(-1, 3)).reshape(w.shape), axis=1)
    assert np.allclose(V @ p(g.points()), ref, rtol=1e-12, atol=1e-15)


def test_transfer_identities(p1):
    st, ip = p1
    ct = st.ct
    # identity when c = c' and B_t' = B_t: use the Grid machinery directly
    g = Grid([0, 0, 0], [1, 1, 1], 3)
    assert np.allclose(g.lagrange(g.points()), np.eye(27), atol=1e-14)
    # kappa = 0: real, rows sum to 1 (partition of unity)
    st0 = DH2Structure(st.xyz, st.tri, 0.0, 3, st.leaf, 1.0, 10.0)
    ip0 = Interpolation(st0)
    tch = int(st0.ct.children[st0.ct.levels[2][0], 0])
    E0 = ip0.E(tch, 0)
    assert np.all(np.abs(E0.imag) == 0) and np.allclose(E0.sum(axis=1), 1.0, atol=1e-13)
    # Kronecker structure E = Ez (x) Ey (x) Ex with nu = jx + m jy + m^2 jz
    l = ct.depth - 1
    tp, c = [p for p in st.row_pairs[l] if not ct.is_leaf(p[0])][0]
    ch = int(ct.children[tp, 0])
    E = ip.E(ch, c)
    m = st.m
    E4 = E.reshape(m, m, m, m, m, m)  # (jz',jy',jx', jz,jy,jx)
    ex = E4[0, 0, :, 0, 0, :] / E4[0, 0, 0, 0, 0, 0]
    ey = E4[0, :, 0, 0, :, 0] / E4[0, 0, 0, 0, 0, 0]
    ez = E4[:, 0, 0, :, 0, 0]
    K = np.kron(ez, np.kron(ey, ex))
    assert np.allclose(K, E, rtol=1e-12, atol=1e-14 * np.abs(E).max())


def test_nestedness_exact_when_same_direction(p1):
    """For c' = c the re-interpolation is exact: V_tc|_{t'} computed with the parent's Lagrange
    polynomials equals V_{t'c} E_{t'c} (polynomial reproduction, Eq. 10 with c = c')."""
    st, ip = p1
    ct = st.ct
    l = ct.depth - 1
    tp = int(ct.levels[l][0])
    ch = int(ct.children[tp, 0])
    c = 5
    # evaluate the child-side formula with c' := c (zero phase factor), i.e. E = L_t(xi_t')
    E = ip.grids[tp].lagrange(ip.points(ch))
    cvec = st.dirs[l][c]
    st_c = st.dirs[l + 1]
    # child basis with the SAME direction vector c (not in D_{l+1} in general): build by hand
    pts, w = triangle_quadrature(st.xyz, st.tri, ct.indices(ch))
    P = pts.reshape(-1, 3)
    phase = np.exp(1j * st.kappa * P @ cvec)
    Vch = ((w.reshape(-1) * phase)[:, None] * ip.grids[ch].lagrange(P)).reshape(len(w), 7, -1).sum(1)
    Vpar = ((w.reshape(-1) * phase)[:, None] * ip.grids[tp].lagrange(P)).reshape(len(w), 7, -1).sum(1)
    assert np.allclose(Vch @ E, Vpar, rtol=1e-12, atol=1e-13 * np.abs(Vpar).max())
    del st_c


def test_coupling_closed_forms(p1):
    st, ip = p1
    t, s, c = (int(v) for v in st.blocks[10])
    S = ip.S(t, s, c)
    xt, xs = ip.points(t), ip.points(s)
    r = np.linalg.norm(xt[:, None, :] - xs[None, :, :], axis=2)
    assert np.allclose(np.abs(S), 1.0 / (4 * np.pi * r), rtol=1e-14)
    # S_(s,t,-c) = S_(t,s,c)^T
    l = int(st.ct.level[t])
    D = st.dirs[l]
    cn = int(np.nonzero(np.all(D == -D[c], axis=1))[0][0])
    assert np.allclose(ip.S(s, t, cn), S.T, rtol=1e-13, atol=0)
    # entries equal g_c at the grid points; g = exp(i k <x-y,c>) g_c
    cvec = D[c]
    assert np.allclose(S, kernel_gc(xt[:, None, :], xs[None, :, :], cvec, st.kappa), rtol=1e-14)
    d = xt[:, None, :] - xs[None, :, :]
    assert np.allclose(np.exp(1j * st.kappa * d @ cvec) * S, kernel_g(xt[:, None, :], xs[None, :, :], st.kappa),
                       rtol=1e-12)


def test_interpolation_error_decays_in_m():
    """V S V^* vs the brute-force 7x7-point product rule applied to g itself on an admissible
    block: pure interpolation error, decreasing in m.  Magnitude: parity
    unpinned (the paper gives no constant)."""
    cfg = get_config("P1")
    xyz, tri = mesh_for(cfg)
    errs = []
    for m in (2, 3, 4, 5):
        st = DH2Structure(xyz, tri, cfg["kappa"], m, cfg["leaf"], cfg["eta1"], cfg["eta2"])
        ip = Interpolation(st)
        ct = st.ct
        b = [i for i in range(len(st.blocks)) if ct.is_leaf(int(st.blocks[i, 0]))][0]
        t, s, c = (int(v) for v in st.blocks[b])
        G = ip.leaf_V(t, c) @ ip.S(t, s, c) @ ip.leaf_V(s, c).conj().T
        pt, wt = triangle_quadrature(xyz, tri, ct.indices(t))
        ps, ws = triangle_quadrature(xyz, tri, ct.indices(s))
        K = kernel_g(pt[:, :, None, None, :], ps[None, None, :, :, :], st.kappa)
        D = np.einsum("iq,iqjr,jr->ij", wt, K, ws)
        errs.append(np.linalg.norm(G - D) / np.linalg.norm(D))
    print("interp errors m=2..5", errs)
    assert all(errs[i + 1] < errs[i] for i in range(len(errs) - 1)), errs
    assert errs[-1] < 0.01 * errs[0], errs  # exponential-type decay
