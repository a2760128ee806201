"""Oracle nearfield: Galerkin entries of the inadmissible leaves (TEST INFRASTRUCTURE ONLY — see
oracle/__init__.py; the product path never imports this module).

PAPER.md:1486-1492 (Section 5): "For constructing the Galerkin stiffness matrix G we use piecewise
constant basis functions and Sauter-Erichsen-Schwab quadrature of order n_q = 5 for triangles that
share a vertex, an edge, or are identical, and otherwise Gauss quadrature with Duffy transformation
of order n_q = 3."  The entry is (D2)

    g_ij = int_{tau_i} int_{tau_j} g(x, y) dy dx,   g(x, y) = exp(i kappa |x-y|) / (4 pi |x-y|),

written over the reference triangle T = {(u1, u2) : 0 <= u2 <= u1 <= 1} (area 1/2) with the affine
map chi(u) = P0 + u1 (P1 - P0) + u2 (P2 - P1), Jacobian 2 |tau|:

    g_ij = (2|tau_i|) (2|tau_j|) int_T int_T g(chi_i(u), chi_j(v)) dv du.

* regular pairs (no common vertex): the Duffy map (s, t) -> (s, s t), Jacobian s, of the unit
  square onto T, n_q Gauss-Legendre points per axis: n_q^2 points per triangle, n_q^4 per pair;
* touching pairs: Sauter-Schwab's relative-coordinate transformations (SASC11, Ch. 5.2) of
  T x T onto [0,1]^4 with (xi, eta1, eta2, eta3), Gauss-Legendre n_q per axis, one integrand per
  sub-region (identical: 6 regions, weight xi^3 eta1^2 eta2; common edge: 5 regions, weights
  xi^3 eta1^2 (first) and xi^3 eta1^2 eta2; common vertex: 2 regions, weight xi^3 eta2).  The
  shared vertices are placed first: common edge P0 P1 in both triangles (the edge is u2 = 0),
  common vertex P0 (u = 0).  Each region's factor xi^3 cancels the 1/|x-y| singularity.

The transformation tables are the textbook ones restated (no code copied); tests pin them by
exactness on polynomials and against the analytic Laplace potential of a flat triangle.
"""
import numpy as np

FOUR_PI = 4.0 * np.pi


def gauss01(n):
    """n-point Gauss-Legendre rule on [0, 1]."""
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def kernel(x, y, kappa):
    """g(x, y) = exp(i kappa r)/(4 pi r) for point arrays (..., 3)."""
    d = x - y
    r = np.sqrt(d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1] + d[..., 2] * d[..., 2])
    return np.exp(1j * kappa * r) / (FOUR_PI * r)


def chi(P, u1, u2):
    """chi(u) = P0 + u1 (P1 - P0) + u2 (P2 - P1) for arrays u1, u2 -> (..., 3)."""
    P0, P1, P2 = P
    return P0 + u1[..., None] * (P1 - P0) + u2[..., None] * (P2 - P1)


def area(P):
    return 0.5 * np.linalg.norm(np.cross(P[1] - P[0], P[2] - P[0]))


def duffy_rule(nq):
    """Points (u1, u2) and weights of the Duffy-Gauss rule on T (weights sum to 1/2)."""
    g, w = gauss01(nq)
    s, t = np.meshgrid(g, g, indexing="ij")
    W = np.outer(w, w) * s
    return s.ravel(), (s * t).ravel(), W.ravel()


def regions(case, xi, e1, e2, e3):
    """Sauter-Schwab sub-regions: list of (weight, (u1, u2), (v1, v2)) on [0,1]^4."""
    if case == "identical":
        w = xi ** 3 * e1 ** 2 * e2
        return [
            (w, (xi, xi * (1 - e1 + e1 * e2)), (xi * (1 - e1 * e2 * e3), xi * (1 - e1))),
            (w, (xi * (1 - e1 * e2 * e3), xi * (1 - e1)), (xi, xi * (1 - e1 + e1 * e2))),
            (w, (xi, xi * e1 * (1 - e2 + e2 * e3)), (xi * (1 - e1 * e2), xi * e1 * (1 - e2))),
            (w, (xi * (1 - e1 * e2), xi * e1 * (1 - e2)), (xi, xi * e1 * (1 - e2 + e2 * e3))),
            (w, (xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), (xi, xi * e1 * (1 - e2))),
            (w, (xi, xi * e1 * (1 - e2)), (xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3))),
        ]
    if case == "edge":
        w1 = xi ** 3 * e1 ** 2
        w = xi ** 3 * e1 ** 2 * e2
        return [
            (w1, (xi, xi * e1 * e3), (xi * (1 - e1 * e2), xi * e1 * (1 - e2))),
            (w, (xi, xi * e1), (xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3))),
            (w, (xi * (1 - e1 * e2), xi * e1 * (1 - e2)), (xi, xi * e1 * e2 * e3)),
            (w, (xi * (1 - e1 * e2 * e3), xi * e1 * e2 * (1 - e3)), (xi, xi * e1)),
            (w, (xi * (1 - e1 * e2 * e3), xi * e1 * (1 - e2 * e3)), (xi, xi * e1 * e2)),
        ]
    if case == "vertex":
        w = xi ** 3 * e2
        return [
            (w, (xi, xi * e1), (xi * e2, xi * e2 * e3)),
            (w, (xi * e2, xi * e2 * e3), (xi, xi * e1)),
        ]
    raise ValueError(case)


def classify(ti, tj):
    """Case of the pair of vertex-index triples and the vertex orders that put the shared vertices
    first: returns (case, order_i, order_j) with order_* permutations of (0, 1, 2)."""
    ti = [int(a) for a in ti]
    tj = [int(a) for a in tj]
    common = [a for a in ti if a in tj]
    if len(common) == 3:
        return "identical", (0, 1, 2), tuple(tj.index(a) for a in ti)
    if len(common) == 2:
        a, b = common
        ci = [ti.index(a), ti.index(b)]
        cj = [tj.index(a), tj.index(b)]
        oi = tuple(ci + [3 - sum(ci)])
        oj = tuple(cj + [3 - sum(cj)])
        return "edge", oi, oj
    if len(common) == 1:
        a = common[0]
        ia, ja = ti.index(a), tj.index(a)
        return "vertex", (ia, (ia + 1) % 3, (ia + 2) % 3), (ja, (ja + 1) % 3, (ja + 2) % 3)
    return "regular", (0, 1, 2), (0, 1, 2)


def singular_reference(case, f, nq):
    """int_T int_T f(u1, u2, v1, v2) by the Sauter-Schwab regions of `case`, n_q points per axis."""
    g, w = gauss01(nq)
    XI, E1, E2, E3 = np.meshgrid(g, g, g, g, indexing="ij")
    W = np.einsum("i,j,k,l->ijkl", w, w, w, w)
    tot = 0.0
    for wt, u, v in regions(case, XI, E1, E2, E3):
        tot = tot + np.sum(W * wt * f(u[0], u[1], v[0], v[1]))
    return tot


def entry(Pi, Pj, ti, tj, kappa, nq_sing=5, nq_reg=3):
    """One Galerkin entry g_ij (Pi, Pj: 3x3 vertex coordinates; ti, tj: vertex indices)."""
    case, oi, oj = classify(ti, tj)
    Pi = np.asarray(Pi, dtype=np.float64)[list(oi)]
    Pj = np.asarray(Pj, dtype=np.float64)[list(oj)]
    jac = 4.0 * area(Pi) * area(Pj)
    if case == "regular":
        u1, u2, wu = duffy_rule(nq_reg)
        x = chi(Pi, u1, u2)
        y = chi(Pj, u1, u2)
        G = kernel(x[:, None, :], y[None, :, :], kappa)
        return jac * np.sum(wu[:, None] * wu[None, :] * G)

    def f(u1, u2, v1, v2):
        return kernel(chi(Pi, u1, u2), chi(Pj, v1, v2), kappa)

    return jac * singular_reference(case, f, nq_sing)


def regular_block(xyz, tri, rows, cols, kappa, nq_reg=3):
    """Duffy-Gauss values for all (i in rows, j in cols) at once (vectorised; the touching pairs
    among them are replaced by entry() in near_block)."""
    u1, u2, wu = duffy_rule(nq_reg)
    def pts(idx):
        P = xyz[tri[idx]]  # (n, 3, 3)
        X = P[:, None, 0, :] + u1[None, :, None] * (P[:, None, 1, :] - P[:, None, 0, :]) + \
            u2[None, :, None] * (P[:, None, 2, :] - P[:, None, 1, :])
        A = 0.5 * np.linalg.norm(np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]), axis=1)
        return X, 2.0 * A
    X, ai = pts(rows)
    Y, aj = pts(cols)
    with np.errstate(divide="ignore", invalid="ignore"):  # (coincident points of identical pairs)
        G = kernel(X[:, None, :, None, :], Y[None, :, None, :, :], kappa)  # (i, j, p, q)
    return ai[:, None] * aj[None, :] * np.einsum("ijpq,p,q->ij", G, wu, wu)


def near_block(xyz, tri, rows, cols, kappa, nq_sing=5, nq_reg=3):
    """Dense nearfield block G|_{rows x cols} (rows/cols: triangle indices)."""
    B = regular_block(xyz, tri, rows, cols, kappa, nq_reg)
    vi = tri[rows]
    vj = tri[cols]
    touch = (vi[:, :, None, None] == vj[None, None, :, :]).any(axis=(1, 3))
    for a, b in zip(*np.nonzero(touch)):
        i, j = int(rows[a]), int(cols[b])
        B[a, b] = entry(xyz[tri[i]], xyz[tri[j]], tri[i], tri[j], kappa, nq_sing, nq_reg)
    return B


def nearfield_blocks(st, xyz, tri, kappa, nq_sing=5, nq_reg=3):
    """All inadmissible leaves (st.near, sorted (t, s)), rows/cols in cluster order
    (perm[begin_t : begin_t + #t])."""
    ct = st.ct
    out = []
    for t, s in st.near:
        rows = ct.perm[ct.begin[t]: ct.begin[t] + ct.size(t)]
        cols = ct.perm[ct.begin[s]: ct.begin[s] + ct.size(s)]
        out.append(near_block(xyz, tri, np.asarray(rows), np.asarray(cols), kappa, nq_sing, nq_reg))
    return out


def near_matvec(st, blocks, x):
    """y = N x in original triangle order (N = the nearfield blocks)."""
    ct = st.ct
    y = np.zeros(len(x), dtype=np.complex128)
    for (t, s), B in zip(st.near, blocks):
        rows = ct.perm[ct.begin[t]: ct.begin[t] + ct.size(t)]
        cols = ct.perm[ct.begin[s]: ct.begin[s] + ct.size(s)]
        y[rows] += B @ x[cols]
    return y
