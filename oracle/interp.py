"""Oracle directional interpolation (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

PAPER.md §2:
  * tensor Chebyshev points of the first kind on B_t (Q6),
    xi_{t,a,j} = mid_a + half_a * cos(pi (2j+1)/(2m)), multi-index nu = jx + m jy + m^2 jz;
  * tensor Lagrange polynomials L_{t,nu}, flat axes (Q7): one node at
    mid_a, L_{a,j} = delta_{j0};
  * modified Lagrange L_{tc,nu}(x) = exp(i kappa <x,c>) L_{t,nu}(x);
  * leaf basis v_{tc,i nu} = int phi_i L_{tc,nu} by Radon's 7-point
    degree-5 triangle rule (Q11);
  * transfers e_{t'c,nu' nu} = exp(i kappa <xi_{t',nu'}, c-c'>) L_{t,nu}(xi_{t',nu'}) (Eq. 10,
    PAPER.md:486-497);
  * couplings s_{b,nu mu} = g_c(xi_{t,nu}, xi_{s,mu}).
"""
import math
import numpy as np

FLAT_REL = 1e-12  # Q7: axis is collapsed if hi_a - lo_a <= 1e-12 * diam(B_t)

# Radon's 7-point rule (degree 5) in barycentric coordinates; weights sum to 1.
_S15 = math.sqrt(15.0)
_A = (6.0 - _S15) / 21.0
_B = (6.0 + _S15) / 21.0
_WA = (155.0 - _S15) / 1200.0
_WB = (155.0 + _S15) / 1200.0
QUAD_BARY = np.array([
    [1.0 / 3.0, 1.0 / 3.0, 1.0 / 3.0],
    [_A, _A, 1.0 - 2.0 * _A], [_A, 1.0 - 2.0 * _A, _A], [1.0 - 2.0 * _A, _A, _A],
    [_B, _B, 1.0 - 2.0 * _B], [_B, 1.0 - 2.0 * _B, _B], [1.0 - 2.0 * _B, _B, _B],
])
QUAD_W = np.array([9.0 / 40.0, _WA, _WA, _WA, _WB, _WB, _WB])


def cheb_ref(m):
    """Chebyshev points of the first kind on [-1,1]."""
    j = np.arange(m)
    return np.cos(np.pi * (2 * j + 1) / (2 * m))


def lagrange_1d(z, xhat):
    """L_j(xhat) = prod_{i != j} (xhat - z_i)/(z_j - z_i), returned as (len(xhat), m)."""
    xhat = np.asarray(xhat, dtype=np.float64)
    m = len(z)
    out = np.ones((xhat.size, m))
    for j in range(m):
        for i in range(m):
            if i != j:
                out[:, j] *= (xhat - z[i]) / (z[j] - z[i])
    return out


class Grid:
    """Tensor Chebyshev grid on a box [lo, hi]."""

    def __init__(self, lo, hi, m):
        lo = np.asarray(lo, dtype=np.float64)
        hi = np.asarray(hi, dtype=np.float64)
        self.m = m
        self.mid = 0.5 * (lo + hi)
        self.half = 0.5 * (hi - lo)
        ext = hi - lo
        diam = math.sqrt((ext[0] * ext[0] + ext[1] * ext[1]) + ext[2] * ext[2])
        self.flat = ext <= FLAT_REL * diam
        z = cheb_ref(m)
        self.z = z
        self.nodes = np.empty((3, m))
        for a in range(3):
            self.nodes[a] = self.mid[a] if self.flat[a] else self.mid[a] + self.half[a] * z

    def points(self):
        """xi_nu, nu = jx + m jy + m^2 jz, shape (m^3, 3)."""
        m = self.m
        nu = np.arange(m ** 3)
        jx, jy, jz = nu % m, (nu // m) % m, nu // (m * m)
        return np.stack([self.nodes[0][jx], self.nodes[1][jy], self.nodes[2][jz]], axis=1)

    def axis_lagrange(self, a, x):
        x = np.asarray(x, dtype=np.float64)
        if self.flat[a]:
            out = np.zeros((x.size, self.m))
            out[:, 0] = 1.0
            return out
        return lagrange_1d(self.z, (x - self.mid[a]) / self.half[a])

    def lagrange(self, X):
        """Tensor Lagrange polynomials L_nu(x) at the rows of X: (npts, m^3)."""
        X = np.atleast_2d(X)
        Lx = self.axis_lagrange(0, X[:, 0])
        Ly = self.axis_lagrange(1, X[:, 1])
        Lz = self.axis_lagrange(2, X[:, 2])
        # nu = jx + m jy + m^2 jz  -> index order (jz, jy, jx) when flattened C-style
        L = Lz[:, :, None, None] * Ly[:, None, :, None] * Lx[:, None, None, :]
        return L.reshape(X.shape[0], -1)


def triangle_quadrature(xyz, tri, idx):
    """Quadrature points (len(idx), 7, 3) and weights |tau_i| w_q (len(idx), 7)."""
    v = xyz[tri[idx]]  # (n,3,3)
    pts = np.einsum("qb,nbd->nqd", QUAD_BARY, v)
    e1 = v[:, 1] - v[:, 0]
    e2 = v[:, 2] - v[:, 0]
    cr = np.cross(e1, e2)
    area = 0.5 * np.sqrt((cr[:, 0] * cr[:, 0] + cr[:, 1] * cr[:, 1]) + cr[:, 2] * cr[:, 2])
    return pts, area[:, None] * QUAD_W[None, :]


class Interpolation:
    """V (leaves), E and S of the directional interpolation DH^2 matrix."""

    def __init__(self, st):
        self.st = st
        ct = st.ct
        self.grids = [Grid(ct.lo[t], ct.hi[t], st.m) for t in range(ct.nclusters)]
        self._pts = [None] * ct.nclusters

    def points(self, t):
        if self._pts[t] is None:
            self._pts[t] = self.grids[t].points()
        return self._pts[t]

    def direction(self, level, c):
        return self.st.dirs[level][c]

    def leaf_V(self, t, c):
        """V_tc[i,nu] = sum_q |tau_i| w_q exp(i kappa <x_iq,c>) L_{t,nu}(x_iq)."""
        st = self.st
        idx = st.ct.indices(t)
        pts, w = triangle_quadrature(st.xyz, st.tri, idx)
        cvec = self.direction(int(st.ct.level[t]), c)
        P = pts.reshape(-1, 3)
        phase = np.exp(1j * st.kappa * ((P[:, 0] * cvec[0] + P[:, 1] * cvec[1]) + P[:, 2] * cvec[2]))
        L = self.grids[t].lagrange(P)  # (n*7, k)
        f = (w.reshape(-1) * phase)[:, None] * L
        return f.reshape(len(idx), 7, -1).sum(axis=1)

    def E(self, tchild, c):
        """E_{t'c} for child t' of t and parent direction c in D_t, c' = sd_t(c) (Eq. 10)."""
        st = self.st
        tp = int(st.ct.parent[tchild])
        lp = int(st.ct.level[tp])
        cvec = st.dirs[lp][c]
        c2 = st.sd(lp, c)
        cvec2 = st.dirs[lp + 1][c2]
        dc = cvec - cvec2
        xi = self.points(tchild)  # xi_{t',nu'}
        phase = np.exp(1j * st.kappa * ((xi[:, 0] * dc[0] + xi[:, 1] * dc[1]) + xi[:, 2] * dc[2]))
        return phase[:, None] * self.grids[tp].lagrange(xi)

    def S(self, t, s, c):
        """S_b[nu,mu] = exp(i kappa (r - <xi_t nu - xi_s mu, c>)) / (4 pi r)."""
        st = self.st
        cvec = st.dirs[int(st.ct.level[t])][c]
        xt = self.points(t)
        xs = self.points(s)
        d = xt[:, None, :] - xs[None, :, :]
        r = np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])
        dc = (d[..., 0] * cvec[0] + d[..., 1] * cvec[1]) + d[..., 2] * cvec[2]
        return np.exp(1j * st.kappa * (r - dc)) / (4.0 * np.pi * r)


def kernel_g(x, y, kappa):
    """Helmholtz kernel g(x,y) = exp(i kappa |x-y|)/(4 pi |x-y|) (Eq. 1)."""
    d = np.asarray(x) - np.asarray(y)
    r = np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])
    return np.exp(1j * kappa * r) / (4.0 * np.pi * r)


def kernel_gc(x, y, c, kappa):
    """g_c(x,y) = exp(i kappa (|x-y| - <x-y,c>))/(4 pi |x-y|)."""
    d = np.asarray(x) - np.asarray(y)
    r = np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])
    dc = (d[..., 0] * c[0] + d[..., 1] * c[1]) + d[..., 2] * c[2]
    return np.exp(1j * kappa * (r - dc)) / (4.0 * np.pi * r)
