"""Surface meshes of the paper's experiments (Section 5).

* sphere: the double pyramid P = {x : |x1|+|x2|+|x3| = 1}, each of its eight faces
  regularly refined into q^2 triangles, vertices shifted to the unit sphere
  (PAPER.md:1483-1485).  Vertices are generated as exact dyadic rationals and
  normalised once at the end.
* cube: each face of the unit cube [0,1]^3 (BASELINE.json configs[4]) represented by
  two triangles per grid square of a q x q grid, diagonal
  (i,j)->(i+1,j+1).  Coordinates i/q are exact for q a power of two.

Triangles are outward oriented.  DoF i is triangle i with phi_i = 1 on tau_i
(PAPER.md:1487).  Returns (xyz float64 [nv,3], tri int64 [nt,3]).
"""
import numpy as np


class _VertexPool:
    def __init__(self):
        self.index = {}
        self.coords = []

    def get(self, p):
        key = (float(p[0]), float(p[1]), float(p[2]))
        idx = self.index.get(key)
        if idx is None:
            idx = len(self.coords)
            self.index[key] = idx
            self.coords.append(key)
        return idx


def sphere_mesh(q):
    """Octahedron refined into 8*q^2 triangles, projected to the unit sphere."""
    if q < 1:
        raise ValueError("q must be >= 1")
    pool = _VertexPool()
    tris = []
    for sx in (1.0, -1.0):
        for sy in (1.0, -1.0):
            for sz in (1.0, -1.0):
                A = np.array([sx, 0.0, 0.0])
                B = np.array([0.0, sy, 0.0])
                C = np.array([0.0, 0.0, sz])
                if sx * sy * sz < 0:  # keep (B-A)x(C-A) pointing outwards
                    B, C = C, B

                def P(i, j):
                    return (A * (q - i - j) + B * i + C * j) / q

                for i in range(q):
                    for j in range(q - i):
                        a = pool.get(P(i, j))
                        b = pool.get(P(i + 1, j))
                        c = pool.get(P(i, j + 1))
                        tris.append((a, b, c))
                        if i + j < q - 1:
                            d = pool.get(P(i + 1, j + 1))
                            tris.append((b, d, c))
    xyz = np.array(pool.coords, dtype=np.float64)
    nrm = np.sqrt(xyz[:, 0] * xyz[:, 0] + xyz[:, 1] * xyz[:, 1] + xyz[:, 2] * xyz[:, 2])
    xyz = xyz / nrm[:, None]
    return xyz, np.array(tris, dtype=np.int64)


def cube_mesh(q):
    """Surface of [0,1]^3, each face a q x q grid of squares split into 2 triangles."""
    if q < 1:
        raise ValueError("q must be >= 1")
    pool = _VertexPool()
    tris = []
    for a in range(3):
        u, w = [ax for ax in range(3) if ax != a]
        # e_u x e_w = +e_a for (a=0) and (a=2), -e_a for a=1
        cross_sign = -1.0 if a == 1 else 1.0
        for v in (0.0, 1.0):
            outward = 1.0 if v == 1.0 else -1.0
            flip = cross_sign != outward

            def P(i, j):
                p = [0.0, 0.0, 0.0]
                p[a] = v
                p[u] = i / q
                p[w] = j / q
                return p

            for i in range(q):
                for j in range(q):
                    p00 = pool.get(P(i, j))
                    p10 = pool.get(P(i + 1, j))
                    p11 = pool.get(P(i + 1, j + 1))
                    p01 = pool.get(P(i, j + 1))
                    t1 = (p00, p10, p11)
                    t2 = (p00, p11, p01)
                    if flip:
                        t1 = (t1[0], t1[2], t1[1])
                        t2 = (t2[0], t2[2], t2[1])
                    tris.append(t1)
                    tris.append(t2)
    return np.array(pool.coords, dtype=np.float64), np.array(tris, dtype=np.int64)


def cut_mesh(xyz, tri, every, offset):
    """The mesh without the triangles i with i % every == offset (an open surface whose size is no
    power-of-two multiple: median splits then leave clusters of sizes that straddle the leaf size,
    so one tree level mixes leaf and inner clusters)."""
    keep = np.arange(len(tri)) % every != offset
    return xyz, np.ascontiguousarray(tri[keep])


def mesh_for(cfg):
    """Mesh of a workload configuration (see synth.configs)."""
    if cfg["mesh"] == "sphere_cut":
        return cut_mesh(*sphere_mesh(cfg["q"]), cfg["cut_every"], cfg["cut_offset"])
    if cfg["mesh"] == "sphere":
        return sphere_mesh(cfg["q"])
    if cfg["mesh"] == "cube":
        return cube_mesh(cfg["q"])
    raise ValueError("unknown mesh kind %r" % (cfg["mesh"],))
