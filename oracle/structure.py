"""Oracle host structures (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Follows PAPER.md §2:
  * cluster tree (Def. 2.1), binary space partitioning
     read as a median split along the longest axis of the tight
    bounding box;
  * boxes, diam, dist, midpoints;
  * directions D_l (Def. 2.3, Remark 2.4) on the origin-centred
    cube [-1,1]^3 (Q2), square centres (2i+1-m)/m, and the maps sd_l;
  * nearest-direction choice c_ts with the symmetric tie rule Q4;
  * admissibility (Eq. 3b, 3c) and the minimal block tree by
    recursion from the root (Def. 2.5);
  * row(t,c), and the active (t,c) pairs: every (t,c_b) of an
    admissible block plus the closure (t', sd_t(c)) needed by Eq. 11 nesting.

All floating-point decisions are written with an explicit evaluation order
(sums left to right, no library norms) so that any independent implementation
that follows the same formulas reaches identical discrete results.
"""
import math
import numpy as np

TIE_TOL = 1e-12  # Q4: candidates within 1e-12 of the minimal squared distance


def _norm3(v):
    """Euclidean norm, summed left to right: sqrt((v0*v0 + v1*v1) + v2*v2)."""
    return np.sqrt((v[..., 0] * v[..., 0] + v[..., 1] * v[..., 1]) + v[..., 2] * v[..., 2])


class ClusterTree:
    """Binary cluster tree in BFS numbering; cluster t covers perm[begin[t]:end[t]]."""

    def __init__(self, xyz, tri, leaf):
        xyz = np.asarray(xyz, dtype=np.float64)
        tri = np.asarray(tri, dtype=np.int64)
        n = tri.shape[0]
        if n < 1 or leaf < 1:
            raise ValueError("empty mesh or leaf < 1")
        self.n = n
        v0, v1, v2 = xyz[tri[:, 0]], xyz[tri[:, 1]], xyz[tri[:, 2]]
        self.centroid = ((v0 + v1) + v2) / 3.0
        perm = np.arange(n, dtype=np.int64)
        begin, end, level, parent = [0], [n], [0], [-1]
        children = [[-1, -1]]
        lo_l, hi_l = [], []
        t = 0
        while t < len(begin):
            b, e = begin[t], end[t]
            idx = perm[b:e]
            pts = xyz[tri[idx]].reshape(-1, 3)
            lo = pts.min(axis=0)
            hi = pts.max(axis=0)
            lo_l.append(lo)
            hi_l.append(hi)
            cnt = e - b
            if cnt > leaf:
                ext = hi - lo
                axis = int(np.argmax(ext))  # first maximum = lowest axis on ties
                key = self.centroid[idx, axis]
                order = np.lexsort((idx, key))  # by centroid, ties by triangle index
                perm[b:e] = idx[order]
                half = (cnt + 1) // 2
                c0 = len(begin)
                for (cb, ce) in ((b, b + half), (b + half, e)):
                    begin.append(cb)
                    end.append(ce)
                    level.append(level[t] + 1)
                    parent.append(t)
                    children.append([-1, -1])
                children[t] = [c0, c0 + 1]
            t += 1
        self.perm = perm
        self.begin = np.array(begin, dtype=np.int64)
        self.end = np.array(end, dtype=np.int64)
        self.level = np.array(level, dtype=np.int64)
        self.parent = np.array(parent, dtype=np.int64)
        self.children = np.array(children, dtype=np.int64)
        self.lo = np.array(lo_l)
        self.hi = np.array(hi_l)
        self.nclusters = len(begin)
        self.depth = int(self.level.max())
        self.levels = [np.nonzero(self.level == l)[0] for l in range(self.depth + 1)]
        ext = self.hi - self.lo
        self.diam = _norm3(ext)
        self.mid = 0.5 * (self.lo + self.hi)

    def is_leaf(self, t):
        return self.children[t, 0] < 0

    def size(self, t):
        return int(self.end[t] - self.begin[t])

    def indices(self, t):
        """Original triangle indices of cluster t, in cluster order."""
        return self.perm[self.begin[t]:self.end[t]]


def box_dist(lo_t, hi_t, lo_s, hi_s):
    """dist(B_t,B_s) = || (max(0, lo_t-hi_s, lo_s-hi_t))_a ||_2 (vectorised over leading dims)."""
    g = np.maximum(0.0, np.maximum(lo_t - hi_s, lo_s - hi_t))
    return _norm3(g)


def admissible(diam_t, diam_s, dist, kappa, eta2):
    """Eq. (3b) and (3c); (3a) then holds by Eq. (12) and the best-approximation c_ts."""
    dmax = np.maximum(diam_t, diam_s)
    return (dmax <= eta2 * dist) & (kappa * (dmax * dmax) <= eta2 * dist)


def direction_set(d_level, kappa, eta1):
    """Remark 2.4: D_l = {0} if kappa*d_l <= eta1, else 6 m^2 normalised square centres."""
    if kappa * d_level <= eta1:
        return np.zeros((1, 3)), 0
    md = int(math.ceil(((math.sqrt(2.0) * kappa) * d_level) / eta1))
    out = []
    for a in range(3):
        u, w = [ax for ax in range(3) if ax != a]
        for sgn in (-1.0, 1.0):  # faces -x,+x,-y,+y,-z,+z
            for iu in range(md):
                for iv in range(md):
                    p = [0.0, 0.0, 0.0]
                    p[a] = sgn
                    p[u] = float(2 * iu + 1 - md) / md
                    p[w] = float(2 * iv + 1 - md) / md
                    out.append(p)
    D = np.array(out, dtype=np.float64)
    D = D / _norm3(D)[:, None]
    return D, md


_W_RAW = np.array([1.0, math.sqrt(2.0), math.sqrt(3.0)])
TIE_W = _W_RAW / math.sqrt((_W_RAW[0] * _W_RAW[0] + _W_RAW[1] * _W_RAW[1]) + _W_RAW[2] * _W_RAW[2])


def nearest_direction(D, Y):
    """Best approximation of each row of Y in D, with the tie rule of
    SURVEY.md §8(c) Q4: among {c : |y-c|^2 <= min + 1e-12} take the one maximising
    s*<c,w>, s = sign<y,w> (+1 if zero), first index on exact ties."""
    Y = np.atleast_2d(Y)
    out = np.empty(Y.shape[0], dtype=np.int64)
    if D.shape[0] == 1:
        out[:] = 0
        return out
    w = TIE_W
    cw = (D[:, 0] * w[0] + D[:, 1] * w[1]) + D[:, 2] * w[2]
    chunk = max(1, 4_000_000 // D.shape[0])
    for c0 in range(0, Y.shape[0], chunk):
        y = Y[c0:c0 + chunk]
        d0 = y[:, 0:1] - D[None, :, 0]
        d1 = y[:, 1:2] - D[None, :, 1]
        d2 = y[:, 2:3] - D[None, :, 2]
        dist2 = (d0 * d0 + d1 * d1) + d2 * d2
        mn = dist2.min(axis=1, keepdims=True)
        cand = dist2 <= mn + TIE_TOL
        yw = (y[:, 0] * w[0] + y[:, 1] * w[1]) + y[:, 2] * w[2]
        s = np.where(yw >= 0.0, 1.0, -1.0)
        score = np.where(cand, s[:, None] * cw[None, :], -np.inf)
        out[c0:c0 + chunk] = np.argmax(score, axis=1)
    return out


class DH2Structure:
    """Everything of the DH^2 matrix that is discrete: tree, directions, blocks, pairs."""

    def __init__(self, xyz, tri, kappa, m, leaf, eta1, eta2):
        self.xyz = np.asarray(xyz, dtype=np.float64)
        self.tri = np.asarray(tri, dtype=np.int64)
        self.kappa, self.m, self.leaf, self.eta1, self.eta2 = float(kappa), int(m), int(leaf), float(eta1), float(eta2)
        self.k = self.m ** 3
        ct = ClusterTree(self.xyz, self.tri, self.leaf)
        self.ct = ct
        self.n = ct.n
        # Remark 2.4: d_l = max diam on level l
        self.d_level = np.array([ct.diam[ct.levels[l]].max() for l in range(ct.depth + 1)])
        self.dirs, self.mdir = [], []
        for l in range(ct.depth + 1):
            D, md = direction_set(self.d_level[l], self.kappa, self.eta1)
            self.dirs.append(D)
            self.mdir.append(md)
        self._build_blocks()
        self._sd_cache = [dict() for _ in range(ct.depth + 1)]
        self._build_pairs()

    # ---- block tree (Def. 2.5), level-synchronous recursion ----
    def _build_blocks(self):
        ct = self.ct
        adm_t, adm_s, adm_c, near = [], [], [], []
        ft = np.array([0], dtype=np.int64)
        fs = np.array([0], dtype=np.int64)
        lvl = 0
        while ft.size:
            dist = box_dist(ct.lo[ft], ct.hi[ft], ct.lo[fs], ct.hi[fs])
            adm = admissible(ct.diam[ft], ct.diam[fs], dist, self.kappa, self.eta2)
            at, as_ = ft[adm], fs[adm]
            if at.size:
                dv = ct.mid[at] - ct.mid[as_]
                y = dv / _norm3(dv)[:, None]
                c = nearest_direction(self.dirs[lvl], y)
                adm_t.append(at)
                adm_s.append(as_)
                adm_c.append(c)
            rt, rs = ft[~adm], fs[~adm]
            has = (ct.children[rt, 0] >= 0) & (ct.children[rs, 0] >= 0)
            for t, s in zip(rt[~has], rs[~has]):
                near.append((int(t), int(s)))
            rt, rs = rt[has], rs[has]
            nt, ns = [], []
            for i in range(2):
                for j in range(2):
                    nt.append(ct.children[rt, i])
                    ns.append(ct.children[rs, j])
            if rt.size:
                ft = np.concatenate(nt)
                fs = np.concatenate(ns)
                o = np.lexsort((fs, ft))
                ft, fs = ft[o], fs[o]
            else:
                ft = np.zeros(0, dtype=np.int64)
                fs = ft
            lvl += 1
        if adm_t:
            bt, bs, bc = np.concatenate(adm_t), np.concatenate(adm_s), np.concatenate(adm_c)
        else:
            bt = bs = bc = np.zeros(0, dtype=np.int64)
        o = np.lexsort((bs, bt))
        self.blocks = np.stack([bt[o], bs[o], bc[o]], axis=1) if bt.size else np.zeros((0, 3), dtype=np.int64)
        self.near = np.array(sorted(near), dtype=np.int64).reshape(-1, 2)
        self.block_level = ct.level[self.blocks[:, 0]] if len(self.blocks) else np.zeros(0, dtype=np.int64)

    def sd(self, level, c):
        """sd_level(c): nearest direction of D_{level+1} to c, tie rule Q4."""
        cache = self._sd_cache[level]
        v = cache.get(c)
        if v is None:
            v = int(nearest_direction(self.dirs[level + 1], self.dirs[level][c][None, :])[0])
            cache[c] = v
        return v

    def sd_many(self, level, cs):
        cs = np.asarray(cs, dtype=np.int64)
        need = [int(c) for c in np.unique(cs) if int(c) not in self._sd_cache[level]]
        if need:
            res = nearest_direction(self.dirs[level + 1], self.dirs[level][need])
            for c, r in zip(need, res):
                self._sd_cache[level][c] = int(r)
        return np.array([self._sd_cache[level][int(c)] for c in cs], dtype=np.int64)

    # ---- row/col pairs: direct pairs plus closure (t', sd_t(c)) ----
    def _closure(self, direct_cluster, direct_dir):
        ct = self.ct
        pairs = [set() for _ in range(ct.depth + 1)]
        for t, c in zip(direct_cluster, direct_dir):
            pairs[int(ct.level[t])].add((int(t), int(c)))
        for l in range(ct.depth):
            cur = sorted(pairs[l])
            if not cur:
                continue
            ts = np.array([p[0] for p in cur])
            cs = np.array([p[1] for p in cur])
            nl = ct.children[ts, 0] >= 0
            if not nl.any():
                continue
            sds = self.sd_many(l, cs[nl])
            for t, c2 in zip(ts[nl], sds):
                for ch in ct.children[t]:
                    pairs[l + 1].add((int(ch), int(c2)))
        return [sorted(p) for p in pairs]

    def _build_pairs(self):
        b = self.blocks
        self.row_pairs = self._closure(b[:, 0], b[:, 2])
        self.col_pairs = self._closure(b[:, 1], b[:, 2])
        self.basis_pairs = [sorted(set(r) | set(c)) for r, c in zip(self.row_pairs, self.col_pairs)]
        self.row_blocks = {}
        self.col_blocks = {}
        for i, (t, s, c) in enumerate(b):
            self.row_blocks.setdefault((int(t), int(c)), []).append(i)
            self.col_blocks.setdefault((int(s), int(c)), []).append(i)
        for d in (self.row_blocks, self.col_blocks):
            for key in d:
                d[key].sort(key=lambda i: (int(b[i, 0]), int(b[i, 1])))
        levels = [l for l in range(self.ct.depth + 1) if self.basis_pairs[l]]
        self.active_levels = levels

    def row(self, t, c):
        """row(t,c) = {s : (t,s,c) in L+}."""
        return [int(self.blocks[i, 1]) for i in self.row_blocks.get((t, c), [])]

    def parent_map(self, pairs_by_level):
        """(t,c) -> sorted [c+ : (t+,c+) active, sd_{t+}(c+) = c], t+ = parent of t.

        This is sd_{t+}^{-1}({c}) restricted to active pairs (Eq. 15)."""
        ct = self.ct
        out = {}
        for l in range(ct.depth):
            for (tp, cp) in pairs_by_level[l]:
                if ct.children[tp, 0] < 0:
                    continue
                c = self.sd(l, cp)
                for ch in ct.children[tp]:
                    out.setdefault((int(ch), c), []).append(cp)
        for key in out:
            out[key].sort()
        return out
