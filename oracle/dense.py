"""Oracle "O-dense": PAPER.md §3.1 compression applied literally to the densely
expanded far field of the interpolation DH^2 matrix (TEST INFRASTRUCTURE ONLY;
tiny meshes, quadratic cost — "only of theoretical interest").

For every active row pair (t,c):
  anc(t,c) = {(t,c)} u  U_{c+ in sd^{-1}(c)} anc(t+,c+)            (Eq. 15)
  G_tc     = [w_b G_b|_{t x s}]  over (t~,c~) in anc(t,c), s in row(t~,c~)
  leaf:     SVD of G_tc, Q_tc = first k_tc left singular vectors
  non-leaf: SVD of Ghat_tc = diag(Q_{t1c1}^*, Q_{t2c2}^*) G_tc     (Eq. Ghat)
with w_b = 1/||G_b||_F computed from the dense block.  §3.2 must reproduce the same
singular values, ranks and projectors "without changing the result".
"""
import numpy as np

from .recompress import select_rank, svd_left
from .ops import expand_V


class DenseCompression:
    def __init__(self, rc, side="row"):
        self.rc = rc
        self.side = side
        st = rc.st
        self.st = st
        vc = {}
        self.G = {}
        self.omega = {}
        for b in range(len(st.blocks)):
            t, s, c = (int(v) for v in st.blocks[b])
            G = expand_V(rc, t, c, vc) @ rc.S(b) @ expand_V(rc, s, c, vc).conj().T
            if side == "col":
                G = G.conj().T
            self.G[b] = G
            nrm = np.linalg.norm(G)
            self.omega[b] = 1.0 if rc.mode == "FROB_CLUSTERREL" else 1.0 / nrm

    def anc(self, t, c, pmap):
        out = [(t, c)]
        tp = int(self.st.ct.parent[t])
        for cp in pmap.get((t, c), []):
            out += self.anc(tp, cp, pmap)
        return out

    def G_tc(self, t, c, pmap):
        st, ct = self.st, self.st.ct
        blocks_of = st.row_blocks if self.side == "row" else st.col_blocks
        cols = []
        for (ta, ca) in self.anc(t, c, pmap):
            off = ct.begin[t] - ct.begin[ta]
            for b in blocks_of.get((ta, ca), []):
                cols.append(self.omega[b] * self.G[b][off:off + ct.size(t), :])
        if not cols:
            return np.zeros((ct.size(t), 0), dtype=np.complex128)
        return np.hstack(cols)

    def run(self):
        rc, st, ct = self.rc, self.st, self.st.ct
        pairs = st.row_pairs if self.side == "row" else st.col_pairs
        pmap = st.parent_map(pairs)
        self.Q, self.rank, self.sigma = {}, {}, {}
        for l in range(ct.depth, -1, -1):
            for (t, c) in pairs[l]:
                G = self.G_tc(t, c, pmap)
                if ct.is_leaf(t):
                    Gh = G
                else:
                    c2 = st.sd(l, c)
                    parts = []
                    for ch in ct.children[t]:
                        ch = int(ch)
                        off = ct.begin[ch] - ct.begin[t]
                        parts.append(self.Q[(ch, c2)].conj().T @ G[off:off + ct.size(ch), :])
                    Gh = np.vstack(parts)
                U, s = svd_left(Gh)
                kk = select_rank(s, rc.eps, rc.mode)
                Qh = U[:, :kk]
                if ct.is_leaf(t):
                    Q = Qh
                else:
                    c2 = st.sd(l, c)
                    Q = np.zeros((ct.size(t), kk), dtype=np.complex128)
                    r0 = 0
                    for ch in ct.children[t]:
                        ch = int(ch)
                        off = ct.begin[ch] - ct.begin[t]
                        Qc = self.Q[(ch, c2)]
                        Q[off:off + ct.size(ch), :] = Qc @ Qh[r0:r0 + Qc.shape[1], :]
                        r0 += Qc.shape[1]
                self.Q[(t, c)] = Q
                self.rank[(t, c)] = kk
                self.sigma[(t, c)] = s
        return self
