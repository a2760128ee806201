"""Oracle "O-lazy": the same §3.2 recompression as oracle/recompress.py (TEST INFRASTRUCTURE
ONLY), evaluated on demand with memoisation, so that single pairs of a configuration too large
for the eager oracle (C3) can be computed one by one together with their dependency cone:

  R_tc      (Eq. 18)       needs the basis weights of the subtree of (t,c)
  w_b                      needs R_tc and R_sc of the block
  Zhat_tc   needs R of the blocks of row(t,c) and Zhat of the parents (t+,c+)
  truncation needs Zhat_tc and, above the leaves, the C of the children

Every formula is the one of recompress.py (same helpers qr_r, svd_left, select_rank); only
the evaluation order differs (the paper's level loops are a schedule, not a definition).
"""
import numpy as np

from .interp import Interpolation
from .recompress import qr_r, select_rank, svd_left


class LazyRecompression:
    def __init__(self, st, eps, mode="FROB_BLOCKREL", interp=None):
        self.st = st
        self.eps = float(eps)
        self.mode = mode
        self.k = st.k
        self.ip = interp if interp is not None else Interpolation(st)
        self._R, self._w, self._Z, self._T = {}, {}, {}, {}
        self._V, self._E, self._S = {}, {}, {}
        self._pmap = {}
        self.block_index = {(int(t), int(s)): i for i, (t, s, c) in enumerate(st.blocks)}

    # interpolation quantities
    def V(self, t, c):
        if (t, c) not in self._V:
            self._V[(t, c)] = self.ip.leaf_V(t, c)
        return self._V[(t, c)]

    def E(self, tchild, c):
        if (tchild, c) not in self._E:
            self._E[(tchild, c)] = self.ip.E(tchild, c)
        return self._E[(tchild, c)]

    def S(self, b):
        if b not in self._S:
            t, s, c = (int(v) for v in self.st.blocks[b])
            self._S[b] = self.ip.S(t, s, c)
        return self._S[b]

    # basis weights (Eq. 18)
    def R(self, t, c):
        key = (t, c)
        if key not in self._R:
            st, ct, k = self.st, self.st.ct, self.k
            if ct.is_leaf(t):
                V = self.V(t, c)
                self._R[key] = V if V.shape[0] <= k else qr_r(V, k)
            else:
                c2 = st.sd(int(ct.level[t]), c)
                X = np.vstack([self.R(int(ch), c2) @ self.E(int(ch), c) for ch in ct.children[t]])
                self._R[key] = qr_r(X, k)
        return self._R[key]

    def omega(self, b):
        if b not in self._w:
            t, s, c = (int(v) for v in self.st.blocks[b])
            n = np.linalg.norm(self.R(t, c) @ self.S(b) @ self.R(s, c).conj().T)
            self._w[b] = 1.0 if self.mode == "FROB_CLUSTERREL" else 1.0 / n
        return self._w[b]

    def parent_map(self, side):
        if side not in self._pmap:
            self._pmap[side] = self.st.parent_map(self.st.row_pairs if side == "row" else self.st.col_pairs)
        return self._pmap[side]

    # total weights
    def Zhat(self, side, t, c):
        key = (side, t, c)
        if key not in self._Z:
            st, ct, k = self.st, self.st.ct, self.k
            blocks_of = st.row_blocks if side == "row" else st.col_blocks
            rows = []
            for b in blocks_of.get((t, c), []):
                bt, bs, _ = (int(v) for v in st.blocks[b])
                if side == "row":
                    rows.append(self.omega(b) * (self.R(bs, c) @ self.S(b).conj().T))
                else:
                    rows.append(self.omega(b) * (self.R(bt, c) @ self.S(b)))
            tp = int(ct.parent[t])
            for cp in self.parent_map(side).get((t, c), []):
                rows.append(self.Zhat(side, tp, cp) @ self.E(t, cp).conj().T)
            Zs = np.vstack(rows) if rows else np.zeros((0, k), dtype=np.complex128)
            self._Z[key] = qr_r(Zs, k)
        return self._Z[key]

    # truncation: returns (sigma, rank, Q or (F1, F2), C)
    def truncate(self, side, t, c):
        key = (side, t, c)
        if key not in self._T:
            st, ct = self.st, self.st.ct
            if ct.is_leaf(t):
                Vt = self.V(t, c)
            else:
                c2 = st.sd(int(ct.level[t]), c)
                Vt = np.vstack([self.truncate(side, int(ch), c2)["C"] @ self.E(int(ch), c) for ch in ct.children[t]])
            U, s = svd_left(Vt @ self.Zhat(side, t, c).conj().T)
            kk = select_rank(s, self.eps, self.mode)
            Q = U[:, :kk]
            self._T[key] = {"sigma": s, "rank": kk, "Q": Q, "C": Q.conj().T @ Vt}
        return self._T[key]
